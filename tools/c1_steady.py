"""C1 steady state and the per-vector-channel shape.

    python tools/c1_steady.py [K] [B_pv]

1. C1 (8x8 16-QAM P=32, 4 RB x 168 RE = 672 vectors): single-shot latency of
   plan + hard detection (CUDA events, eager launches), and the steady state of
   K back-to-back C1 batches replayed as ONE CUDA graph (time / K).
2. The reference's own bench shape (cli.py:223-247, `mpnlsim bench`: one H per
   instance, README config 8x8 16-QAM P=32, 8192 instances): n_ch = B
   channels with V = 1 vector each, plan + detect through the same C ABI;
   the unmodified reference on host cores on a sample of the same instances.
Prints one JSON line per measurement (bench-line fields + roofline)."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2409_14355_b200 import _lib
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
BPV = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
PEAK = 148 * 128 * 2 * 1.965e9
cfg = CONFIGS["C1"]
c = constellation_for(cfg.order)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
lib = _lib.load()


def make_step(h, y, nv):
    plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    ex = plan.expansions
    nvec = y.shape[0] * y.shape[1]
    hard = torch.empty((y.shape[0], y.shape[1], cfg.n), dtype=torch.uint8, device=dev)
    metric = torch.empty((y.shape[0], y.shape[1]), dtype=torch.float32, device=dev)
    ws = torch.empty(int(lib.mpnl_workspace_bytes(nvec, cfg.n, cfg.order, ex.ctypes.data)),
                     dtype=torch.uint8, device=dev)

    def step():
        p = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
        _lib.check(lib.mpnl_detect_hard(p.perm_dev.data_ptr(), p.r_dev.data_ptr(),
                                        p.qh_dev.data_ptr(), p.tables.data_ptr(), y.data_ptr(), 0,
                                        y.shape[0], y.shape[1], cfg.m, cfg.n, cfg.order,
                                        ex.ctypes.data, nv, hard.data_ptr(), metric.data_ptr(),
                                        None, ws.data_ptr(), ws.numel(), stream.cuda_stream),
                   "detect")
    return step, plan, hard, metric, nvec


def ev_time(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


# ---- 1. C1 single shot + K-batch graph ----
d = generate(cfg)
h = torch.from_numpy(d["h"]).to(dev)
y = torch.from_numpy(d["y"]).to(dev)
nv = float(d["nv"][0])
step, plan, hard, metric, nvec = make_step(h, y, nv)
for _ in range(5):
    step()
single_ms = ev_time(step, 20)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for _ in range(K):
        step()
g.replay()
torch.cuda.synchronize()
graph_ms = ev_time(g.replay, 5)
fl = cfg.flops_per_vector(plan.n_paths)
per_batch = graph_ms / K
print(json.dumps({
    "metric": "detected MIMO vectors/sec", "unit": "vectors/s", "config": {
        "workload": f"C1: 8x8 16-QAM P={plan.n_paths}, 4 RB x 168 RE = {nvec} vectors"},
    "single_shot": {"ms": round(single_ms, 4), "vectors/s": round(nvec / (single_ms * 1e-3), 1),
                    "frac": round(nvec * fl / (single_ms * 1e-3) / PEAK, 5)},
    "steady_state": {"batches": K, "ms_per_batch": round(per_batch, 4),
                     "vectors/s": round(nvec / (per_batch * 1e-3), 1),
                     "frac": round(nvec * fl / (per_batch * 1e-3) / PEAK, 5),
                     "how": f"{K} dependent plan+detect steps captured as one CUDA graph"},
    "note": "launch-latency bound: 672 vectors are ~0.1 us of FP32 work at peak"}), flush=True)

# ---- 2. per-vector channels (the reference's cli bench shape) ----
dd = generate(cfg, n_rb=BPV, seed=77)
hpv = torch.from_numpy(dd["h"]).to(dev)                   # (B, 8, 8): one H per instance
ypv = torch.from_numpy(np.ascontiguousarray(dd["y"][:, :1])).to(dev)   # (B, 1, 8)
step2, plan2, hard2, metric2, nvec2 = make_step(hpv, ypv, nv)
for _ in range(3):
    step2()
pv_ms = ev_time(step2, 10)
line = {"metric": "detected MIMO vectors/sec", "unit": "vectors/s", "config": {
    "workload": f"per-vector channels (cli.py:223-247 shape): {nvec2} instances of 8x8 16-QAM "
                f"P={plan2.n_paths}, one H each"},
    "value": round(nvec2 / (pv_ms * 1e-3), 1), "ms_per_step": round(pv_ms, 4),
    "roofline": {"bound": "fp32", "frac": round(nvec2 * fl / (pv_ms * 1e-3) / PEAK, 5)}}
try:
    from oracle import reference_runner as rr
    if rr.available():
        cores = len(os.sched_getaffinity(0))
        nsmp = min(BPV, 64 * cores)
        tasks = [(dd["h"][i:i + 1], dd["y"][i:i + 1, :1], nv, cfg.n_paths, cfg.order)
                 for i in range(nsmp)]
        with rr.make_pool(cores) as pool:
            list(pool.map(int, [0] * cores))
            t0 = time.perf_counter()
            outs = list(pool.map(rr.detect_rb_hard, tasks, chunksize=8))
            dt = time.perf_counter() - t0
        ref_hard = np.concatenate([o[0] for o in outs])[:, 0]
        gh = hard2[:nsmp, 0].cpu().numpy()
        m1 = np.concatenate([o[1] for o in outs])[:, 0]
        m2 = np.concatenate([o[2] for o in outs])[:, 0]
        bad = np.any(gh != ref_hard, axis=-1) & ~((m2 - m1) <= 1e-5 * m1)
        line["cpu_baseline"] = {"value": round(nsmp / dt, 1), "unit": "vectors/s",
                                "cores": cores, "kind": "reference",
                                "sample": f"{nsmp} instances, plan per instance (as cli.py)"}
        line["parity"] = {"vectors": int(nsmp), "non_exempt_mismatches": int(bad.sum())}
except Exception as e:   # noqa: BLE001
    line["cpu_baseline"] = {"unavailable": str(e)}
print(json.dumps(line), flush=True)
