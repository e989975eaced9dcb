"""Soft-output (list max-log LLR) path throughput: the link simulator's MPNL
branch (linksim.py:151-155) = mpnl_plan_batch + mpnl_detect_batch (the fp64
full candidate list, exact_kernel) + _candidate_llrs_batch (candidate_llr_kernel).

    python tools/soft_bench.py [CFG] [n_rb] [check_rb]

Device-resident seeded inputs of a BASELINE config (first SNR point); CUDA
events per stage (L2 flushed between reps); the end-to-end call through the
public shim `detect.mpnl_detect_llrs` with host numpy in / out; LLR parity
against the CPU oracle (fp64 full list -> candidate_llrs) on `check_rb` RBs
(tolerance: LLRs within 1e-9 * max(metric) / nv absolute, saturated ones equal).
Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
n_rb = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_rb
check_rb = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = generate(cfg, n_rb=n_rb)
c = constellation_for(cfg.order)
V = 168
h_np, y_np = d["h"], np.ascontiguousarray(d["y"][:, :V])
nv = float(d["nv"][0])
dev = torch.device("cuda", 0)
h, y = torch.from_numpy(h_np).to(dev), torch.from_numpy(y_np).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
B = n_rb * V
reps = 5


def timed(fn):
    ts = []
    out = None
    for r in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
t_plan, _ = timed(lambda: det.mpnl_plan_batch(h, nv, cfg.n_paths, c))
t_list, (lab, met, best) = timed(lambda: det.mpnl_detect_batch(plan, h, y, c))
P = lab.shape[-2]
t_llr, llr = timed(lambda: det._candidate_llrs_batch(lab.reshape(-1, P, cfg.n),
                                                     met.reshape(-1, P), nv, c))
# fp32 fused traversal + LLR kernel (mpnl_detect_llrs_fast) + fp64 recomputation of flagged vectors
t_fast, (llr_fast, fl_fast) = timed(lambda: det.mpnl_detect_llrs(plan, h, y, c, precision="fp32",
                                                                 return_flags=True))
fast_err = (llr_fast - llr.reshape(llr_fast.shape)).abs()
fast_scale = 2.0 * met.max(dim=-1).values / nv
fast_rel = float((fast_err / fast_scale[..., None, None]).max().item())
t0 = time.perf_counter()
for _ in range(3):
    pl = det.mpnl_plan_batch(h_np, nv, cfg.n_paths, c)
    det.mpnl_detect_llrs(pl, h_np, y_np, c, precision="fp32")
e2e_fast_s = (time.perf_counter() - t0) / 3
# end to end through the public shim from host numpy arrays
t0 = time.perf_counter()
for _ in range(3):
    pl = det.mpnl_plan_batch(h_np, nv, cfg.n_paths, c)
    llr_np = det.mpnl_detect_llrs(pl, h_np, y_np, c)
e2e_s = (time.perf_counter() - t0) / 3
# parity vs the oracle on the first check_rb RBs
ok = True
worst = 0.0
for rb in range(min(check_rb, n_rb)):
    op = orc.plan_channels(h_np[rb:rb + 1], nv, cfg.n_paths, cfg.order).tile(V)
    olab, omet, _ = orc.detect_batch(op, np.repeat(h_np[rb:rb + 1].astype(complex), V, 0),
                                     y_np[rb].astype(complex), c.points)
    ollr = orc.candidate_llrs(olab, omet, nv, cfg.order)
    g = llr_np[rb]
    tol = 1e-9 * omet.max() / nv
    sat = np.abs(ollr) >= 20.0
    err = np.where(sat, (g != ollr) * 1.0, np.abs(g - ollr))
    worst = max(worst, float(np.max(np.where(sat, 0, err))))
    ok &= bool(np.all(g[sat] == ollr[sat]) and np.all(err[~sat] <= tol))
bps = c.bits_per_symbol
llr_bytes = B * (P * (cfg.n + 8) + 8 * cfg.n * bps)
print(json.dumps({
    "what": "soft output: plan + fp64 full list (mpnl_detect_batch) + list max-log LLRs",
    "config": f"{name}: {cfg.n}x{cfg.m} {cfg.order}-QAM P={P}, {n_rb} RB x {V} RE = {B} vectors",
    "ms": {"plan": round(t_plan, 4), "full_list": round(t_list, 4), "llr": round(t_llr, 4)},
    "device_vectors_per_s": round(B / ((t_plan + t_list + t_llr) * 1e-3), 1),
    "e2e_vectors_per_s": round(B / e2e_s, 1),
    "e2e_api": "detect.mpnl_plan_batch + detect.mpnl_detect_llrs, host numpy in/out",
    "llr_kernel_hbm_gbs": round(llr_bytes / (t_llr * 1e-3) / 1e9, 1),
    "parity": {"rbs": min(check_rb, n_rb), "ok": ok, "max_abs_err_unsaturated": worst},
    "fp32": {"what": "detect.mpnl_detect_llrs(precision='fp32'): prep + fused fp32 traversal/LLR "
                     "kernel + fp64 recomputation of flagged vectors",
             "ms": round(t_fast, 4),
             "device_vectors_per_s": round(B / ((t_plan + t_fast) * 1e-3), 1),
             "e2e_vectors_per_s": round(B / e2e_fast_s, 1),
             "recomputed_fraction": float(fl_fast.float().mean().item()),
             "max_err_over_2maxmetric_by_nv": fast_rel,
             "speedup_vs_fp64_list": round((t_list + t_llr) / t_fast, 2)},
}), flush=True)
