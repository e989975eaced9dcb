"""Does splitting a step into channel halves on two streams hide the
latency-bound kernels?  Times (graph replay, L2 flushed) the plain step and
the 2-stream split step of one config.

    python tools/overlap_probe.py C2 [parts]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2409_14355_b200 import _lib
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[name]
d = generate(cfg)
c = constellation_for(cfg.order)
dev = torch.device("cuda", 0)
main = torch.cuda.Stream(dev)
torch.cuda.set_stream(main)
h = torch.from_numpy(d["h"]).to(dev)
y = torch.from_numpy(d["y"]).to(dev)
nv = float(d["nv"][0])
lib = _lib.load()
plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
ex = plan.expansions
n_ch, V = y.shape[0], y.shape[1]
hard = torch.empty((n_ch, V, cfg.n), dtype=torch.uint8, device=dev)
metric = torch.empty((n_ch, V), dtype=torch.float32, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
bounds = [round(i * n_ch / parts) for i in range(parts + 1)]
wss = [torch.empty(int(lib.mpnl_workspace_bytes((b1 - b0) * V, cfg.n, cfg.order, ex.ctypes.data)),
                   dtype=torch.uint8, device=dev) for b0, b1 in zip(bounds, bounds[1:])]
streams = [torch.cuda.Stream(dev) for _ in range(parts)]
ws_all = torch.empty(int(lib.mpnl_workspace_bytes(n_ch * V, cfg.n, cfg.order, ex.ctypes.data)),
                     dtype=torch.uint8, device=dev)


def stages(p, c0, c1, ws, st):
    tl = p.tables.numel() // n_ch
    args = (p.perm_dev[c0:].data_ptr(), p.r_dev[c0:].data_ptr(), p.qh_dev[c0:].data_ptr(),
            p.tables.view(-1)[c0 * tl:].data_ptr(), y[c0:].data_ptr(), 0, c1 - c0, V, cfg.m,
            cfg.n, cfg.order, ex.ctypes.data, nv, hard[c0:].data_ptr(), metric[c0:].data_ptr(),
            None, ws.data_ptr(), ws.numel(), st.cuda_stream)
    for s in range(1, 5):
        _lib.check(lib.mpnl_detect_hard_stage(s, *args), f"stage{s}")


def step_plain():
    p = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    stages(p, 0, n_ch, ws_all, main)


def step_split():
    p = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    ev = torch.cuda.Event()
    ev.record(main)
    for i, st in enumerate(streams):
        st.wait_event(ev)
        stages(p, bounds[i], bounds[i + 1], wss[i], st)
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        main.wait_event(e)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(main)
        g.replay()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


tp = timed(step_plain)
ref_h, ref_m = hard.clone(), metric.clone()
ts = timed(step_split)
same = bool(torch.equal(ref_h, hard) and torch.equal(ref_m, metric))
print(f"{name}: plain {tp * 1e3:.1f} us, split x{parts} {ts * 1e3:.1f} us, identical {same}")
