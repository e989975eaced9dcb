"""Warm per-stage device times of one plan + hard-detection step (CUDA events
around each C-ABI stage on the launching stream, L2 flushed before each step).

    python tools/stage_times.py C2 [reps]

stage 0 = plan (QR + tables), 1 = reset + prep + select, 2 = traversal,
3 = verify + check, 4 = fp64 fix-up."""
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
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pv = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # > 0: pv instances, one channel each (V = 1)
cfg = CONFIGS[name]
d = generate(cfg, n_rb=pv) if pv else generate(cfg)
if pv:
    d["y"] = np.ascontiguousarray(d["y"][:, :1])
c = constellation_for(cfg.order)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
h = torch.from_numpy(d["h"]).to(dev)
y = torch.from_numpy(d["y"]).to(dev)
nv = float(d["nv"][0])
lib = _lib.load()
plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
ex = plan.expansions
nvec = y.shape[0] * y.shape[1]
hard = torch.empty((y.shape[0], y.shape[1], cfg.n), dtype=torch.uint8, device=dev)
metric = torch.empty((y.shape[0], y.shape[1]), dtype=torch.float32, device=dev)
ws = torch.empty(int(lib.mpnl_workspace_bytes(nvec, cfg.n, cfg.order, ex.ctypes.data)),
                 dtype=torch.uint8, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
times = np.zeros((reps, 5))
for r in range(reps + 3):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record(stream)
    p = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    ev[1].record(stream)
    args = (p.perm_dev.data_ptr(), p.r_dev.data_ptr(), p.qh_dev.data_ptr(), p.tables.data_ptr(),
            y.data_ptr(), 0, y.shape[0], y.shape[1], cfg.m, cfg.n, cfg.order, ex.ctypes.data, nv,
            hard.data_ptr(), metric.data_ptr(), None, ws.data_ptr(), ws.numel(), stream.cuda_stream)
    for s in range(1, 5):
        _lib.check(lib.mpnl_detect_hard_stage(s, *args), f"stage{s}")
        ev[s + 1].record(stream)
    torch.cuda.synchronize()
    if r >= 3:
        times[r - 3] = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(5)]
med = np.median(times, axis=0)
names = ["plan", "prep+select", "traverse", "verify+check", "fixup"]
print(name, f"{nvec} vectors; median us per stage:",
      ", ".join(f"{n} {t:.1f}" for n, t in zip(names, med)), f"| total {med.sum():.1f}")
