"""Probe the host pipeline: H2D/D2H bandwidth and mpnl_hard_output vs chunking."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
c = constellation_for(cfg.order)
d = generate(cfg)
nv = float(d["nv"][0])
h = torch.from_numpy(d["h"]).pin_memory()
y = torch.from_numpy(d["y"]).pin_memory()
yd = torch.empty(y.shape, dtype=y.dtype, device="cuda")
s = torch.cuda.current_stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    return min(t[0] for t in ts), min(t[1] for t in ts)


nb = y.numel() * 8
ms, _ = timeit(lambda: yd.copy_(y, non_blocking=True))
print(f"H2D {nb/1e6:.1f} MB: {ms:.3f} ms = {nb/ms/1e6:.1f} GB/s")
yh = torch.empty_like(y).pin_memory()
ms, _ = timeit(lambda: yh.copy_(yd, non_blocking=True))
print(f"D2H {nb/1e6:.1f} MB: {ms:.3f} ms = {nb/ms/1e6:.1f} GB/s")
out = (torch.empty((y.shape[0], y.shape[1], cfg.n), dtype=torch.uint8).pin_memory(),
       torch.empty((y.shape[0], y.shape[1]), dtype=torch.float32).pin_memory())
for ch in (cfg.n_rb, -(-cfg.n_rb // 2), -(-cfg.n_rb // 4), -(-cfg.n_rb // 6),
           -(-cfg.n_rb // 12), -(-cfg.n_rb // 24)):
    ms, wall = timeit(lambda: det.mpnl_hard_output(h, y, nv, cfg.n_paths, c, chunk_channels=ch,
                                                   out=out))
    print(f"chunk {ch:5d} channels: {ms:.3f} ms (wall {wall:.3f} ms) -> {y.shape[0]*y.shape[1]/ms/1e3:.3e} vec/s")
