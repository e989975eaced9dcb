"""e2e host-pipeline time vs chunk count: python tools/e2e_chunks.py C2"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
d = generate(cfg)
c = constellation_for(cfg.order)
h = torch.from_numpy(d["h"]).pin_memory()
y = torch.from_numpy(d["y"]).pin_memory()
nv = float(d["nv"][0])
n_ch = h.shape[0]
out = (torch.empty((n_ch, y.shape[1], cfg.n), dtype=torch.uint8).pin_memory(),
       torch.empty((n_ch, y.shape[1]), dtype=torch.float32).pin_memory())
torch.cuda.set_device(0)
for chunks in (1, 2, 3, 4, 6, 8, 12, 16):
    cc = max(1, -(-n_ch // chunks))
    ts = []
    for i in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        det.mpnl_hard_output(h, y, nv, cfg.n_paths, c, chunk_channels=cc, out=out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(f"{name} chunks {chunks} ({cc} ch): {ms:.3f} ms -> {y.shape[0] * y.shape[1] / ms / 1e3:.3e} vec/s")
