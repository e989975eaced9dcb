"""Whole-job device time of plan + hard detection through mpnl_plan_detect_hard
for 1..4 channel groups (CUDA graph replay, L2 flushed before each step), and
identity of the outputs with the single-stream path.

    python tools/group_times.py C2 [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[name]
d = generate(cfg)
c = constellation_for(cfg.order)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
h = torch.from_numpy(d["h"]).to(dev)
y = torch.from_numpy(d["y"]).to(dev)
nv = float(d["nv"][0])
plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
ref_h, ref_m = det.mpnl_detect_hard(plan, h, y, c)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = []
for g in (1, 2, 3, 4):
    out = (torch.empty_like(ref_h), torch.empty_like(ref_m))
    for _ in range(3):
        det.mpnl_hard_output_device(h, y, nv, cfg.n_paths, c, groups=g, out=out)
    torch.cuda.synchronize()
    same = bool(torch.equal(out[0], ref_h) and torch.equal(out[1], ref_m))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        det.mpnl_hard_output_device(h, y, nv, cfg.n_paths, c, groups=g, out=out)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    same = same and bool(torch.equal(out[0], ref_h) and torch.equal(out[1], ref_m))
    res.append(f"g={g} {np.median(ts):.1f}us same={same}")
print(name, " | ".join(res))
