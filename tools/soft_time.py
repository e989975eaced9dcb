"""Device time of the fp32 soft-output call (prep + fused traversal/LLR kernel,
C-ABI mpnl_detect_llrs_fast; CUDA events over 10 calls) and its flagged fraction.

    python tools/soft_time.py CFG n_rb"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2409_14355_b200 import detect as det, _lib
from paper_2409_14355_b200.core import constellation_for, LLR_CLIP
from paper_2409_14355_b200.workloads import CONFIGS, generate
name, n_rb = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]; d = generate(cfg, n_rb=n_rb); c = constellation_for(cfg.order)
nv = float(d["nv"][0])
h = torch.from_numpy(d["h"]).cuda(); y = torch.from_numpy(np.ascontiguousarray(d["y"][:, :168])).cuda()
plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
lib = _lib.load()
nch, v, m = y.shape; n = cfg.n; bps = c.bits_per_symbol
ws = torch.empty(int(lib.mpnl_workspace_bytes(nch*v, n, c.order, plan.expansions.ctypes.data)), dtype=torch.uint8, device='cuda')
llr = torch.empty((nch, v, n, bps), dtype=torch.float64, device='cuda'); flags = torch.empty((nch, v), dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream().cuda_stream
def run():
    return lib.mpnl_detect_llrs_fast(plan.perm_dev.data_ptr(), plan.r_dev.data_ptr(), plan.qh_dev.data_ptr(), plan.tables.data_ptr(), y.data_ptr(), 0, nch, v, m, n, c.order, plan.expansions.ctypes.data, plan.noise_var, nv, float(LLR_CLIP), llr.data_ptr(), flags.data_ptr(), ws.data_ptr(), ws.numel(), st)
for _ in range(3): run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
print(name, nch*v, "vectors: prep + soft kernel ms", e0.elapsed_time(e1)/10, "flag frac", flags.float().mean().item(), "nv", nv)
