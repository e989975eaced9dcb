"""One plan + hard detection of a config (for ncu captures).
usage: python tools/profile_one.py C2 [n_rb] [reps] [soft]   (soft: also the fp32 soft output)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
n_rb = (int(sys.argv[2]) or cfg.n_rb) if len(sys.argv) > 2 else cfg.n_rb
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = generate(cfg, n_rb=n_rb)
c = constellation_for(cfg.order)
h = torch.from_numpy(d["h"]).cuda()
y = torch.from_numpy(d["y"]).cuda()
from paper_2409_14355_b200 import _lib
lib = _lib.load()
plan = det.mpnl_plan_batch(h, float(d["nv"][0]), cfg.n_paths, c)
ws = torch.empty(int(lib.mpnl_workspace_bytes(y.shape[0] * y.shape[1], cfg.n, cfg.order,
                                              plan.expansions.ctypes.data)),
                 dtype=torch.uint8, device="cuda")
for _ in range(reps):
    plan = det.mpnl_plan_batch(h, float(d["nv"][0]), cfg.n_paths, c)
    hard, metric, flags = det.mpnl_detect_hard(plan, h, y, c, return_flags=True, workspace=ws)
if len(sys.argv) > 4 and sys.argv[4] == "soft":
    det.mpnl_detect_llrs(plan, h, y[:, :168].contiguous(), c, precision="fp32")
torch.cuda.synchronize()
nv_ = y.shape[0] * y.shape[1]
st = det.workspace_stats(ws)
print(name, "vectors", nv_, "flag rate", float(flags.float().mean()),
      "per vector (last call):", {k: v / nv_ for k, v in st.items()})
