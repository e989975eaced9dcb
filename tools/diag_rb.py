"""Diagnose an RB whose GPU hard output differs from the cached reference run.
usage: python tools/diag_rb.py C4 60"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

name, rb = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
c = constellation_for(cfg.order)
d = generate(cfg, n_rb=1, rb_offset=rb)
z = np.load(ROOT / "baseline" / "_ref" / "oracle_full" / f"{name}.npz")
ref, m1, m2 = z["hard"][rb], z["m1"][rb], z["m2"][rb]
h = torch.from_numpy(d["h"]).cuda()
y = torch.from_numpy(d["y"]).cuda()
nv = float(d["nv"][0])
plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
oplan = orc.plan_channels(d["h"], nv, cfg.n_paths, cfg.order)
print("perm equal:", np.array_equal(plan.perm, oplan.perm), "R maxdiff",
      np.abs(plan.r - oplan.r).max(), "expansions", plan.expansions[::-1][:4])
hard, metric, flags = det.mpnl_detect_hard(plan, h, y, c, return_flags=True)
hard = hard.cpu().numpy()[0]
metric = metric.cpu().numpy()[0]
flags = flags.cpu().numpy()[0]
bad = np.nonzero(np.any(hard != ref, axis=-1))[0]
print("mismatching vectors:", bad.tolist())
lab, met, best = det.mpnl_detect_batch(plan, h, y, c)
lab, met, best = lab.cpu().numpy()[0], met.cpu().numpy()[0], best.cpu().numpy()[0]
for v in bad[:10]:
    print(f"v={v} flag={flags[v]} gpu_metric={metric[v]!r} ref m1={m1[v]!r} m2={m2[v]!r}")
    print("   gpu hard ", hard[v].tolist())
    print("   ref hard ", ref[v].tolist())
    print("   fp64 full-list best", best[v], "label", lab[v, best[v]].tolist(), "metric",
          met[v, best[v]])
    # oracle on this vector
    oh, om1, om2 = orc.detect_rb(d["h"], d["y"][:, v:v + 1], nv, cfg.n_paths, cfg.order,
                                 c.points)
    print("   oracle   ", oh[0, 0].tolist(), om1[0, 0], om2[0, 0])
    gp = np.nonzero(np.all(lab[v] == hard[v], axis=-1))[0]
    rp = np.nonzero(np.all(lab[v] == ref[v], axis=-1))[0]
    print("   path of gpu hard in full list:", gp.tolist(), "path of ref hard:", rp.tolist())
