"""Link-level frames/s: the GPU simulate_frames vs the reference's
(linksim.py:159-232) on the same configuration, one channel, a batch of frames
(measure_per takes 25 at a time).

    python tools/linksim_bench.py [frames] [detector] [n_streams] [m] [rb]"""
import json
import sys
import time
from fractions import Fraction
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2409_14355_b200 import linksim as L
from paper_2409_14355_b200.core import constellation_for

f = int(sys.argv[1]) if len(sys.argv) > 1 else 25
det = sys.argv[2] if len(sys.argv) > 2 else "mpnl"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
m = int(sys.argv[4]) if len(sys.argv) > 4 else 8
rb = int(sys.argv[5]) if len(sys.argv) > 5 else 2
q, rate = 16, Fraction(245, 512)
rng = np.random.default_rng(1)
h = (rng.standard_normal((14, 12 * rb, m, n)) + 1j * rng.standard_normal((14, 12 * rb, m, n))) / np.sqrt(2)
nv = n / 10 ** (11.0 / 10)
mcs = SimpleNamespace(constellation=constellation_for(q), code_rate=rate)
cfg = L.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, rb_per_vehicle=rb, detector=det, n_paths=32)
for _ in range(2):
    L.simulate_frames(cfg, h, nv, 0, range(f))
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = 5
for r in range(reps):
    ok = L.simulate_frames(cfg, h, nv, 0, range(r * f, (r + 1) * f))
gpu_s = (time.perf_counter() - t0) / reps
line = {"what": "simulate_frames (one channel, a batch of frames), wall clock incl. host RNG",
        "config": f"{n}x{m} 16-QAM r={rate}, {rb} RB, detector {det} P=32, genie CSI, {f} frames",
        "gpu_frames_per_s": round(f / gpu_s, 1), "gpu_ms_per_batch": round(gpu_s * 1e3, 2)}
if det == "mpnl":   # the fp32 soft output (fused traversal + LLR kernel)
    for _ in range(2):
        L.simulate_frames(cfg, h, nv, 0, range(f), soft_precision="fp32")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(reps):
        ok32 = L.simulate_frames(cfg, h, nv, 0, range(r * f, (r + 1) * f), soft_precision="fp32")
    s32 = (time.perf_counter() - t0) / reps
    line["gpu_fp32_soft_frames_per_s"] = round(f / s32, 1)
    line["fp32_soft_outcomes_equal_fp64"] = bool(np.array_equal(ok32, ok))
try:
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    sys.dont_write_bytecode = True
    from mpnlsim import channel, core, linksim
    rmcs = next(e for e in core.MCS_TABLE if e.modulation_order == q and e.code_rate == rate)
    rcfg = linksim.LinkConfig(n_streams=n, m_antennas=m, mcs=rmcs, detector=det, n_paths=32,
                              rb_per_vehicle=rb)
    t0 = time.perf_counter()
    rok = linksim.simulate_frames(rcfg, channel.ChannelGrid(h=h), nv, 0, range(f))
    ref_s = time.perf_counter() - t0
    gok = L.simulate_frames(cfg, h, nv, 0, range(f))
    line["reference_frames_per_s"] = round(f / ref_s, 2)
    line["reference_cores"] = 1
    line["outcomes_identical"] = bool(np.array_equal(rok, gok))
except ImportError:
    pass
print(json.dumps(line), flush=True)
