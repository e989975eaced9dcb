"""Roofline measurement of the list-LLR kernel (`mpnl_candidate_llrs`).

Full C2-shaped candidate lists (45,864 vectors = 273 RB x 168 RE at one SNR, P = 64,
N = 12, 16-QAM) resident in HBM: labels (B,P,N) uint8 + metrics (B,P) fp64 in,
LLRs (B,N,4) fp64 out.  Algorithmic bytes per vector = P(N + 8) + 8 N log2Q.
Kernel time by CUDA events on the launching stream (L2 flushed before each
rep), achieved GB/s vs the measured HBM peak.  Also checks the output against
the oracle on a sample.  Prints one JSON line.

    python tools/llr_bench.py [B] [P] [N] [Q]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200 import detect as det
from paper_2409_14355_b200.core import constellation_for

B = int(sys.argv[1]) if len(sys.argv) > 1 else 45864
P = int(sys.argv[2]) if len(sys.argv) > 2 else 64
N = int(sys.argv[3]) if len(sys.argv) > 3 else 12
Q = int(sys.argv[4]) if len(sys.argv) > 4 else 16
c = constellation_for(Q)
bps = c.bits_per_symbol
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
lab = torch.randint(0, Q, (B, P, N), dtype=torch.uint8, device=dev, generator=g)
met = torch.rand((B, P), dtype=torch.float64, device=dev, generator=g) * 20.0
nv = 0.25
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    out = det._candidate_llrs_batch(lab, met, nv, c)
torch.cuda.synchronize()
ts = []
st = torch.cuda.current_stream()
for _ in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    out = det._candidate_llrs_batch(lab, met, nv, c)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
t = float(np.median(ts))
bytes_per_vec = P * (N + 8) + 8 * N * bps
k = 512
ok = np.array_equal(out[:k].cpu().numpy(),
                    orc.candidate_llrs(lab[:k].cpu().numpy(), met[:k].cpu().numpy(), nv, Q),
                    equal_nan=True)
try:
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = float(next(v for k_, v in peaks.items() if "hbm" in k_.lower() and
                     isinstance(v, (int, float))))
    src = "MEASURED_PEAKS.json"
except Exception:
    hbm, src = 6456.2, "B200_PROFILING.md fallback"
gbs = B * bytes_per_vec / t / 1e9
print(json.dumps({"kernel": "candidate_llr_kernel", "workload": f"B={B} P={P} N={N} Q={Q}",
                  "vectors_per_s": B / t, "us": t * 1e6, "bytes_per_vector": bytes_per_vec,
                  "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm,
                               "unit": "GB/s", "frac": round(gbs / hbm, 3), "peak_source": src},
                  "matches_oracle": bool(ok), "l2": "flushed before each rep"}))
