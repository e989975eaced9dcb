"""LDPC decoder throughput on one B200.

    python tools/ldpc_bench.py [--words 16384] [--snr 2.5 1.0] [--reps 10]

Device-resident float64 LLRs of seeded AWGN-BPSK codewords of the default
rate-1/2 code (n = 1296), decoded with max_iter = 10 (CUDA events, L2 flushed
between reps).  Prints one JSON line per SNR point: codewords/s, info Gbit/s,
mean iterations, the HBM roofline of the LLR stream (n*8 B in, k B + 1 out per
word) and the fp64 pipe utilisation of the edge arithmetic (2 DADD per edge
and iteration + 2 DMUL per check and iteration), plus the reference decoder
(`mpnlsim.fec.ldpc_decode`, numpy, one process) on a sample of the same LLRs
when it is importable.
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

from paper_2409_14355_b200 import fec

ap = argparse.ArgumentParser()
ap.add_argument("--words", type=int, default=16384)
ap.add_argument("--snr", type=float, nargs="+", default=[2.5, 1.0])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--ref-words", type=int, default=256)
a = ap.parse_args()

code = fec.default_code()
n, k = code.n, code.k
m = n - k
edges = int(code.parity_check.sum())
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
hbm = peaks.get("hbm_gbs", 6549.8)
fp64_peak = 148 * 64 * 1.965e9   # DP instructions/s (64 fp64 lanes per SM per clock)
for snr in a.snr:
    rng = np.random.default_rng(int(snr * 1000))
    info = torch.from_numpy(rng.integers(0, 2, (a.words, k)).astype(np.uint8)).to(dev)
    tx = fec.ldpc_encode(code, info)
    nv = 10 ** (-snr / 10)
    noise = torch.from_numpy(rng.normal(0, np.sqrt(nv), (a.words, n))).to(dev)
    llr = (2 * ((1 - 2.0 * tx.double()) + noise) / nv).contiguous()
    for _ in range(2):
        dec, conv, iters = fec.ldpc_decode(code, llr, return_iterations=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        dec, conv, iters = fec.ldpc_decode(code, llr, return_iterations=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    it_mean = float(iters.float().mean())
    cw_s = a.words / (ms * 1e-3)
    bytes_alg = a.words * (8 * n + k + 1)
    dp_ops = float(iters.double().sum()) * (2 * edges + 2 * m) + a.words * edges   # + final syndrome pass subs
    line = {"what": "ldpc_decode (normalized min-sum, fp64, bit-identical)", "snr_db": snr,
            "words": a.words, "ms": round(ms, 4), "codewords/s": round(cw_s, 1),
            "info_gbit_s": round(cw_s * k / 1e9, 3), "mean_iterations": round(it_mean, 3),
            "converged": float(conv.float().mean()),
            "hbm": {"algorithmic_bytes": bytes_alg, "achieved_gbs": round(bytes_alg / (ms * 1e-3) / 1e9, 1),
                    "peak_gbs": hbm, "frac": round(bytes_alg / (ms * 1e-3) / 1e9 / hbm, 4)},
            "fp64": {"dp_ops": dp_ops, "achieved_gops": round(dp_ops / (ms * 1e-3) / 1e9, 1),
                     "peak_gops": round(fp64_peak / 1e9, 1),
                     "frac": round(dp_ops / (ms * 1e-3) / fp64_peak, 4)}}
    try:
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        from mpnlsim import fec as rfec
        rc = rfec.default_code()
        sample = llr[:a.ref_words].cpu().numpy()
        t0 = time.perf_counter()
        rdec, rconv = rfec.ldpc_decode(rc, sample)
        dt = time.perf_counter() - t0
        line["reference_cpu"] = {"codewords/s": round(a.ref_words / dt, 1), "cores": 1,
                                 "sample_words": a.ref_words,
                                 "bit_identical": bool(np.array_equal(rdec, dec[:a.ref_words].cpu().numpy())
                                                       and np.array_equal(rconv, conv[:a.ref_words].cpu().numpy()))}
    except ImportError:
        pass
    print(json.dumps(line), flush=True)
