"""Throughput of the batched ZF / MMSE kernel (mpnl_linear_detect) on one GPU.

    python tools/linear_bench.py [M N Q mode B]

Device-resident inputs, CUDA events around `iters` launches on the current
stream; prints one JSON line (vectors/s, GB/s of algorithmic bytes:
16 (M N + M) in + N (1 + 8 log2 Q) out per vector)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_14355_b200 import _lib  # noqa: E402
from paper_2409_14355_b200.core import constellation_for  # noqa: E402


def main():
    a = sys.argv[1:]
    m, n, q = (int(a[0]), int(a[1]), int(a[2])) if len(a) >= 3 else (12, 12, 16)
    mode = a[3] if len(a) >= 4 else "mmse"
    b = int(a[4]) if len(a) >= 5 else 275184
    c = constellation_for(q)
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn((b, m, n), dtype=torch.complex128, device="cuda", generator=g) / m ** 0.5
    y = torch.randn((b, m), dtype=torch.complex128, device="cuda", generator=g)
    lab = torch.empty((b, n), dtype=torch.uint8, device="cuda")
    llr = torch.empty((b, n, c.bits_per_symbol), dtype=torch.float64, device="cuda")
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream

    def run():
        rc = lib.mpnl_linear_detect(h.data_ptr(), y.data_ptr(), b, m, n, q,
                                    {"zf": 0, "mmse": 1}[mode], 0.05, None, 20.0,
                                    lab.data_ptr(), llr.data_ptr(), None, None, s)
        _lib.check(rc, "linear")
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    iters = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    byt = b * (16 * (m * n + m) + n * (1 + 8 * c.bits_per_symbol))
    # algorithmic fp64 flops: Gram lower triangle 4MN(N+1) + H^H y 8MN + Cholesky
    # 4N^3/3 + two triangular solves 8N^2 + diag(A^-1) via L^-1 4N^3/3
    fl = b * (4 * m * n * (n + 1) + 8 * m * n + 8 * n ** 3 / 3 + 8 * n * n)
    fp64_peak = 148 * 64 * 2 * 1.965e9
    hbm = 6549.8e9
    t = ms * 1e-3
    print(json.dumps({"kernel": "linear_detect_kernel", "mode": mode, "M": m, "N": n, "Q": q,
                      "vectors": b, "ms": round(ms, 4), "vectors_per_s": b / t,
                      "algorithmic_GBps": byt / t / 1e9, "hbm_frac": round(byt / t / hbm, 4),
                      "fp64_tflops": fl / t / 1e12, "fp64_frac": round(fl / t / fp64_peak, 4),
                      "bound": "hbm" if byt / hbm > fl / fp64_peak else "fp64"}))


if __name__ == "__main__":
    main()
