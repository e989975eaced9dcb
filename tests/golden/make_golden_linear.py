"""Golden ZF / MMSE fixtures from the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_linear.py

Runs the reference's ``linear_detect_batch`` (detect.py:528-557) on seeded
Rayleigh channels for QPSK / 16-QAM / 64-QAM, square and tall H, scalar and
per-vector noise variance, and writes ``linear.npz``.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mpnlsim import detect as det                      # noqa: E402  (reference)
from mpnlsim.core import constellation_for             # noqa: E402

CASES = [  # (name, M, N, order, B)
    ("q4_2x2", 2, 2, 4, 64), ("q16_4x4", 4, 4, 16, 64), ("q64_8x8", 8, 8, 64, 32),
    ("q16_12x12", 12, 12, 16, 32), ("q4_6x4", 6, 4, 4, 64), ("q64_16x16", 16, 16, 64, 16),
    # N > 16 (the C5 / C4 shapes and a ragged tall one), added in round 2
    ("q64_24x24", 24, 24, 64, 16), ("q16_32x32", 32, 32, 16, 8), ("q16_28x19", 28, 19, 16, 16),
]


def main():
    rng = np.random.default_rng(2409)
    out = {}
    for name, m, n, order, b in CASES:
        c = constellation_for(order)
        h = (rng.standard_normal((b, m, n)) + 1j * rng.standard_normal((b, m, n))) / np.sqrt(2 * m)
        x = c.points[rng.integers(0, order, (b, n))]
        nv = 0.05
        nv_vec = nv * (0.5 + rng.random(b))
        y = np.einsum("bmn,bn->bm", h, x) + np.sqrt(nv / 2) * (
            rng.standard_normal((b, m)) + 1j * rng.standard_normal((b, m)))
        out[f"{name}_h"], out[f"{name}_y"], out[f"{name}_nv_vec"] = h, y, nv_vec
        out[f"{name}_meta"] = np.array([m, n, order, b])
        for mode in ("zf", "mmse"):
            lab, llr = det.linear_detect_batch(h, y, nv, c, mode)
            out[f"{name}_{mode}_labels"], out[f"{name}_{mode}_llr"] = lab, llr
            lab, llr = det.linear_detect_batch(h, y, nv_vec, c, mode)
            out[f"{name}_{mode}_labels_vec"], out[f"{name}_{mode}_llr_vec"] = lab, llr
    out["names"] = np.array([c[0] for c in CASES])
    np.savez_compressed(HERE / "linear.npz", **out)
    print({k: v.shape for k, v in out.items() if k.endswith("_h")})


if __name__ == "__main__":
    main()
