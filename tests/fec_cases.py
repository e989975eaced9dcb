"""Seeded LDPC test cases shared by the golden generator (run against the
reference in the build container) and the tests (CPU oracle, GPU kernels).

Only the reference's OUTPUTS (encoded words, decoded info bits, converged
flags) and the payload bits are stored in tests/golden/fec.npz; the channel
LLRs are regenerated here from the seeds (numpy PCG64 is deterministic) and
checked against a stored sha256.
"""

from __future__ import annotations

import hashlib
from fractions import Fraction

import numpy as np

# name: (words, seed, kind, param, max_iter, rate match (rate, n_tx) or None)
CASES = {
    "awgn_m1db": (24, 11, "awgn", -1.0, 10, None),
    "awgn_2db": (24, 12, "awgn", 2.0, 10, None),
    "awgn_2p5db": (24, 13, "awgn", 2.5, 10, None),
    "awgn_3db": (16, 14, "awgn", 3.0, 10, None),
    "awgn_2p5db_it5": (16, 15, "awgn", 2.5, 5, None),
    "awgn_1db_it1": (8, 16, "awgn", 1.0, 1, None),
    "awgn_1db_it0": (8, 17, "awgn", 1.0, 0, None),
    "clip20": (16, 18, "clip", 2.5, 10, None),          # +-20 clipped (detector LLRs)
    "ties": (12, 19, "ties", 0.0, 10, None),            # small integers: min ties, zeros
    "noise": (8, 20, "noise", 0.0, 10, None),           # no codeword: never converges
    "rm_1_3_900": (16, 21, "awgn", 1.0, 10, (Fraction(1, 3), 900)),
    "rm_193_576": (16, 22, "awgn", 0.5, 10, (Fraction(193, 1024), 576)),
    "rm_3_4_800": (16, 23, "awgn", 5.0, 10, (Fraction(3, 4), 800)),
    "rm_1_4_864": (16, 24, "awgn", 1.5, 10, (Fraction(1, 4), 864)),
}


def payload(name, k_bits):
    words, seed = CASES[name][:2]
    rng = np.random.default_rng(np.random.SeedSequence((seed, 1)))
    return rng.integers(0, 2, (words, k_bits)).astype(np.uint8)


def channel_llrs(name, tx_bits):
    """LLRs (positive = bit 0) of the transmitted bits through the case's channel."""
    words, seed, kind, param = CASES[name][:4]
    rng = np.random.default_rng(np.random.SeedSequence((seed, 2)))
    x = 1.0 - 2.0 * tx_bits.astype(np.float64)
    if kind == "awgn" or kind == "clip":
        nv = 10 ** (-param / 10)
        y = x + rng.normal(0.0, np.sqrt(nv), x.shape)
        llr = 2.0 * y / nv
        return np.clip(llr, -20.0, 20.0) if kind == "clip" else llr
    if kind == "ties":
        mag = rng.integers(0, 4, x.shape).astype(np.float64)        # many equal magnitudes
        flip = rng.random(x.shape) < 0.08
        return np.where(flip, -x, x) * mag
    if kind == "noise":
        return rng.normal(0.0, 1.0, x.shape)
    raise ValueError(kind)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
