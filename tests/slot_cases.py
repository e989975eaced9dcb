"""Seeded slot-grid cases shared by the golden generator (reference) and the
tests: (name, n_streams, m_antennas, rb_per_vehicle, frames, unit_pilots)."""

import hashlib

import numpy as np

CASES = [("s2m4rb1", 2, 4, 1, 2, True), ("s4m8rb2", 4, 8, 2, 3, False),
         ("s12m16rb1", 12, 16, 1, 1, False), ("s7m7rb3", 7, 7, 3, 2, False)]
SYMBOLS, DMRS_SYMBOLS = 14, 2


def inputs(case):
    name, n, m, rb, f, unit = case
    sc = 12 * rb
    rng = np.random.default_rng(np.random.SeedSequence((77, n, m, rb)))
    cn = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)   # noqa: E731
    obs = cn(SYMBOLS, sc, m)
    pilots = np.ones((n, sc // 6), complex) if unit else cn(n, sc // 6)
    h = cn(SYMBOLS, sc, m, n)
    x = cn(f, SYMBOLS, sc, n)
    noise = 0.1 * cn(f, SYMBOLS, sc, m)
    return obs, pilots, h, x, noise


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
