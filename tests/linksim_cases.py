"""Seeded link-level cases (reference simulate_frames vs the GPU one), shared by
tests/golden/make_golden_linksim.py (reference side) and the tests.
(name, n_streams, m, mcs (order, rate num, rate den), rb, detector, csi, n_paths,
snr_db, frames)"""

import numpy as np

CASES = [
    ("mpnl_genie_q4", 4, 8, (4, 679, 1024), 2, "mpnl", "genie", 32, 6.0, 12),
    ("mpnl_genie_q16", 4, 6, (16, 245, 512), 2, "mpnl", "genie", 32, 10.5, 12),
    ("mpnl_ls_q4", 3, 6, (4, 679, 1024), 2, "mpnl", "ls_dmrs", 16, 14.0, 8),
    ("mmse_genie_q16", 4, 6, (16, 245, 512), 2, "mmse", "genie", 32, 9.0, 12),
    ("zf_ls_q4", 3, 6, (4, 679, 1024), 2, "zf", "ls_dmrs", 32, 14.0, 8),
]


def channel(case):
    """Rayleigh grid (symbols 14, subcarriers 12 rb, M, N), unit-power entries:
    i.i.d. per resource element for genie CSI, one block-constant matrix for the
    LS-DMRS cases (nearest-pilot interpolation needs a smooth channel)."""
    name, n, m, mcs, rb, det, csi, p, snr, f = case
    rng = np.random.default_rng(np.random.SeedSequence((2409, n, m, rb)))
    sc = 12 * rb
    shape = (14, sc, m, n) if csi == "genie" else (1, 1, m, n)
    h = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)
    return np.ascontiguousarray(np.broadcast_to(h, (14, sc, m, n)))


def noise_var(case):
    return case[1] / 10 ** (case[8] / 10)
