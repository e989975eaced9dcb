"""CPU oracle for the slot I/O around the detector — TEST INFRASTRUCTURE ONLY
(SURVEY §8f row 4).  Only tests/ may import it, as a checker.

numpy restatement of the reference link simulator's grid steps
(`/root/reference/pkg/src/mpnlsim/linksim.py`):

* ``dmrs_pattern``        <- linksim.py:103-114 (6 combs per DMRS symbol 3, 12)
* ``estimate_channel_ls`` <- linksim.py:117-137 (obs / pilot at the nearest
                             pilot subcarrier, constant over the slot)
* ``receive_grid``        <- linksim.py:207 (einsum + noise)
* ``data_re_batch``       <- linksim.py:211-216
Pinned by tests/golden/slot.json (sha256 of the reference's own outputs,
made by tests/golden/make_golden_slot.py).
"""

from __future__ import annotations

import numpy as np

DMRS_COMBS = 6


def dmrs_pattern(dmrs_symbols, n_streams, n_sc):
    if n_streams > DMRS_COMBS * dmrs_symbols:
        raise ValueError("too many streams for the pilot book")
    syms = (3, 12)[:dmrs_symbols]
    return syms, [(syms[v // DMRS_COMBS], np.arange(v % DMRS_COMBS, n_sc, DMRS_COMBS))
                  for v in range(n_streams)]


def estimate_channel_ls(grid_obs, pilots, symbols, dmrs_symbols, n_sc, m, n):
    _, ports = dmrs_pattern(dmrs_symbols, n, n_sc)
    h = np.empty((symbols, n_sc, m, n), dtype=complex)
    for v, (sym, sc_idx) in enumerate(ports):
        h_pilot = grid_obs[sym, sc_idx, :] / pilots[v][:, None]
        nearest = np.abs(np.arange(n_sc)[:, None] - sc_idx[None, :]).argmin(axis=1)
        h[:, :, :, v] = h_pilot[nearest][None]
    return h


def receive_grid(h, x, noise=None):
    y = np.einsum("tfmn,btfn->btfm", h, x)
    return y if noise is None else y + noise


def data_re_batch(h, y, data_syms):
    s = len(data_syms)
    return (h[data_syms].reshape(s * h.shape[1], *h.shape[2:]),
            y[:, data_syms].reshape(y.shape[0], s * y.shape[2], y.shape[3]))
