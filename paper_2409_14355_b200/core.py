"""Gray-mapped square-QAM tables used by the MPNL path.

Restates the constellation convention of the reference
(`pkg/src/mpnlsim/core.py:24-92` and `bits_from_labels` at `core.py:209-213`):

* per axis, the amplitude levels L-1, L-3, ..., -(L-1) sit at *level index*
  ``pos = 0..L-1`` and carry the Gray label ``pos ^ (pos >> 1)``;
* the integer point label is ``(I_label << h) | Q_label`` with h = log2(Q)/2;
* points are scaled to unit average energy, norm^2 = 2 (4^h - 1) / 3.

The CUDA kernels never touch complex points: they slice in *level-index*
space (one integer per axis) and convert to Gray labels only for the winner.
The helpers here give the host the same maps (``level_to_label`` etc.).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LLR_CLIP = 20.0
SUPPORTED_ORDERS = (4, 16, 64)


def gray(i):
    return i ^ (i >> 1)


@dataclass(frozen=True)
class Constellation:
    """Unit-energy Gray square QAM; ``points[label]`` as in the reference."""

    order: int
    points: np.ndarray = field(repr=False)
    bits_per_symbol: int = field(init=False)

    def __post_init__(self):
        if self.order not in SUPPORTED_ORDERS:
            raise ValueError(f"unsupported constellation order {self.order}")
        object.__setattr__(self, "bits_per_symbol", self.order.bit_length() - 1)

    # -- level-index view used by the kernels -------------------------------
    @property
    def levels_per_axis(self) -> int:
        return 1 << (self.bits_per_symbol // 2)

    @property
    def norm(self) -> float:
        h = self.bits_per_symbol // 2
        return float(np.sqrt(2.0 * (4 ** h - 1) / 3.0))

    @property
    def labels(self) -> np.ndarray:
        b = self.bits_per_symbol
        return (np.arange(self.order)[:, None] >> np.arange(b - 1, -1, -1)) & 1

    def nearest(self, y) -> np.ndarray:
        d = np.abs(np.asarray(y)[..., None] - self.points) ** 2
        return np.argmin(d, axis=-1)


def make_constellation(order: int) -> Constellation:
    if order not in SUPPORTED_ORDERS:
        raise ValueError(f"unsupported constellation order {order}")
    h = (order.bit_length() - 1) // 2
    n_lv = 1 << h
    # amplitude of the level carrying each Gray label
    amp = np.empty(n_lv)
    for pos in range(n_lv):
        amp[gray(pos)] = n_lv - 1 - 2 * pos
    lab = np.arange(order)
    pts = (amp[lab >> h] + 1j * amp[lab & (n_lv - 1)]) / np.sqrt(2.0 * (4 ** h - 1) / 3.0)
    return Constellation(order=order, points=pts)


QPSK = make_constellation(4)
QAM16 = make_constellation(16)
QAM64 = make_constellation(64)
_BY_ORDER = {4: QPSK, 16: QAM16, 64: QAM64}


def constellation_for(order: int) -> Constellation:
    if order not in _BY_ORDER:
        raise ValueError(f"unsupported constellation order {order}")
    return _BY_ORDER[order]


def bits_from_labels(labels, c: Constellation) -> np.ndarray:
    """(..., ) integer labels -> (..., bits_per_symbol) bits, MSB first."""
    lab = np.asarray(labels, dtype=np.int64)
    return (lab[..., None] >> np.arange(c.bits_per_symbol - 1, -1, -1)) & 1


def level_index_to_label(i_re, i_im, order: int):
    """Kernel level indices (per axis, 0 = most positive) -> point labels."""
    h = (order.bit_length() - 1) // 2
    return (gray(np.asarray(i_re)) << h) | gray(np.asarray(i_im))


def label_to_level_index(label, order: int):
    """Point labels -> (i_re, i_im) level indices (inverse Gray per axis)."""
    h = (order.bit_length() - 1) // 2
    lab = np.asarray(label)
    g_re, g_im = lab >> h, lab & ((1 << h) - 1)

    def inv_gray(g):
        g = np.array(g, dtype=np.int64, copy=True)
        out = g.copy()
        s = g >> 1
        while np.any(s):
            out ^= s
            s >>= 1
        return out

    return inv_gray(g_re), inv_gray(g_im)
