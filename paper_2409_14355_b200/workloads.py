"""Seeded synthetic workloads for the five BASELINE configurations.

There is no public dataset behind BASELINE.json: the configs are synthetic
uplink MU-MIMO slots, and these generators stand in for them.
Draw order per config: channel -> correlation / gains -> transmit labels ->
noise, all from ``SeedSequence((seed, config_id))`` in float64, stored as
complex64 (the oracle upcasts the very same arrays).

* one channel per resource block (RB) of 12 subcarriers x 14 symbols
  = 168 received vectors;
* symbols uniform over the Q labels, mapped with the reference's Gray tables;
* per-receive-antenna SNR convention ``nv = N / 10^(SNR/10)``
  (reference `channel.py:197-208`, `cli.py:232`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import constellation_for

VECTORS_PER_RB = 12 * 14


@dataclass(frozen=True)
class MimoConfig:
    name: str
    cid: int
    n: int                 # users / streams
    m: int                 # receive antennas
    order: int             # QAM order
    n_paths: int
    n_rb: int
    snr_db: tuple          # one entry per SNR point (C2 sweeps 6)
    channel: str = "iid"   # iid | kron | lognormal_pc
    rho_rx: float = 0.0
    rho_tx: float = 0.0
    gain_sigma_db: float = 0.0

    @property
    def vectors_per_channel(self) -> int:
        return VECTORS_PER_RB * len(self.snr_db)

    @property
    def n_vectors(self) -> int:
        return self.n_rb * self.vectors_per_channel

    def flops_per_vector(self, realized_paths=None) -> int:
        p = realized_paths or self.n_paths
        return p * 4 * self.n * (self.n + 1)

    def bytes_per_vector(self) -> float:
        return 8 * self.m + 8 * self.m * self.n / self.vectors_per_channel + self.n + 4


CONFIGS = {
    "C1": MimoConfig("C1", 1, 8, 8, 16, 32, 4, (15.0,)),
    "C2": MimoConfig("C2", 2, 12, 12, 16, 64, 273, (10.0, 12.0, 14.0, 16.0, 18.0, 20.0)),
    "C3": MimoConfig("C3", 3, 16, 16, 64, 128, 273, (22.0,), "kron", 0.5, 0.3),
    "C4": MimoConfig("C4", 4, 32, 32, 16, 256, 273, (14.0,), "lognormal_pc",
                     gain_sigma_db=6.0),
    "C5P16": MimoConfig("C5P16", 51, 24, 24, 64, 16, 2048, (24.0,)),
    "C5P64": MimoConfig("C5P64", 52, 24, 24, 64, 64, 2048, (24.0,)),
    "C5P256": MimoConfig("C5P256", 53, 24, 24, 64, 256, 2048, (24.0,)),
    "C5P1024": MimoConfig("C5P1024", 54, 24, 24, 64, 1024, 2048, (24.0,)),
}


def _expo_corr_sqrt(n, rho):
    idx = np.arange(n)
    r = rho ** np.abs(idx[:, None] - idx[None, :])
    w, v = np.linalg.eigh(r)                       # symmetric square root
    return (v * np.sqrt(np.maximum(w, 0.0))) @ v.T


def generate(cfg: MimoConfig | str, seed: int = 2409, n_rb: int | None = None,
             rb_offset: int = 0):
    """Returns dict(h (C,M,N) c64, y (C,V,M) c64, labels (C,V,N) int64,
    nv (V,) float64 per vector slot, cfg).

    ``n_rb``/``rb_offset`` select a sub-range of the config's RBs; the RNG is
    advanced per RB so a sub-range equals the same rows of the full draw.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n_rb = cfg.n_rb if n_rb is None else n_rb
    c = constellation_for(cfg.order)
    v = cfg.vectors_per_channel
    m, n = cfg.m, cfg.n
    h_all = np.empty((n_rb, m, n), np.complex64)
    y_all = np.empty((n_rb, v, m), np.complex64)
    lab_all = np.empty((n_rb, v, n), np.int64)
    nv_slots = np.repeat([n / 10 ** (s / 10) for s in cfg.snr_db], VECTORS_PER_RB)
    if cfg.channel == "kron":
        sr, st = _expo_corr_sqrt(m, cfg.rho_rx), _expo_corr_sqrt(n, cfg.rho_tx)
    for k in range(n_rb):
        rng = np.random.default_rng(np.random.SeedSequence((seed, cfg.cid, rb_offset + k)))
        hw = (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))) / np.sqrt(2)
        if cfg.channel == "kron":
            h = sr @ hw @ st
        elif cfg.channel == "lognormal_pc":
            g = 10 ** (rng.normal(0.0, cfg.gain_sigma_db, n) / 10)   # large-scale gains
            h = (hw * np.sqrt(g)) * np.sqrt(1.0 / g)                  # power control
        else:
            h = hw
        h = h.astype(np.complex64)
        lab = rng.integers(0, cfg.order, (v, n))
        x = c.points[lab]
        noise = np.sqrt(nv_slots / 2)[:, None] * (rng.standard_normal((v, m))
                                                  + 1j * rng.standard_normal((v, m)))
        y = x @ h.astype(np.complex128).T + noise
        h_all[k], y_all[k], lab_all[k] = h, y.astype(np.complex64), lab
    return {"h": h_all, "y": y_all, "labels": lab_all, "nv": nv_slots, "cfg": cfg}
