"""Link-level frames on the GPU (simulate_frames: LDPC encode -> modulation ->
DMRS -> receive grid -> genie or LS-DMRS CSI -> MPNL / ZF / MMSE soft output ->
rate-matched LDPC decoding) against the reference's own simulate_frames
(linksim.py:159-232) on the same seeded channel grids and per-frame random
streams: the per-frame, per-stream decode outcomes must be identical
(tests/golden/linksim.npz, make_golden_linksim.py)."""

from fractions import Fraction
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

import linksim_cases as lc
from paper_2409_14355_b200.core import constellation_for

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "linksim.npz")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", lc.CASES, ids=[c[0] for c in lc.CASES])
def test_simulate_frames_matches_reference(case):
    from paper_2409_14355_b200 import linksim as L
    name, n, m, (q, rn, rd), rb, det, csi, p, snr, f = case
    mcs = SimpleNamespace(constellation=constellation_for(q), code_rate=Fraction(rn, rd))
    cfg = L.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, rb_per_vehicle=rb, detector=det,
                       n_paths=p, csi=csi)
    ok = L.simulate_frames(cfg, lc.channel(case), lc.noise_var(case), 3, range(f))
    assert ok.shape == (f, n) and ok.dtype == bool
    assert np.array_equal(ok, GOLD[name]), f"{name}: {int((ok != GOLD[name]).sum())} outcomes differ"


@pytest.mark.parametrize("case", [c for c in lc.CASES if c[5] == "mpnl"],
                         ids=[c[0] for c in lc.CASES if c[5] == "mpnl"])
def test_simulate_frames_fp32_soft_output(case):
    """The fp32 soft output (fused traversal + LLR kernel) perturbs LLRs by
    ~1e-6 of the metrics / noise_var: on these seeded cases every decode outcome
    still equals the reference's."""
    from paper_2409_14355_b200 import linksim as L
    name, n, m, (q, rn, rd), rb, det, csi, p, snr, f = case
    mcs = SimpleNamespace(constellation=constellation_for(q), code_rate=Fraction(rn, rd))
    cfg = L.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, rb_per_vehicle=rb, detector=det,
                       n_paths=p, csi=csi)
    ok = L.simulate_frames(cfg, lc.channel(case), lc.noise_var(case), 3, range(f),
                           soft_precision="fp32")
    assert np.array_equal(ok, GOLD[name]), f"{name}: {int((ok != GOLD[name]).sum())} outcomes differ"


def test_config_validation_like_reference():
    from paper_2409_14355_b200 import linksim as L
    mcs = SimpleNamespace(constellation=constellation_for(4), code_rate=Fraction(1, 2))
    for kw in ({"n_streams": 13}, {"m_antennas": 0}, {"detector": "ml"}, {"csi": "perfect"}):
        args = dict(n_streams=2, m_antennas=2, mcs=mcs, rb_per_vehicle=1)
        args.update(kw)
        with pytest.raises(ValueError):
            L.LinkConfig(**args)
    cfg = L.LinkConfig(n_streams=2, m_antennas=4, mcs=mcs, rb_per_vehicle=3)
    assert cfg.n_subcarriers == 36 and cfg.bits_per_block == 36 * 12 * 2
    with pytest.raises(ValueError, match="smaller"):
        L.simulate_frames(cfg, np.zeros((14, 12, 4, 2), complex), 0.1, 0, range(1))


def test_measure_per_matches_reference():
    """measure_per (linksim.py:241-271) over two channels, plain and with the
    early stop armed: the same frames and errors as the reference."""
    from paper_2409_14355_b200 import linksim as L
    case = lc.CASES[0]
    name, n, m, (q, rn, rd), rb, det, csi, p, snr, f = case
    mcs = SimpleNamespace(constellation=constellation_for(q), code_rate=Fraction(rn, rd))
    cfg = L.LinkConfig(n_streams=n, m_antennas=m, mcs=mcs, rb_per_vehicle=rb, detector=det,
                       n_paths=p, csi=csi)
    grids = [lc.channel(case), np.ascontiguousarray(lc.channel(case)[:, ::-1])]
    nvs = [lc.noise_var(case), 0.8 * lc.noise_var(case)]
    r = L.measure_per(cfg, grids, nvs, frames_per_channel=60)
    r2 = L.measure_per(cfg, grids, nvs, frames_per_channel=200, stop_threshold=0.9,
                       min_frames=100)
    assert [r.frames, r.errors, r2.frames, r2.errors] == GOLD["measure_per"].tolist()
    with pytest.raises(ValueError):
        L.measure_per(cfg, grids, nvs, frames_per_channel=0)
