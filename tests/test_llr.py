"""List max-log LLR soft output: `_candidate_llrs_batch`
(detect.py:439-453) and the link simulator's MPNL branch (linksim.py:151-155).

CPU: the oracle restatement is pinned bit-exactly to the reference's own
outputs (tests/golden/llr_*.npz, made by tests/golden/make_golden_llr.py) and,
where the reference tree is mounted, to the live reference on fresh inputs.
GPU: the K6 kernel through the C ABI is bit-identical to those goldens (both
fp64: one subtraction and one correctly rounded division), and the fused
detect + LLR path reproduces them from the channel/observation inputs.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import mpnl_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden"
LLR_CASES = sorted(p.stem[4:] for p in GOLD.glob("llr_*.npz"))


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("case", LLR_CASES)
def test_oracle_llrs_match_reference_golden(case):
    g = np.load(GOLD / f"llr_{case}.npz")
    q = int(g["order"])
    assert _same(orc.candidate_llrs(g["labels"], g["metrics"], g["nv"], q), g["llr"])
    assert _same(orc.candidate_llrs(g["labels"], g["metrics"], g["nv_vec"], q), g["llr_vec"])
    assert _same(orc.candidate_llrs(g["labels"], g["metrics"], g["nv"], q, clip=3.0),
                 g["llr_clip3"])


def test_oracle_llrs_match_live_reference(reference_module):
    from mpnlsim.core import constellation_for as ref_c
    rng = np.random.default_rng(5)
    for q, p, n in ((4, 7, 3), (16, 33, 12), (64, 130, 5)):
        lab = rng.integers(0, q, (9, p, n))
        met = rng.exponential(1.0, (9, p))
        met[0, :] = met[0, 0]                       # all-equal metrics
        ref = reference_module._candidate_llrs_batch(lab, met, 0.07, ref_c(q))
        assert _same(orc.candidate_llrs(lab, met, 0.07, q), ref)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

def _det():
    from paper_2409_14355_b200 import detect
    return detect


@pytest.mark.gpu
@pytest.mark.parametrize("case", LLR_CASES)
def test_gpu_llrs_match_reference_golden(case):
    import torch
    det = _det()
    from paper_2409_14355_b200.core import constellation_for
    g = np.load(GOLD / f"llr_{case}.npz")
    c = constellation_for(int(g["order"]))
    assert _same(det._candidate_llrs_batch(g["labels"], g["metrics"], float(g["nv"]), c),
                 g["llr"])
    assert _same(det._candidate_llrs_batch(g["labels"], g["metrics"], g["nv_vec"], c),
                 g["llr_vec"])
    assert _same(det._candidate_llrs_batch(g["labels"], g["metrics"], float(g["nv"]), c,
                                           clip=3.0), g["llr_clip3"])
    # device tensors in, device tensor out
    lab = torch.from_numpy(g["labels"]).cuda()
    met = torch.from_numpy(g["metrics"]).cuda()
    out = det._candidate_llrs_batch(lab, met, float(g["nv"]), c)
    assert out.is_cuda and _same(out.cpu().numpy(), g["llr"])


@pytest.mark.gpu
@pytest.mark.parametrize("q,p,n,b", [(4, 1, 1, 3), (16, 1024, 24, 37), (64, 257, 32, 2000),
                                     (16, 5, 12, 0)])
def test_gpu_llrs_match_oracle_random(q, p, n, b):
    det = _det()
    from paper_2409_14355_b200.core import constellation_for
    rng = np.random.default_rng(q * 1000 + p)
    lab = rng.integers(0, q, (b, p, n)).astype(np.uint8)
    met = rng.exponential(3.0, (b, p))
    if b:
        met[0] = 1.25                                   # all-equal metrics
    nv = rng.uniform(0.05, 2.0, b)
    got = det._candidate_llrs_batch(lab, met, nv, constellation_for(q))
    assert _same(got, orc.candidate_llrs(lab, met, nv, q))


@pytest.mark.gpu
def test_gpu_llr_errors():
    det = _det()
    from paper_2409_14355_b200.core import constellation_for
    c = constellation_for(16)
    with pytest.raises(ValueError, match="empty candidate list"):
        det._candidate_llrs_batch(np.zeros((2, 0, 4), np.uint8), np.zeros((2, 0)), 0.1, c)
    with pytest.raises(ValueError):
        det._candidate_llrs_batch(np.zeros((2, 3, 4), np.uint8), np.zeros((2, 4)), 0.1, c)
    with pytest.raises(ValueError):
        det._candidate_llrs_batch(np.full((1, 3, 4), 16, np.uint8), np.zeros((1, 3)), 0.1, c)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "c2", "c5p16", "q4x4", "over2x3"])
def test_gpu_detect_llrs_end_to_end(case):
    """Channel + observations -> plan -> full list -> LLRs on the device,
    against the reference's LLRs of its own candidate lists.  The fp64 list
    metrics agree with the reference to 1e-9 relative (test_gpu_parity), so
    each LLR agrees to 2e-9 * max(metric) / nv absolute; saturated LLRs
    (bits without a counter-hypothesis, or beyond the clip) are identical."""
    det = _det()
    from paper_2409_14355_b200.core import constellation_for
    f = np.load(GOLD / f"full_{case}.npz")
    g = np.load(GOLD / f"llr_{case}.npz")
    c = constellation_for(int(f["order"]))
    h, y = f["h"], f["y"]
    if h.ndim == 3 and y.ndim == 3:            # one RB channel, (1, V, M) observations
        plan = det.mpnl_plan_batch(h, float(f["nv"]), int(f["n_paths"]), c)
        llr = det.mpnl_detect_llrs(plan, h, y, c)[0]
    else:                                      # a channel per vector
        plan = det.mpnl_plan_batch(h, float(f["nv"]), int(f["n_paths"]), c)
        llr = det.mpnl_detect_llrs(plan, h, y, c)
    ref = g["llr"]
    assert llr.shape == ref.shape
    tol = 2e-9 * float(np.max(g["metrics"])) / float(f["nv"])
    np.testing.assert_allclose(llr, ref, rtol=0, atol=tol)
    sat = np.abs(ref) == 20.0
    assert np.array_equal(llr[sat], ref[sat])


@pytest.mark.gpu
def test_single_instance_llrs_match_reference_golden():
    det = _det()
    from paper_2409_14355_b200.core import constellation_for
    f = np.load(GOLD / "full_q16_4x4.npz")
    g = np.load(GOLD / "llr_q16_4x4.npz")
    c = constellation_for(16)
    for i in range(4):
        inp = det.DetectorInput(f["h"][i], f["y"][i], float(f["nv"]), c)
        plan = det.mpnl_preprocess(inp.h, inp.noise_var, int(f["n_paths"]), c)
        _, out = det.mpnl_detect(plan, inp)
        tol = 2e-9 * float(np.max(g["metrics"][i])) / float(f["nv"])
        np.testing.assert_allclose(out.llrs, g["llr"][i], rtol=0, atol=tol)
