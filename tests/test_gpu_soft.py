"""fp32 soft output: the fused traversal + list max-log LLR kernel
(`mpnl_detect_llrs_fast`) against the reference semantics of
`mpnl_detect_batch` + `_candidate_llrs_batch` (detect.py:473-488, 439-453;
linksim.py:151-155).

The checker is the CPU oracle (full candidate lists + list LLRs, pinned to the
reference by tests/test_oracle.py and tests/test_llr.py) and the fp64 GPU path
(bit-identical to the reference, tests/test_llr.py).  Tolerance: the fp32 path's
metrics carry the traversal's fp32 PED error, so an LLR may differ from the
reference's by 2 ped_tol / noise_var; the bound asserted here is
    |llr_fp32 - llr_ref| <= 2e-5 * (m_max / noise_var) + 1e-9
with m_max the vector's largest finite list minimum (ped_tol is below 1e-5 of
the metric on every BASELINE config), and clipped LLRs must be equal.
"""

import numpy as np
import pytest

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.core import LLR_CLIP, constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

pytestmark = pytest.mark.gpu


def _det():
    from paper_2409_14355_b200 import detect
    return detect


def _check(llr, ref, nv, scale, what):
    llr, ref = np.asarray(llr), np.asarray(ref)
    assert llr.shape == ref.shape, what
    sat = np.abs(ref) >= LLR_CLIP
    # an LLR within the tolerance of the clip may be clipped on one side only
    tol = 2e-5 * scale / nv + 1e-9
    err = np.abs(llr - ref)
    assert np.all(err <= tol[..., None, None]), (
        f"{what}: max err {err.max():.3e} vs tol {tol.max():.3e}")
    far = sat & (np.abs(np.abs(llr) - LLR_CLIP) > tol[..., None, None])
    assert not far.any(), f"{what}: clipped LLRs differ"


@pytest.mark.parametrize("name,n_rb,nvec", [("C1", 4, 168), ("C2", 3, 56), ("C3", 2, 24),
                                            ("C4", 1, 8), ("C5P16", 2, 40), ("C5P64", 1, 24),
                                            ("C5P256", 1, 6)])
def test_fp32_llrs_vs_oracle(name, n_rb, nvec):
    import torch
    det = _det()
    cfg = CONFIGS[name]
    d = generate(cfg, n_rb=n_rb)
    c = constellation_for(cfg.order)
    nv = float(d["nv"][0])
    y = np.ascontiguousarray(d["y"][:, :nvec])
    plan = det.mpnl_plan_batch(torch.from_numpy(d["h"]).cuda(), nv, cfg.n_paths, c)
    llr, flags = det.mpnl_detect_llrs(plan, torch.from_numpy(d["h"]).cuda(),
                                      torch.from_numpy(y).cuda(), c, precision="fp32",
                                      return_flags=True)
    llr, flags = llr.cpu().numpy(), flags.cpu().numpy()
    # oracle: full lists + list LLRs, one plan per RB tiled over its vectors
    for rb in range(n_rb):
        p = orc.plan_channels(d["h"][rb:rb + 1], nv, cfg.n_paths, cfg.order).tile(nvec)
        lab, met, _ = orc.detect_batch(p, np.repeat(d["h"][rb:rb + 1], nvec, 0).astype(complex),
                                       y[rb].astype(complex), c.points)
        ref = orc.candidate_llrs(lab, met, nv, cfg.order)
        bits = ((lab[..., None] >> np.arange(c.bits_per_symbol - 1, -1, -1)) & 1).astype(bool)
        mm = met[:, :, None, None]
        mins = np.minimum(np.where(bits, mm, np.inf).min(1), np.where(~bits, mm, np.inf).min(1))
        scale = np.where(np.isfinite(mins), mins, 0).max(axis=(1, 2)) + met.min(1)
        _check(llr[rb], ref, nv, scale, f"{name} rb {rb}")
        # recomputed (flagged) vectors went through the fp64 list path
        for v in np.nonzero(flags[rb])[0]:
            np.testing.assert_allclose(llr[rb, v], ref[v], rtol=0, atol=1e-9 * scale[v] / nv)


@pytest.mark.parametrize("name,n_rb", [("C2", 12), ("C5P64", 4)])
def test_fp32_llrs_vs_fp64_gpu_path(name, n_rb):
    """Larger samples against the fp64 GPU path (bit-identical to the reference)."""
    import torch
    det = _det()
    cfg = CONFIGS[name]
    d = generate(cfg, n_rb=n_rb)
    c = constellation_for(cfg.order)
    nv = float(d["nv"][0])
    h = torch.from_numpy(d["h"]).cuda()
    y = torch.from_numpy(np.ascontiguousarray(d["y"][:, :168])).cuda()
    plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    fast, flags = det.mpnl_detect_llrs(plan, h, y, c, precision="fp32", return_flags=True)
    ref = det.mpnl_detect_llrs(plan, h, y, c)
    _, metrics, _ = det.mpnl_detect_batch(plan, h, y, c)
    scale = 2.0 * metrics.max(dim=-1).values.cpu().numpy()
    _check(fast.cpu().numpy(), ref.cpu().numpy(), nv, scale, name)
    # the fp64 recomputation (near-tie selections only) is rare
    assert flags.float().mean().item() < 0.01


def test_fp32_llrs_numpy_and_squeeze():
    det = _det()
    cfg = CONFIGS["C1"]
    d = generate(cfg, n_rb=2)
    c = constellation_for(cfg.order)
    nv = float(d["nv"][0])
    plan = det.mpnl_plan_batch(d["h"], nv, cfg.n_paths, c)
    a = det.mpnl_detect_llrs(plan, d["h"], d["y"], c, precision="fp32")
    assert isinstance(a, np.ndarray) and a.shape == d["y"].shape[:2] + (cfg.n, 4)
    b = det.mpnl_detect_llrs(plan, d["h"], d["y"][:, 0], c, precision="fp32")
    assert b.shape == (2, cfg.n, 4)
    ref = det.mpnl_detect_llrs(plan, d["h"], d["y"][:, 0], c)
    assert np.abs(b - ref).max() < 1e-3
    with pytest.raises(ValueError):
        det.mpnl_detect_llrs(plan, d["h"], d["y"], c, precision="fp16")


def test_fp32_llrs_fall_back_without_fp32_path():
    """Overloaded channels (N > M) have no fp32 path: the fp64 list path answers."""
    det = _det()
    rng = np.random.default_rng(3)
    h = ((rng.standard_normal((3, 2, 3)) + 1j * rng.standard_normal((3, 2, 3))) / np.sqrt(2))
    y = rng.standard_normal((3, 5, 2)) + 1j * rng.standard_normal((3, 5, 2))
    c = constellation_for(4)
    plan = det.mpnl_plan_batch(h, 0.1, 16, c)
    assert plan.augmented
    a, flags = det.mpnl_detect_llrs(plan, h, y, c, precision="fp32", return_flags=True)
    b = det.mpnl_detect_llrs(plan, h, y, c)
    assert np.array_equal(a, b, equal_nan=True) and flags.all()
