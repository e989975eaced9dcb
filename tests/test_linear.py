"""Batched linear ZF / MMSE detection (detect.py:528-557).

CPU: the oracle restatement reproduces the reference's own outputs
(tests/golden/linear.npz, made by make_golden_linear.py from the reference).
GPU: the CUDA kernel (mpnl_linear_detect through detect.linear_detect_batch)
against the same goldens and against the oracle on larger seeded batches.
Hard labels must match exactly; LLRs within atol 1e-6 (fp64 Cholesky here vs a
LAPACK inverse in the reference — same quantities, different rounding) and the
equalised symbols within 1e-9 relative.  Mirrors the reference's own linear
tests (test_detect.py:25-100): identity / closed-form MMSE, ZF noiseless
consistency, MMSE -> ZF limit, singular channel rejection, unknown mode.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import mpnl_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden" / "linear.npz"
LLR_ATOL = 1e-6


def _cases():
    d = np.load(GOLD)
    return d, [str(n) for n in d["names"]]


@pytest.mark.parametrize("mode", ["zf", "mmse"])
def test_oracle_linear_matches_reference_golden(mode):
    d, names = _cases()
    for name in names:
        m, n, order, b = d[f"{name}_meta"]
        for suffix, nv in (("", 0.05), ("_vec", d[f"{name}_nv_vec"])):
            lab, llr, _ = orc.linear_detect(d[f"{name}_h"], d[f"{name}_y"], nv, int(order), mode)
            np.testing.assert_array_equal(lab, d[f"{name}_{mode}_labels{suffix}"])
            np.testing.assert_allclose(llr, d[f"{name}_{mode}_llr{suffix}"], rtol=0, atol=1e-12)


def _rand(rng, b, m, n, order, nv):
    pts = orc._points(order)
    h = (rng.standard_normal((b, m, n)) + 1j * rng.standard_normal((b, m, n))) / np.sqrt(2 * m)
    x = pts[rng.integers(0, order, (b, n))]
    y = np.einsum("bmn,bn->bm", h, x) + np.sqrt(nv / 2) * (
        rng.standard_normal((b, m)) + 1j * rng.standard_normal((b, m)))
    return h, y, x


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["zf", "mmse"])
def test_gpu_linear_matches_reference_golden(mode):
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    d, names = _cases()
    for name in names:
        m, n, order, b = d[f"{name}_meta"]
        c = constellation_for(int(order))
        for suffix, nv in (("", 0.05), ("_vec", d[f"{name}_nv_vec"])):
            lab, llr = D.linear_detect_batch(d[f"{name}_h"], d[f"{name}_y"], nv, c, mode)
            assert lab.dtype == np.int64 and llr.shape == (b, n, c.bits_per_symbol)
            np.testing.assert_array_equal(lab, d[f"{name}_{mode}_labels{suffix}"])
            np.testing.assert_allclose(llr, d[f"{name}_{mode}_llr{suffix}"], rtol=0,
                                       atol=LLR_ATOL)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["zf", "mmse"])
@pytest.mark.parametrize("m,n,order", [(12, 12, 16), (4, 4, 64), (16, 8, 4), (16, 16, 16),
                                       (24, 24, 64), (32, 32, 16), (40, 17, 64), (9, 9, 4)])
def test_gpu_linear_matches_oracle_random(mode, m, n, order):
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    rng = np.random.default_rng(m * 1000 + n * 10 + order)
    h, y, _ = _rand(rng, 4096, m, n, order, 0.03)
    lab, llr, est = D.linear_detect_batch(h, y, 0.03, constellation_for(order), mode,
                                          return_est=True)
    olab, ollr, oest = orc.linear_detect(h, y, 0.03, order, mode)
    # both sides solve A soft = H^H y in fp64 (LAPACK inverse there, Cholesky
    # here): the difference is bounded by ~eps * cond(A) * |soft|
    a = h.conj().transpose(0, 2, 1) @ h + (0.03 * np.eye(n) if mode == "mmse" else 0)
    tol = 1e-9 + 8 * 2.2e-16 * np.linalg.cond(a)[:, None]
    assert np.all(np.abs(est - oest) <= tol * np.abs(oest).max(axis=1, keepdims=True) + 1e-12)
    np.testing.assert_array_equal(lab, olab)
    np.testing.assert_allclose(llr, ollr, rtol=0, atol=LLR_ATOL)


@pytest.mark.gpu
def test_gpu_linear_reference_properties():
    """test_detect.py:28-86 restated on the batch entry."""
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    q4, q16 = constellation_for(4), constellation_for(16)
    # identity channel: ZF returns the nearest labels, MMSE soft = y / (1 + nv)
    h = np.broadcast_to(np.eye(2, dtype=complex), (3, 2, 2)).copy()
    y = np.array([[q4.points[0], q4.points[3]]] * 3)
    lab, _ = D.linear_detect_batch(h, y, 0.1, q4, "zf")
    np.testing.assert_array_equal(lab, [[0, 3]] * 3)
    for nv in (0.01, 0.5, 2.0):
        _, _, est = D.linear_detect_batch(h, y, nv, q4, "mmse", return_est=True)
        np.testing.assert_allclose(est, y / (1 + nv), rtol=1e-12)   # raw (biased) MMSE
    # noiseless consistency and the MMSE -> ZF limit
    rng = np.random.default_rng(5)
    h, _, x = _rand(rng, 256, 6, 4, 16, 0.0)
    labels = np.argmin(np.abs(x[..., None] - q16.points) ** 2, axis=-1)
    y = np.einsum("bmn,bn->bm", h, x)
    np.testing.assert_array_equal(D.linear_detect_batch(h, y, 1e-3, q16, "zf")[0], labels)
    np.testing.assert_array_equal(D.linear_detect_batch(h, y, 1e-9, q16, "mmse")[0], labels)
    # singular channel and unknown mode
    hs = np.zeros((2, 2, 2), complex)
    hs[:, :, 0] = hs[:, :, 1] = 1.0
    with pytest.raises(np.linalg.LinAlgError):
        D.linear_detect_batch(hs, np.ones((2, 2), complex), 0.1, q4, "zf")
    with pytest.raises(ValueError):
        D.linear_detect_batch(h, y, 0.1, q16, "lmmse")


@pytest.mark.gpu
def test_gpu_linear_nearly_dependent_columns_like_reference():
    """A Gram matrix that is numerically near-singular but has no exactly zero
    LU pivot: np.linalg.inv (the reference) returns without raising, so the
    batch must not raise either (the old 64-ulp Cholesky test raised
    here); an exactly singular one raises in both."""
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    q16 = constellation_for(16)
    rng = np.random.default_rng(3)
    h, y, _ = _rand(rng, 8, 4, 4, 16, 0.05)
    h[3, :, 3] = h[3, :, 2] + 1e-7 * h[3, :, 1]       # cond(H^H H) ~ 1e14-1e16
    gram = h.conj().transpose(0, 2, 1) @ h
    np.linalg.inv(gram)                               # the reference's step: no raise
    lab, llr = D.linear_detect_batch(h, y, 0.05, q16, "zf")
    assert lab.shape == (8, 4)
    olab, ollr, _ = orc.linear_detect(h[:3], y[:3], 0.05, 16, "zf")
    np.testing.assert_array_equal(lab[:3], olab)      # the well-conditioned rows agree
    hs = h.copy()
    hs[0] = 0.0                                       # exactly singular
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.inv(hs.conj().transpose(0, 2, 1) @ hs)
    with pytest.raises(np.linalg.LinAlgError):
        D.linear_detect_batch(hs, y, 0.05, q16, "zf")


@pytest.mark.gpu
def test_gpu_linear_device_tensors():
    import torch
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    rng = np.random.default_rng(11)
    h, y, _ = _rand(rng, 1000, 8, 8, 64, 0.02)
    lab, llr = D.linear_detect_batch(torch.from_numpy(h).cuda(), torch.from_numpy(y).cuda(),
                                     0.02, constellation_for(64), "mmse")
    assert lab.is_cuda and llr.is_cuda
    olab, ollr, _ = orc.linear_detect(h, y, 0.02, 64, "mmse")
    np.testing.assert_array_equal(lab.cpu().numpy(), olab)
    np.testing.assert_allclose(llr.cpu().numpy(), ollr, rtol=0, atol=LLR_ATOL)


@pytest.mark.gpu
def test_gpu_single_instance_zf_mmse():
    """zf_detect / mmse_detect / detect("zf"|"mmse") (detect.py:100-145, 563-576)
    restated from test_detect.py:28-86 on the single-instance shims."""
    from paper_2409_14355_b200 import detect as D
    from paper_2409_14355_b200.core import constellation_for
    q4, q16 = constellation_for(4), constellation_for(16)
    inp = D.DetectorInput(h=np.eye(2, dtype=complex), y=np.array([q4.points[0], q4.points[3]]),
                          noise_var=0.1, constellation=q4)
    np.testing.assert_array_equal(D.zf_detect(inp).hard_labels, [0, 3])
    np.testing.assert_array_equal(D.detect("zf", inp).hard_labels, [0, 3])
    for nv in (0.01, 0.5):
        y = np.array([0.3 + 0.1j, -0.2 - 0.7j])
        out = D.mmse_detect(D.DetectorInput(h=np.eye(2, dtype=complex), y=y, noise_var=nv,
                                            constellation=q4))
        np.testing.assert_allclose(out.soft, y / (1 + nv), rtol=1e-12)
    rng = np.random.default_rng(8)
    for _ in range(20):
        h, y, _ = _rand(rng, 1, 6, 4, 16, 0.02)
        inp = D.DetectorInput(h=h[0], y=y[0], noise_var=0.02, constellation=q16)
        for name, mode in (("zf", "zf"), ("mmse", "mmse")):
            out = D.detect(name, inp)
            olab, ollr, osoft = orc.linear_detect(h, y, 0.02, 16, mode)
            np.testing.assert_array_equal(out.hard_labels, olab[0])
            np.testing.assert_allclose(out.llrs, ollr[0], rtol=0, atol=LLR_ATOL)
            np.testing.assert_allclose(out.soft, osoft[0], rtol=1e-9)
            np.testing.assert_allclose(out.hard, q16.points[olab[0]])
    with pytest.raises(D.SingularChannelError):
        D.zf_detect(D.DetectorInput(h=np.ones((2, 2), complex), y=np.ones(2, complex),
                                    noise_var=0.1, constellation=q4))
    with pytest.raises(D.SingularChannelError):
        D.zf_detect(D.DetectorInput(h=np.ones((2, 3), complex), y=np.ones(2, complex),
                                    noise_var=0.1, constellation=q4))
