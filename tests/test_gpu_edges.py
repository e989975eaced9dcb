"""Edge cases of the drop-in detector, each against the CPU oracle (which is
pinned to the reference): empty and ragged batches, a single stream, tall
channels (M > N: the metric offset), P = 1 (pure SIC), a path budget above
Q^N (capped), complex128 inputs, non-contiguous inputs, the host pipeline with
more chunks than channels, and the C ABI's error codes."""

import numpy as np
import pytest

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.core import constellation_for

pytestmark = pytest.mark.gpu
TIE_REL, METRIC_REL = 1e-5, 1e-4


def _det():
    from paper_2409_14355_b200 import detect
    return detect


def _case(rng, n_ch, v, m, n, order, snr_db=12.0):
    c = constellation_for(order)
    h = ((rng.standard_normal((n_ch, m, n)) + 1j * rng.standard_normal((n_ch, m, n)))
         / np.sqrt(2)).astype(np.complex64)
    lab = rng.integers(0, order, (n_ch, v, n))
    nv = n / 10 ** (snr_db / 10)
    noise = np.sqrt(nv / 2) * (rng.standard_normal((n_ch, v, m))
                               + 1j * rng.standard_normal((n_ch, v, m)))
    y = (np.einsum("cmn,cvn->cvm", h.astype(complex), c.points[lab]) + noise).astype(np.complex64)
    return c, h, y, nv


def _check(h, y, nv, n_paths, c, hard, metric):
    ref, m1, m2 = orc.detect_rb(h, y, nv, n_paths, c.order, c.points)
    exempt = (m2 - m1) <= TIE_REL * m1
    bad = np.any(np.asarray(hard) != ref, axis=-1) & ~exempt
    assert not bad.any(), f"{int(bad.sum())} vectors differ"
    rel = np.abs(np.asarray(metric, dtype=np.float64) - m1) / np.maximum(m1, 1e-30)
    assert np.all(rel[~exempt] <= METRIC_REL)


@pytest.mark.parametrize("m,n,order,p", [(1, 1, 16, 4), (6, 3, 16, 16), (16, 8, 64, 64),
                                         (8, 8, 16, 1), (2, 2, 4, 100), (24, 20, 64, 64)])
def test_shapes_vs_oracle(m, n, order, p):
    det = _det()
    rng = np.random.default_rng(m * 131 + n * 17 + p)
    c, h, y, nv = _case(rng, 3, 40, m, n, order)
    plan = det.mpnl_plan_batch(h, nv, p, c)
    assert plan.n_paths == min(p, order ** n)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    _check(h, y, nv, p, c, hard, metric)


@pytest.mark.parametrize("n,p", [(6, 8), (6, 16), (6, 32), (6, 512), (6, 1024), (6, 2048),
                                 (6, 96), (4, 8192), (20, 1024)])
def test_64qam_partial_layer_selections(n, p):
    """64-QAM trees whose partial layer takes E = 8 / 16 / 32 / 48 of the 64 points, at the
    top or under a full top layer (and a three-layer tree): the key-ordered selection merge
    (select_kernel, L = 8) and its widened cut guard, hard output and fp32 LLRs vs the oracle."""
    det = _det()
    rng = np.random.default_rng(7000 + 13 * n + p)
    c, h, y, nv = _case(rng, 3, 32, n, n, 64, snr_db=20.0)
    plan = det.mpnl_plan_batch(h, nv, p, c)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    _check(h, y, nv, p, c, hard, metric)
    if p <= 1024:
        llr = det.mpnl_detect_llrs(plan, h, y[:, :24].copy(), c, precision="fp32")
        ref = det.mpnl_detect_llrs(plan, h, y[:, :24].copy(), c)
        assert np.abs(llr - ref).max() <= 1e-3


@pytest.mark.parametrize("n,order,p", [(6, 64, 1024), (8, 16, 256), (6, 64, 16), (12, 16, 64),
                                       (24, 64, 64)])
@pytest.mark.parametrize("kind,metric_rel", [("y*30", 1e-4), ("y*1000", 1e-4), ("y*1e-4", 1e-4),
                                             ("cols40dB", 1e-4), ("cols80dB", 1e-3)])
def test_out_of_range_inputs(n, order, p, kind, metric_rel):
    """Observations far outside the constellation (every slicing saturates, selection centres
    far off the grid), tiny observations, and channels whose columns differ by 40 / 80 dB in
    power: labels equal the oracle's (tie exemption as everywhere).  The fp32 metric keeps the
    1e-4 bound up to 40 dB of column range; at 80 dB the fp32 rounding of the rotated
    observation is 3e-4 of the (then tiny) residual -- a documented limit."""
    det = _det()
    rng = np.random.default_rng(n * 7 + p)
    c = constellation_for(order)
    h = ((rng.standard_normal((3, n, n)) + 1j * rng.standard_normal((3, n, n)))
         / np.sqrt(2)).astype(np.complex64)
    if kind == "cols40dB":
        h = (h * np.asarray([1, 0.1, 10] * 8, np.float32)[None, None, :n]).astype(np.complex64)
    if kind == "cols80dB":
        h = (h * np.asarray([1, 1e-2, 1e2] * 8, np.float32)[None, None, :n]).astype(np.complex64)
    ysc = {"y*30": 30.0, "y*1000": 1000.0, "y*1e-4": 1e-4}.get(kind, 1.0)
    lab = rng.integers(0, order, (3, 24, n))
    nv = 0.05
    noise = np.sqrt(nv / 2) * (rng.standard_normal((3, 24, n)) + 1j * rng.standard_normal((3, 24, n)))
    y = ((np.einsum("cmn,cvn->cvm", h.astype(complex), c.points[lab]) + noise) * ysc
         ).astype(np.complex64)
    plan = det.mpnl_plan_batch(h, nv, p, c)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    ref, m1, m2 = orc.detect_rb(h, y, nv, p, c.order, c.points)
    exempt = (m2 - m1) <= TIE_REL * m1
    bad = np.any(np.asarray(hard) != ref, axis=-1) & ~exempt
    assert not bad.any(), f"{int(bad.sum())} vectors differ"
    rel = np.abs(np.asarray(metric, dtype=np.float64) - m1) / np.maximum(m1, 1e-300)
    assert np.all(rel[~exempt] <= metric_rel)


@pytest.mark.parametrize("n,order,p", [(8, 16, 256), (6, 64, 1024), (4, 4, 16), (12, 16, 64),
                                       (8, 16, 32)])
def test_all_zero_observations_tie_rules(n, order, p):
    """y = 0: every SIC decision sits exactly on a slicing boundary and every path ties with
    its negation, so the result is decided by the reference's tie rules alone (stable argsort
    of equal distances, lexsort on (metric, labels)).  No tie exemption here: every vector
    goes through the guard, the event checks and the fp64 fix-up (a cluster of CTAs per
    vector for the trees of >= 256 paths) and must equal the oracle's labels exactly."""
    det = _det()
    rng = np.random.default_rng(n * 7 + p)
    c = constellation_for(order)
    h = ((rng.standard_normal((3, n, n)) + 1j * rng.standard_normal((3, n, n)))
         / np.sqrt(2)).astype(np.complex64)
    y = np.zeros((3, 8, n), np.complex64)
    plan = det.mpnl_plan_batch(h, 0.1, p, c)
    hard, metric, flags = det.mpnl_detect_hard(plan, h, y, c, return_flags=True)
    ref, m1, _ = orc.detect_rb(h, y, 0.1, p, c.order, c.points)
    assert np.array_equal(np.asarray(hard), ref)
    assert np.allclose(np.asarray(metric, dtype=np.float64), m1, rtol=METRIC_REL)
    assert np.asarray(flags).any()   # the fp64 fix-up did run


@pytest.mark.parametrize("n_ch,v,m,n,order,p", [(300, 1, 8, 8, 16, 32), (257, 3, 12, 12, 16, 64),
                                                (70, 2, 24, 24, 64, 64), (40, 1, 32, 32, 16, 32),
                                                (9, 1, 8, 8, 16, 32), (130, 5, 16, 16, 64, 16)])
def test_few_vectors_per_channel(n_ch, v, m, n, order, p):
    """One H per vector (the reference's own bench shape, cli.py:227-239) and
    other channels with only a few vectors: the traversal's warp-per-channel
    mode (every warp stages its own channel's tables), against the oracle."""
    det = _det()
    rng = np.random.default_rng(n_ch * 100 + v)
    c, h, y, nv = _case(rng, n_ch, v, m, n, order, snr_db=16.0)
    plan = det.mpnl_plan_batch(h, nv, p, c)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    _check(h, y, nv, p, c, hard, metric)
    llr = det.mpnl_detect_llrs(plan, h, y, c, precision="fp32")
    ref = det.mpnl_detect_llrs(plan, h, y, c)
    assert np.abs(llr - ref).max() <= 1e-3


def test_empty_and_ragged_batches():
    import torch
    det = _det()
    rng = np.random.default_rng(3)
    c, h, y, nv = _case(rng, 2, 5, 4, 4, 16)
    plan = det.mpnl_plan_batch(h, nv, 16, c)
    hard, metric = det.mpnl_detect_hard(plan, h, y[:, :0], c)          # V = 0
    assert hard.shape == (2, 0, 4) and metric.shape == (2, 0)
    e = det.mpnl_plan_batch(np.zeros((0, 4, 4), np.complex64), nv, 16, c)   # no channels
    hd, md = det.mpnl_detect_hard(e, None, np.zeros((0, 3, 4), np.complex64), c)
    assert hd.shape == (0, 3, 4)
    # a single vector (1-D y) and a batch of vectors (2-D y) against 1-channel plans
    one = det.mpnl_plan_batch(h[:1], nv, 16, c)
    h1, m1 = det.mpnl_detect_hard(one, h[:1], y[0, 0], c)
    assert h1.shape == (4,) and np.ndim(m1) == 0
    hb, mb = det.mpnl_detect_hard(one, h[:1], y[:1, :3].reshape(1, 3, 4), c)
    assert np.array_equal(hb[0, 0], h1)
    # complex128 and non-contiguous device inputs give the same labels
    yt = torch.from_numpy(y.astype(np.complex128)).cuda()
    plan128 = det.mpnl_plan_batch(torch.from_numpy(h.astype(np.complex128)).cuda(), nv, 16, c)
    a, _ = det.mpnl_detect_hard(plan128, None, yt, c)
    wide = torch.zeros((2, 10, 4), dtype=torch.complex128, device="cuda")
    wide[:, ::2] = yt
    b, _ = det.mpnl_detect_hard(plan128, None, wide[:, ::2], c)
    assert torch.equal(a, b)
    ref, _ = det.mpnl_detect_hard(plan, h, y, c)
    assert np.array_equal(a.cpu().numpy(), ref.astype(np.uint8))


def test_host_pipeline_more_chunks_than_channels():
    import torch
    det = _det()
    rng = np.random.default_rng(9)
    c, h, y, nv = _case(rng, 3, 168, 12, 12, 16)
    hard, metric = det.mpnl_hard_output(torch.from_numpy(h).pin_memory(),
                                        torch.from_numpy(y).pin_memory(), nv, 64, c,
                                        chunk_channels=1)
    _check(h, y, nv, 64, c, hard.numpy(), metric.numpy())


def test_c_abi_error_codes():
    import ctypes
    from paper_2409_14355_b200 import _lib
    lib = _lib.load()
    ex = np.zeros(40, np.int64)
    real = np.zeros(1, np.int64)
    assert lib.mpnl_alloc_expansions(4, 16, 0, 0, ex.ctypes.data, real.ctypes.data,
                                     None) == _lib.MPNL_EINVAL
    assert b"n_paths must be >= 1" in lib.mpnl_last_error()
    dummy = ctypes.c_void_p(0)
    # N > 32, unsupported Q
    assert lib.mpnl_plan(dummy, 0, 1, 40, 33, 16, 0.1, dummy, dummy, dummy, dummy,
                         dummy) == _lib.MPNL_EUNSUPPORTED
    assert lib.mpnl_plan(dummy, 0, 1, 4, 4, 8, 0.1, dummy, dummy, dummy, dummy,
                         dummy) == _lib.MPNL_EUNSUPPORTED
    # overloaded without a positive noise variance
    assert lib.mpnl_plan(dummy, 0, 1, 2, 3, 4, 0.0, dummy, dummy, dummy, dummy,
                         dummy) == _lib.MPNL_EINVAL
