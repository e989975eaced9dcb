"""The reference's own MPNL tests (pkg/tests/test_detect.py:184-354,
test_acceptance.py criterion 2) restated against the drop-in API, so they read
like the reference's tests but run the B200 kernels."""

import numpy as np
import pytest

from paper_2409_14355_b200.core import QAM16, QPSK

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def det():
    from paper_2409_14355_b200 import detect
    return detect


def rand_channel(rng, m, n):
    return (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))) / np.sqrt(2)


def rand_instance(det, rng, m, n, c, snr_db):
    h = rand_channel(rng, m, n)
    labels = rng.integers(0, c.order, n)
    nv = n / 10 ** (snr_db / 10)
    noise = np.sqrt(nv / 2) * (rng.standard_normal(m) + 1j * rng.standard_normal(m))
    return det.DetectorInput(h=h, y=h @ c.points[labels] + noise, noise_var=nv,
                             constellation=c), labels


def ml_brute(inp):
    """Exhaustive ML with lexicographic tie-break (test-side oracle)."""
    c, n = inp.constellation, inp.n
    idx = np.arange(c.order ** n)
    labs = np.stack([(idx // c.order ** (n - 1 - j)) % c.order for j in range(n)], axis=1)
    res = inp.y[None, :] - c.points[labs] @ inp.h.T
    met = np.sum(np.abs(res) ** 2, axis=1)
    b = int(np.argmin(met))
    r = inp.y - inp.h @ c.points[labs[b]]
    return labs[b], float(np.real(np.vdot(r, r)))


def test_plan_invariants(det):
    rng = np.random.default_rng(21)
    h = rand_channel(rng, 4, 4)
    plan = det.mpnl_preprocess(h, 0.1, 32, QPSK)
    r = plan.r_factor
    assert np.allclose(np.tril(r, -1), 0)
    assert np.all(np.diag(r).real > 0)
    assert np.all(np.abs(np.diag(r).imag) < 1e-12)
    assert np.prod(plan.expansions) == plan.n_paths == 32
    assert sorted(plan.ordering) == list(range(4))
    diag = np.diag(r).real
    assert diag[0] == max(diag)


def test_plan_reconstructs_channel(det):
    rng = np.random.default_rng(22)
    h = rand_channel(rng, 6, 4)
    plan = det.mpnl_preprocess(h, 0.1, 16, QPSK)
    assert np.allclose(plan.q_factor @ plan.r_factor, h[:, plan.ordering], atol=1e-10)


def test_plan_warns_when_budget_below_forced(det):
    rng = np.random.default_rng(23)
    with pytest.warns(UserWarning, match="rank-deficient"):
        det.mpnl_preprocess(rand_channel(rng, 1, 3), 0.1, 8, QPSK)


@pytest.mark.parametrize("n", [2, 4])
def test_full_enumeration_equals_ml(det, n):
    rng = np.random.default_rng(31 + n)
    for _ in range(100):
        inp, _ = rand_instance(det, rng, n, n, QPSK, 10.0)
        plan = det.mpnl_preprocess(inp.h, inp.noise_var, 4 ** n, QPSK)
        _, out = det.mpnl_detect(plan, inp)
        lab, met = ml_brute(inp)
        assert np.array_equal(out.hard_labels, lab)
        assert out.min_metric == met


def test_single_path_equals_sic(det):
    rng = np.random.default_rng(41)
    for _ in range(200):
        inp, _ = rand_instance(det, rng, 4, 4, QPSK, 12.0)
        plan = det.mpnl_preprocess(inp.h, inp.noise_var, 1, QPSK)
        _, out = det.mpnl_detect(plan, inp)
        hp = inp.h[:, plan.ordering]
        q, r = np.linalg.qr(hp)
        ph = np.diag(r) / np.abs(np.diag(r))
        r = (r.T * ph.conj()).T
        z = (q * ph).conj().T @ inp.y
        sic = np.zeros(4, dtype=np.int64)
        x = np.zeros(4, dtype=complex)
        for i in range(3, -1, -1):
            sic[i] = QPSK.nearest((z[i] - r[i, i + 1:] @ x[i + 1:]) / r[i, i])
            x[i] = QPSK.points[sic[i]]
        expect = np.empty(4, dtype=np.int64)
        expect[plan.ordering] = sic
        assert np.array_equal(out.hard_labels, expect)
        # the fast hard path agrees
        hard, _ = det.mpnl_detect_hard(plan._batch, inp.h[None], inp.y[None], QPSK)
        assert np.array_equal(hard[0], expect)


def test_noiseless_any_budget(det):
    rng = np.random.default_rng(51)
    for npaths in (1, 2, 4, 8, 32):
        h = rand_channel(rng, 4, 4)
        labels = rng.integers(0, 4, 4)
        inp = det.DetectorInput(h=h, y=h @ QPSK.points[labels], noise_var=0.01,
                                constellation=QPSK)
        _, out = det.mpnl_detect(det.mpnl_preprocess(h, 0.01, npaths, QPSK), inp)
        assert np.array_equal(out.hard_labels, labels)


def test_metric_dominates_ml(det):
    rng = np.random.default_rng(61)
    for _ in range(100):
        inp, _ = rand_instance(det, rng, 4, 4, QPSK, 5.0)
        _, out = det.mpnl_detect(det.mpnl_preprocess(inp.h, inp.noise_var, 8, QPSK), inp)
        assert out.min_metric >= ml_brute(inp)[1] - 1e-12


def test_candidates_nested_under_doubling(det):
    rng = np.random.default_rng(71)
    inp, _ = rand_instance(det, rng, 4, 4, QPSK, 8.0)
    prev = None
    for k in (1, 2, 4, 8, 16, 32):
        clist, _ = det.mpnl_detect(det.mpnl_preprocess(inp.h, inp.noise_var, k, QPSK), inp)
        cur = {tuple(row) for row in clist.labels}
        assert len(cur) == k
        if prev is not None:
            assert prev <= cur
        prev = cur


def test_candidate_metrics_consistent(det):
    rng = np.random.default_rng(81)
    inp, _ = rand_instance(det, rng, 4, 4, QAM16, 15.0)
    clist, out = det.mpnl_detect(det.mpnl_preprocess(inp.h, inp.noise_var, 16, QAM16), inp)
    for cand, metric in zip(clist.candidates, clist.metrics):
        assert metric == pytest.approx(np.sum(np.abs(inp.y - inp.h @ cand) ** 2), rel=1e-9)
    assert out.min_metric == pytest.approx(clist.metrics.min(), rel=1e-12)


def test_fingerprint_mismatch_rejected(det):
    rng = np.random.default_rng(91)
    inp, _ = rand_instance(det, rng, 2, 2, QPSK, 10.0)
    plan = det.mpnl_preprocess(rand_channel(rng, 2, 2), inp.noise_var, 4, QPSK)
    with pytest.raises(ValueError, match="fingerprint"):
        det.mpnl_detect(plan, inp)


def test_overloaded_runs(det):
    rng = np.random.default_rng(101)
    h = rand_channel(rng, 2, 3)
    labels = rng.integers(0, 4, 3)
    inp = det.DetectorInput(h=h, y=h @ QPSK.points[labels], noise_var=1e-4,
                            constellation=QPSK)
    plan = det.mpnl_preprocess(h, 1e-4, 32, QPSK)
    assert plan.expansions[2] == 4
    _, out = det.mpnl_detect(plan, inp)
    assert np.array_equal(out.hard_labels, labels)
    hard, _ = det.mpnl_detect_hard(plan._batch, h[None], inp.y[None], QPSK)
    assert np.array_equal(hard[0], labels)


def test_detect_dispatch(det):
    rng = np.random.default_rng(7)
    inp, _ = rand_instance(det, rng, 4, 4, QAM16, 20.0)
    out = det.detect("mpnl", inp, n_paths=16)
    assert out.hard_labels.shape == (4,) and out.llrs.shape == (4, 4)
    with pytest.raises(ValueError):
        det.detect("nope", inp)


def test_invalid_arguments(det):
    with pytest.raises(ValueError, match="n_paths must be >= 1"):
        det.allocate_expansions(3, 4, 0)
    rng = np.random.default_rng(3)
    plan = det.mpnl_plan_batch(rand_channel(rng, 4, 4)[None], 0.1, 8, QPSK)
    with pytest.raises(ValueError):
        det.mpnl_detect_hard(plan, None, np.zeros((2, 4), complex), QPSK)   # batch mismatch
    with pytest.raises(NotImplementedError):
        det.mpnl_plan_batch(rand_channel(rng, 33, 33)[None], 0.1, 8, QPSK)


def test_detect_requires_the_planned_channel():
    """The metric is the plan's PED, which is the reference's true residual
    ||y - Hx||^2 (detect.py:484-486) for the PLANNED channel: the same channel
    (object or equal data) is accepted, another one raises."""
    import torch
    from paper_2409_14355_b200 import detect as det
    rng = np.random.default_rng(4)
    h = (rng.standard_normal((3, 4, 4)) + 1j * rng.standard_normal((3, 4, 4))) / np.sqrt(2)
    y = (rng.standard_normal((3, 5, 4)) + 1j * rng.standard_normal((3, 5, 4)))
    plan = det.mpnl_plan_batch(h, 0.1, 16, QPSK)
    a = det.mpnl_detect_hard(plan, h, y, QPSK)
    b = det.mpnl_detect_hard(plan, h.copy(), y, QPSK)            # equal data: fine
    c = det.mpnl_detect_hard(plan, torch.from_numpy(h).cuda(), y, QPSK)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[0], c[0])
    with pytest.raises(ValueError, match="differs"):
        det.mpnl_detect_hard(plan, 2 * h, y, QPSK)
    with pytest.raises(ValueError, match="differs"):
        det.mpnl_detect_batch(plan, 2 * h, y, QPSK)
