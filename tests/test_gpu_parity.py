"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs (tests/golden, made by importing the reference) and against
the CPU oracle on fresh seeded inputs.

Bar (BASELINE.json north star):
* hard labels identical except where the oracle's two lowest path metrics
  tie within 1e-5 relative;
* winning metric within 1e-4 relative (fp32 fast path);
* full candidate list (fp64 kernel): labels/best identical, metrics 1e-9.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

GOLD = Path(__file__).resolve().parent / "golden"
pytestmark = pytest.mark.gpu

TIE_REL = 1e-5
METRIC_REL = 1e-4


def _det():
    from paper_2409_14355_b200 import detect
    return detect


def _check_hard(hard, metric, ref_hard, m1, m2, what):
    hard = np.asarray(hard).reshape(ref_hard.shape)
    metric = np.asarray(metric).reshape(m1.shape)
    exempt = (m2 - m1) <= TIE_REL * m1
    bad = np.any(hard != ref_hard, axis=-1) & ~exempt
    assert not bad.any(), f"{what}: {int(bad.sum())} vectors differ (of {bad.size}), " \
                          f"first at {np.argwhere(bad)[:3].tolist()}"
    rel = np.abs(metric - m1) / np.maximum(m1, 1e-30)
    assert np.all(rel[~exempt] <= METRIC_REL), f"{what}: metric rel err {rel.max():.2e}"
    return int(exempt.sum())


@pytest.mark.parametrize("name", ["C1", "C3", "C4", "C5P64"])
def test_plan_matches_reference(name):
    det = _det()
    g = np.load(GOLD / "plan.npz")
    h = g[f"{name}_h"]
    cfg = CONFIGS[name]
    plan = det.mpnl_plan_batch(h, 0.1, cfg.n_paths, constellation_for(cfg.order))
    assert np.array_equal(plan.perm, g[f"{name}_perm"])
    assert np.array_equal(plan.expansions, g[f"{name}_exp"])
    np.testing.assert_allclose(plan.r, g[f"{name}_r"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(plan.qh, g[f"{name}_qh"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("m,n,dt", [(8, 8, np.complex64), (16, 8, np.complex64), (24, 5, np.complex128),
                                    (32, 8, np.complex64), (12, 12, np.complex128),
                                    (24, 16, np.complex64), (32, 12, np.complex64),
                                    (24, 24, np.complex64), (32, 24, np.complex128),
                                    (32, 32, np.complex64), (31, 17, np.complex64),
                                    (40, 24, np.complex64), (64, 32, np.complex64),
                                    (3, 5, np.complex64), (20, 12, np.complex64),
                                    (12, 20, np.complex128), (24, 28, np.complex64),
                                    (1, 1, np.complex64), (7, 1, np.complex64)])
def test_plan_shapes_vs_oracle(m, n, dt):
    """Every plan-kernel instance (row-count bucket x lane-group width of the
    register kernel, the shared-memory CTA kernel beyond 32 rows; plain and
    augmented channels; both input types) against the oracle's sorted QR
    (itself pinned to the reference): same permutation, R and Q^H to 1e-11."""
    det = _det()
    rng = np.random.default_rng(1000 * m + n)
    nch = 37
    h = ((rng.standard_normal((nch, m, n)) + 1j * rng.standard_normal((nch, m, n)))
         / np.sqrt(2)).astype(dt)
    order = 16
    plan = det.mpnl_plan_batch(h, 0.2, 8, constellation_for(order))
    ref = orc.plan_channels(h, 0.2, 8, order)
    assert plan.augmented == (n > m)
    assert np.array_equal(plan.perm, ref.perm)
    np.testing.assert_allclose(plan.r, ref.r, rtol=0, atol=1e-11)
    np.testing.assert_allclose(plan.qh, ref.qh, rtol=0, atol=1e-11)


def test_plan_overloaded_matches_reference():
    det = _det()
    g = np.load(GOLD / "plan.npz")
    plan = det.mpnl_plan_batch(g["over_h"], 0.1, 32, constellation_for(4))
    assert plan.augmented
    assert np.array_equal(plan.perm, g["over_perm"])
    assert np.array_equal(plan.expansions, g["over_exp"])
    np.testing.assert_allclose(plan.r, g["over_r"], atol=1e-11)
    np.testing.assert_allclose(plan.qh, g["over_qh"], atol=1e-11)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_hard_matches_reference_golden(name):
    det = _det()
    g = np.load(GOLD / f"hard_{name}.npz")
    c = constellation_for(int(g["order"]))
    plan = det.mpnl_plan_batch(g["h"], float(g["nv"]), int(g["n_paths"]), c)
    hard, metric, flags = det.mpnl_detect_hard(plan, g["h"], g["y"], c, return_flags=True)
    _check_hard(hard, metric, g["hard"], g["m1"], g["m2"], name)
    print(f"{name}: flagged {flags.mean():.4%}")


@pytest.mark.parametrize("tag", ["c1", "c2", "c5p16", "c5p256"])
def test_full_list_matches_reference_golden(tag):
    det = _det()
    g = np.load(GOLD / f"full_{tag}.npz")
    c = constellation_for(int(g["order"]))
    plan = det.mpnl_plan_batch(g["h"], float(g["nv"]), int(g["n_paths"]), c)
    lab, met, best = det.mpnl_detect_batch(plan, g["h"], g["y"], c)
    lab, met, best = lab[0], met[0], best[0]
    assert np.array_equal(lab, g["labels"]), "path-ordered labels differ"
    np.testing.assert_allclose(met, g["metrics"], rtol=1e-9)
    assert np.array_equal(best, g["best"])


@pytest.mark.parametrize("tag", ["q4x4", "q4full", "over2x3", "q16_4x4"])
def test_full_list_small_cases(tag):
    det = _det()
    g = np.load(GOLD / f"full_{tag}.npz")
    c = constellation_for(int(g["order"]))
    plan = det.mpnl_plan_batch(g["h"], float(g["nv"]), int(g["n_paths"]), c)
    assert np.array_equal(plan.perm, g["perm"])
    lab, met, best = det.mpnl_detect_batch(plan, g["h"], g["y"], c)
    assert np.array_equal(lab, g["labels"])
    np.testing.assert_allclose(met, g["metrics"], rtol=1e-9, atol=1e-12)
    assert np.array_equal(best, g["best"])
    hard, m1 = det.mpnl_detect_hard(plan, g["h"], g["y"], c)
    rows = np.arange(len(best))
    assert np.array_equal(hard, g["labels"][rows, g["best"]])
    np.testing.assert_allclose(m1, g["metrics"][rows, g["best"]], rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("name,n_rb", [("C1", 4), ("C2", 6), ("C3", 6), ("C4", 3),
                                       ("C5P16", 12), ("C5P64", 6), ("C5P256", 3)])
def test_hard_vs_oracle_fresh_inputs(name, n_rb):
    """Fresh seeded RBs (not in the golden set) against the CPU oracle."""
    det = _det()
    d = generate(name, seed=99, n_rb=n_rb, rb_offset=1000)
    cfg = d["cfg"]
    c = constellation_for(cfg.order)
    ref_hard, m1, m2 = orc.detect_rb_parallel(d["h"], d["y"], d["nv"][0], cfg.n_paths,
                                              cfg.order, rbs_per_task=1)
    plan = det.mpnl_plan_batch(d["h"], d["nv"][0], cfg.n_paths, c)
    hard, metric = det.mpnl_detect_hard(plan, d["h"], d["y"], c)
    _check_hard(hard, metric, ref_hard.astype(np.uint8), m1, m2, name)


def test_deterministic_across_chunking():
    """Bit-identical outputs regardless of how vectors are grouped into calls."""
    import torch
    det = _det()
    d = generate("C2", n_rb=3)
    c = constellation_for(16)
    h = torch.from_numpy(d["h"]).cuda()
    y = torch.from_numpy(d["y"]).cuda()
    plan = det.mpnl_plan_batch(h, 0.5, 64, c)
    a_h, a_m = det.mpnl_detect_hard(plan, h, y, c)
    b_h, b_m = det.mpnl_detect_hard(plan, h, y, c)
    assert torch.equal(a_h, b_h) and torch.equal(a_m, b_m)
    # per-channel calls with half the vectors each
    for ch in range(3):
        sub = det.mpnl_plan_batch(h[ch:ch + 1], 0.5, 64, c)
        for lo, hi in ((0, 500), (500, 1008)):
            s_h, s_m = det.mpnl_detect_hard(sub, h[ch:ch + 1], y[ch:ch + 1, lo:hi].contiguous(), c)
            assert torch.equal(s_h[0], a_h[ch, lo:hi])
            assert torch.equal(s_m[0], a_m[ch, lo:hi])


@pytest.mark.parametrize("name", ["C2", "C5P1024"])
def test_noiseless_round_trip_full_size(name):
    """Size-independent property at full config size: y = Hx exactly ->
    every vector decodes to x (reference test_detect.py:290-299 at scale)."""
    import torch
    det = _det()
    cfg = CONFIGS[name]
    n_rb = cfg.n_rb if name == "C2" else 256
    d = generate(name, seed=5, n_rb=n_rb)
    c = constellation_for(cfg.order)
    h = torch.from_numpy(d["h"]).cuda()
    x = torch.from_numpy(c.points[d["labels"]]).cuda()
    y = torch.einsum("cmn,cvn->cvm", h.to(torch.complex128), x).to(torch.complex64)
    plan = det.mpnl_plan_batch(h, 0.01, cfg.n_paths, c)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    assert torch.equal(hard.long().cpu(), torch.from_numpy(d["labels"]))
    assert float(metric.max()) < 1e-4


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5P64"])
def test_host_pipeline_matches_reference_golden(name):
    """The host-buffer drop-in (C-ABI mpnl_detect_hard_host) against the
    reference goldens."""
    import torch
    det = _det()
    g = np.load(GOLD / f"hard_{name}.npz")
    cfg = CONFIGS[name]
    c = constellation_for(cfg.order)
    h = torch.from_numpy(np.ascontiguousarray(g["h"])).pin_memory()
    y = torch.from_numpy(np.ascontiguousarray(g["y"])).pin_memory()
    hard, metric = det.mpnl_hard_output(h, y, float(g["nv"]), cfg.n_paths, c, chunk_channels=1)
    _check_hard(hard.numpy().astype(np.int64), metric.numpy().astype(np.float64), g["hard"],
                g["m1"], g["m2"], f"{name} host pipeline")


@pytest.mark.parametrize("name,n_rb,chunk", [("C2", 7, 2), ("C5P16", 5, 1), ("C3", 9, 4)])
def test_host_pipeline_equals_device_path(name, n_rb, chunk):
    """Chunked, three-stream pipelined host path == one-shot device path,
    bit for bit (ragged last chunk, both device slots reused)."""
    import torch
    det = _det()
    cfg = CONFIGS[name]
    c = constellation_for(cfg.order)
    d = generate(cfg, seed=77, n_rb=n_rb)
    nv = float(d["nv"][0])
    h = torch.from_numpy(d["h"]).pin_memory()
    y = torch.from_numpy(d["y"]).pin_memory()
    hard, metric = det.mpnl_hard_output(h, y, nv, cfg.n_paths, c, chunk_channels=chunk)
    plan = det.mpnl_plan_batch(h.cuda(), nv, cfg.n_paths, c)
    hd, md = det.mpnl_detect_hard(plan, h.cuda(), y.cuda(), c)
    assert torch.equal(hd.cpu(), hard)
    assert torch.equal(md.cpu(), metric)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5P16", "C5P256"])
def test_large_batch_tiled_golden(name):
    """The golden RBs tiled into a batch of >= 151,552 vectors, which takes the
    large-batch kernel variants (one prep thread per vector, fused selection):
    every copy must reproduce the reference golden."""
    import torch
    det = _det()
    g = np.load(GOLD / f"hard_{name}.npz")
    cfg = CONFIGS[name]
    c = constellation_for(cfg.order)
    n_ch, V = g["y"].shape[:2]
    reps = -(-151552 // (n_ch * V))
    h = torch.from_numpy(np.ascontiguousarray(g["h"])).cuda().repeat(reps, 1, 1)
    y = torch.from_numpy(np.ascontiguousarray(g["y"])).cuda().repeat(reps, 1, 1)
    plan = det.mpnl_plan_batch(h, float(g["nv"]), int(g["n_paths"]), c)
    hard, metric = det.mpnl_detect_hard(plan, h, y, c)
    hard = hard.cpu().numpy().reshape(reps, n_ch, V, -1)
    metric = metric.cpu().numpy().reshape(reps, n_ch, V)
    for r in (0, reps // 2, reps - 1):
        _check_hard(hard[r].astype(np.int64), metric[r].astype(np.float64), g["hard"], g["m1"],
                    g["m2"], f"{name} tile {r}")
    assert (hard == hard[:1]).all() and (metric == metric[:1]).all()


@pytest.mark.parametrize("name,n_rb", [("C2", 9), ("C3", 5), ("C5P16", 3)])
def test_device_one_call_matches_staged_path(name, n_rb):
    """mpnl_plan_detect_hard (one C-ABI call, 1..4 channel groups on forked
    streams) is identical to mpnl_plan_batch + mpnl_detect_hard."""
    import torch
    det = _det()
    d = generate(name, n_rb=n_rb)
    cfg = d["cfg"]
    c = constellation_for(cfg.order)
    h = torch.from_numpy(d["h"]).cuda()
    y = torch.from_numpy(d["y"]).cuda()
    nv = float(d["nv"][0])
    plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    ref_h, ref_m = det.mpnl_detect_hard(plan, h, y, c)
    for g in (1, 2, 3, 4):
        hd, md = det.mpnl_hard_output_device(h, y, nv, cfg.n_paths, c, groups=g)
        torch.cuda.synchronize()
        assert torch.equal(hd, ref_h) and torch.equal(md, ref_m), f"groups={g}"
    with pytest.raises(ValueError):
        det.mpnl_hard_output_device(h, y, nv, cfg.n_paths, c, groups=5)


@pytest.mark.parametrize("m,n,order", [(8, 8, 16), (12, 12, 16), (16, 16, 64), (3, 5, 4)])
def test_plan_kernels_bit_identical(m, n, order):
    """Plans never depend on the batch size: channels of m (+ n) <= 32 rows all
    take the register-resident lane-group kernel (one arithmetic order whatever
    the number of channels, groups per warp or CTAs)."""
    import torch
    det = _det()
    c = constellation_for(order)
    rng = np.random.default_rng(m * 100 + n)
    h = ((rng.standard_normal((1100, m, n)) + 1j * rng.standard_normal((1100, m, n)))
         / np.sqrt(2)).astype(np.complex64)
    big = det.mpnl_plan_batch(torch.from_numpy(h).cuda(), 0.3, 32, c)
    small = det.mpnl_plan_batch(torch.from_numpy(h[:40]).cuda(), 0.3, 32, c)
    # (the table blob mixes fp64 and fp32 fields: compare its bits)
    for a, b in ((big.perm_dev, small.perm_dev), (big.r_dev, small.r_dev),
                 (big.qh_dev, small.qh_dev),
                 (big.tables.view(torch.int32), small.tables.view(torch.int32))):
        assert torch.equal(a[:40], b), "plan kernels disagree"
