"""Full-size parity: every vector of every BASELINE config against the
UNMODIFIED reference (north-star bar: bit-matching detected symbols on all
five configs).

`tools/oracle_full.py` ran the reference package (`mpnlsim` 0.1.0 from
`baseline/_ref`, plan per RB tiled, `mpnl_detect_batch` + the hard composition
of `cli.py:236-239`) over ALL resource blocks of each config and committed,
per config, the sha256 of the (C, V, N) uint8 hard labels, a crc32 per RB, the
per-RB sum of winning metrics and the per-SNR bit-error counts
(`tests/golden/full_digests.json`).  The full outputs (hard, m1, m2) are
cached in `baseline/_ref/oracle_full/` (git-ignored, shipped to the GPU box).

Here the CUDA path detects the same full workload and must
* reproduce every RB's label crc32 (and the whole-config sha256); an RB whose
  crc differs is inspected vector by vector against the cache, where only a
  tie within 1e-5 relative of the two lowest reference metrics is exempt;
* keep every per-RB metric sum within 1e-4 relative (and, with the cache,
  every vector's winning metric within 1e-4 relative);
* give the same bit-error rate per SNR point within the reference's
  Monte-Carlo 95% interval (linksim.py:93-96) — C2's BER-vs-SNR curve.
"""

import hashlib
import json
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

ROOT = Path(__file__).resolve().parents[1]
DIGESTS = json.loads((ROOT / "tests" / "golden" / "full_digests.json").read_text())
CACHE = ROOT / "baseline" / "_ref" / "oracle_full"
pytestmark = pytest.mark.gpu

TIE_REL = 1e-5
METRIC_REL = 1e-4


def _detect_full_config(name):
    import torch
    from paper_2409_14355_b200 import detect as det
    d = generate(name)
    cfg = d["cfg"]
    c = constellation_for(cfg.order)
    h = torch.from_numpy(d["h"]).cuda()
    y = torch.from_numpy(d["y"]).cuda()
    plan = det.mpnl_plan_batch(h, float(d["nv"][0]), cfg.n_paths, c)
    hard, metric, flags = det.mpnl_detect_hard(plan, h, y, c, return_flags=True)
    torch.cuda.synchronize()
    return d, hard.cpu().numpy(), metric.cpu().numpy().astype(np.float64), flags.cpu().numpy()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_config_matches_reference(name):
    if name not in DIGESTS:
        pytest.fail(f"no reference digest for {name}: run tools/oracle_full.py {name}")
    ref = DIGESTS[name]
    d, hard, metric, flags = _detect_full_config(name)
    cfg = d["cfg"]
    assert hard.shape == (cfg.n_rb, cfg.vectors_per_channel, cfg.n)
    crc = [zlib.crc32(np.ascontiguousarray(hard[i]).tobytes()) for i in range(cfg.n_rb)]
    bad_rb = [i for i in range(cfg.n_rb) if crc[i] != ref["rb_crc32"][i]]
    cache = CACHE / f"{name}.npz"
    exempt = 0
    if bad_rb:
        assert cache.exists(), f"{name}: RBs {bad_rb[:8]} differ from the reference " \
                               "and no cached reference output to check the tie exemption"
        z = np.load(cache)
        bad_vec = []
        for i in bad_rb:
            m1, m2 = z["m1"][i], z["m2"][i]
            tie = (m2 - m1) <= TIE_REL * m1
            diff = np.any(hard[i] != z["hard"][i], axis=-1)
            bad_vec += [(i, int(v)) for v in np.nonzero(diff & ~tie)[0]]
            exempt += int(np.sum(diff & tie))
        assert not bad_vec, f"{name}: {len(bad_vec)} non-exempt mismatches (rb, re): {bad_vec[:10]}"
    else:
        assert hashlib.sha256(hard.tobytes()).hexdigest() == ref["sha256_hard"]
    # winning metric: per-RB sums always, every vector when the cache is present
    sums = metric.sum(axis=1)
    rel = np.abs(sums - np.asarray(ref["rb_m1_sum"])) / np.asarray(ref["rb_m1_sum"])
    assert rel.max() <= METRIC_REL, f"{name}: per-RB metric sum rel err {rel.max():.2e}"
    if cache.exists():
        z = np.load(cache)
        m1 = z["m1"]
        same = np.all(hard == z["hard"], axis=-1)
        r = np.abs(metric - m1) / np.maximum(m1, 1e-30)
        assert r[same].max() <= METRIC_REL, f"{name}: metric rel err {r[same].max():.2e}"
    # BER per SNR point within the reference's Monte-Carlo interval
    bps = cfg.order.bit_length() - 1
    for s, blk in enumerate(ref["ber_per_snr"]):
        sl = slice(s * 168, (s + 1) * 168)
        diff = hard[:, sl].astype(np.int64) ^ d["labels"][:, sl]
        errs = int(sum(int(np.sum((diff >> b) & 1)) for b in range(bps)))
        p = errs / blk["bits"]
        ci = 1.96 * np.sqrt(max(p * (1 - p), 1e-12) / blk["bits"])
        assert abs(p - blk["ber"]) <= blk["ci95"] + ci, \
            f"{name} @ {blk['snr_db']} dB: BER {p:.5f} vs reference {blk['ber']:.5f}"
    print(f"{name}: {hard.shape[0] * hard.shape[1]} vectors, {len(bad_rb)} RBs with tie-exempt "
          f"differences ({exempt} vectors), fp64 fix-up rate {flags.mean():.2e}")
