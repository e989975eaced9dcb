"""Full-size reference outputs for every BASELINE config (test infrastructure).

    PYTHONDONTWRITEBYTECODE=1 python tools/oracle_full.py [CFG ...] [--workers W]

Runs the UNMODIFIED reference package (`baseline/_ref/mpnlsim`, installed from
/root/reference/pkg with pip --target; falls back to /root/reference/pkg/src)
on ALL resource blocks of each config's seeded workload (`workloads.generate`):
one `mpnl_plan_batch` per RB whose perm / qh / r rows are tiled over the RB's
vectors (`dataclasses.replace`; bit-identical to planning per vector, SURVEY
§0.7), then `mpnl_detect_batch` and the hard composition of `cli.py:236-239`.

Writes `baseline/_ref/oracle_full/<cfg>.npz` (git-ignored, shipped to the GPU
box by gpurun) with hard (C,V,N) uint8, m1 / m2 (C,V) float64 (winning and
second-lowest path metric, for the tie exemption), and appends the sha256 of
the hard labels and the per-RB digests to `tests/golden/full_digests.json`
(committed), so the GPU parity test can check every vector even on a box where
the cache is absent.
"""

from __future__ import annotations

import argparse
import dataclasses
import hashlib
import json
import os
import sys
import time
import zlib

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "baseline" / "_ref" / "oracle_full"
DIGESTS = ROOT / "tests" / "golden" / "full_digests.json"


def _ref_path():
    cand = ROOT / "baseline" / "_ref"
    if (cand / "mpnlsim").is_dir():
        return str(cand)
    return "/root/reference/pkg/src"


def _worker(args):
    h_rb, y_rb, nv, n_paths, order = args
    sys.dont_write_bytecode = True
    if _ref_path() not in sys.path:
        sys.path.insert(0, _ref_path())
    from mpnlsim import detect as det
    from mpnlsim.core import constellation_for
    c = constellation_for(order)
    nch, v, m = y_rb.shape
    n = h_rb.shape[2]
    hard = np.empty((nch, v, n), np.uint8)
    m1 = np.empty((nch, v))
    m2 = np.empty((nch, v))
    for i in range(nch):
        h1 = h_rb[i:i + 1].astype(complex)
        plan = det.mpnl_plan_batch(h1, nv, n_paths, c)
        tiled = dataclasses.replace(plan, perm=np.repeat(plan.perm, v, 0),
                                    qh=np.repeat(plan.qh, v, 0), r=np.repeat(plan.r, v, 0))
        h = np.repeat(h1, v, axis=0)
        y = y_rb[i].astype(complex)
        lab, met, best = det.mpnl_detect_batch(tiled, h, y, c)
        rows = np.arange(v)
        hard[i] = lab[rows, best]
        m1[i] = met[rows, best]
        m2[i] = np.partition(met, 1, axis=1)[:, 1] if met.shape[1] > 1 else np.inf
    return hard, m1, m2


def rb_digests(hard):
    """crc32 of each RB's (V, N) uint8 label block."""
    return [zlib.crc32(np.ascontiguousarray(hard[i]).tobytes()) for i in range(hard.shape[0])]


def run(name, workers):
    from paper_2409_14355_b200.workloads import generate
    d = generate(name)
    cfg = d["cfg"]
    nv = d["nv"]
    snrs = len(cfg.snr_db)
    tasks = []
    # one task per (RB, SNR point); nv is scalar per task (the reference API)
    for i in range(cfg.n_rb):
        for s in range(snrs):
            ys = d["y"][i:i + 1, s * 168:(s + 1) * 168]
            tasks.append((d["h"][i:i + 1], ys, float(nv[s * 168]), cfg.n_paths, cfg.order))
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=workers) as pool:
        parts = list(pool.map(_worker, tasks, chunksize=1))
    v = cfg.vectors_per_channel
    hard = np.empty((cfg.n_rb, v, cfg.n), np.uint8)
    m1 = np.empty((cfg.n_rb, v))
    m2 = np.empty((cfg.n_rb, v))
    k = 0
    for i in range(cfg.n_rb):
        for s in range(snrs):
            sl = slice(s * 168, (s + 1) * 168)
            hard[i, sl], m1[i, sl], m2[i, sl] = (p[0] for p in parts[k])
            k += 1
    dt = time.time() - t0
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez(OUT / f"{name}.npz", hard=hard, m1=m1, m2=m2)
    digs = json.loads(DIGESTS.read_text()) if DIGESTS.exists() else {}
    truth_err = float(np.mean(hard.astype(np.int64) != d["labels"]))
    digs[name] = {
        "n_rb": cfg.n_rb, "vectors": int(cfg.n_vectors), "n": cfg.n,
        "sha256_hard": hashlib.sha256(hard.tobytes()).hexdigest(),
        "sha256_m1": hashlib.sha256(m1.tobytes()).hexdigest(),
        "rb_crc32": rb_digests(hard),
        "rb_m1_sum": [float(x) for x in m1.sum(axis=1)],
        "n_tie_exempt": int(np.sum((m2 - m1) <= 1e-5 * m1)),
        "symbol_error_rate_vs_tx": truth_err,
        "reference": "mpnlsim 0.1.0 (unmodified, " + _ref_path() + ")",
        "seconds": round(dt, 1), "workers": workers,
    }
    digs[name]["ber_per_snr"] = ber_per_snr(hard, d["labels"], cfg)
    DIGESTS.write_text(json.dumps(digs, indent=1) + "\n")
    print(f"{name}: {cfg.n_vectors} vectors in {dt:.1f} s, SER {truth_err:.4f}", flush=True)


def ber_per_snr(hard, tx_labels, cfg):
    """Bit errors of detected vs transmitted labels per SNR point, bits via the
    Gray label bits (core.py:209-213), with the reference's normal-approximation
    95% half-width (linksim.py:93-96)."""
    bps = cfg.order.bit_length() - 1
    out = []
    for s, snr in enumerate(cfg.snr_db):
        sl = slice(s * 168, (s + 1) * 168)
        diff = (hard[:, sl].astype(np.int64) ^ tx_labels[:, sl])
        errs = int(sum(int(np.sum((diff >> b) & 1)) for b in range(bps)))
        bits = int(diff.size * bps)
        p = errs / bits
        out.append({"snr_db": snr, "bit_errors": errs, "bits": bits, "ber": p,
                    "ci95": 1.96 * float(np.sqrt(max(p * (1 - p), 1e-12) / bits))})
    return out


def summarize(name):
    """(Re)compute the BER block of an existing cache."""
    from paper_2409_14355_b200.workloads import generate
    d = generate(name)
    hard = np.load(OUT / f"{name}.npz")["hard"]
    digs = json.loads(DIGESTS.read_text())
    digs[name]["ber_per_snr"] = ber_per_snr(hard, d["labels"], d["cfg"])
    DIGESTS.write_text(json.dumps(digs, indent=1) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5P16", "C5P64",
                                                   "C5P256", "C5P1024"])
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--summarize", action="store_true", help="only recompute BER blocks")
    a = ap.parse_args()
    for name in a.configs:
        summarize(name) if a.summarize else run(name, a.workers)


if __name__ == "__main__":
    main()
