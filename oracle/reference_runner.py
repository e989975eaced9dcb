"""Runs the UNMODIFIED reference package on resource blocks — TEST / BASELINE
INFRASTRUCTURE ONLY (tests/, tools/oracle_full.py, bench.py's reference arm and
cpu_baseline leg; never the product path).

The reference (`mpnlsim` 0.1.0, pure Python/NumPy) is installed unchanged with
    python -m pip install --no-index --no-build-isolation --no-deps \
        --target baseline/_ref <copy of /root/reference/pkg>
(`baseline/_ref` is git-ignored and shipped to the GPU box by gpurun).  When it
is absent the read-only tree `/root/reference/pkg/src` is used (build
container only); `available()` says which.

`detect_rb_hard` is the reference's own hard-output composition
(`cli.py:236-239`: `mpnl_plan_batch` -> `mpnl_detect_batch` ->
`take_along_axis(labels, best)`) with one plan per RB whose rows are tiled over
the RB's vectors (`dataclasses.replace`, bit-identical to planning per vector).
"""

from __future__ import annotations

import dataclasses
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def ref_path():
    for p in _CANDIDATES:
        if (p / "mpnlsim" / "detect.py").exists():
            return p
    return None


def available():
    return ref_path() is not None


def _import():
    p = ref_path()
    if p is None:
        raise ImportError("reference package not installed (baseline/_ref) and "
                          "/root/reference not mounted")
    sys.dont_write_bytecode = True
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    from mpnlsim import detect as det
    from mpnlsim.core import constellation_for
    return det, constellation_for


def detect_rb_hard(args):
    """args = (h_rb (C,M,N), y_rb (C,V,M), noise_var, n_paths, order) ->
    (hard (C,V,N) uint8, m1 (C,V) f64 winning metric, m2 (C,V) f64 second-lowest)."""
    h_rb, y_rb, nv, n_paths, order = args
    det, constellation_for = _import()
    c = constellation_for(order)
    nch, v, _ = y_rb.shape
    n = h_rb.shape[2]
    hard = np.empty((nch, v, n), np.uint8)
    m1 = np.empty((nch, v))
    m2 = np.empty((nch, v))
    for i in range(nch):
        h1 = np.asarray(h_rb[i:i + 1], dtype=complex)
        plan = det.mpnl_plan_batch(h1, nv, n_paths, c)
        tiled = dataclasses.replace(plan, perm=np.repeat(plan.perm, v, 0),
                                    qh=np.repeat(plan.qh, v, 0), r=np.repeat(plan.r, v, 0))
        lab, met, best = det.mpnl_detect_batch(tiled, np.repeat(h1, v, axis=0),
                                               np.asarray(y_rb[i], dtype=complex), c)
        rows = np.arange(v)
        hard[i] = lab[rows, best]
        m1[i] = met[rows, best]
        m2[i] = np.partition(met, 1, axis=1)[:, 1] if met.shape[1] > 1 else np.inf
    return hard, m1, m2


def _init_worker():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:   # numpy may already have started its BLAS pool in a forked child
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def make_pool(workers):
    """A process pool of single-threaded workers (the cli.py:250-263 pattern)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    return ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                               initializer=_init_worker)


def split_tasks(h_rb, y_rb, nv, n_paths, order, vectors_per_task):
    """Whole RBs, or RBs cut into sub-batches of `vectors_per_task` vectors (each
    re-plans its RB: the QR is a few ms against seconds of path search)."""
    tasks, index = [], []
    v = y_rb.shape[1]
    step = max(1, min(int(vectors_per_task), v))
    for i in range(h_rb.shape[0]):
        for s in range(0, v, step):
            tasks.append((h_rb[i:i + 1], y_rb[i:i + 1, s:s + step], nv, n_paths, order))
            index.append((i, s, min(v, s + step)))
    return tasks, index


def run_tasks(pool, tasks, index, shape_cvn):
    c, v, n = shape_cvn
    hard = np.empty((c, v, n), np.uint8)
    m1 = np.empty((c, v))
    m2 = np.empty((c, v))
    for (i, s, e), (hh, a, b) in zip(index, pool.map(detect_rb_hard, tasks, chunksize=1)):
        hard[i, s:e], m1[i, s:e], m2[i, s:e] = hh[0], a[0], b[0]
    return hard, m1, m2
