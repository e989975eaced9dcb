"""CPU oracle for the MPNL hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import this module, and only as a checker / reported baseline.  The product
path (`paper_2409_14355_b200`) never calls it: it runs on the CUDA library and
fails loudly when that library is missing.

This is a numpy restatement of the reference detector
(`/root/reference/pkg/src/mpnlsim/detect.py`), step by step:

* ``allocate_expansions``  <- detect.py:221-280 (integer rule, same search order)
* ``sorted_qr``            <- detect.py:321-358 (column-pivoted right-looking MGS,
                              downdated norms, first-max pivot, r_kk floor 1e-300)
* ``plan_channels``        <- detect.py:361-388 (augmented [H; sqrt(nv) I] if N>M)
* ``expand_tree``          <- detect.py:403-428 (per layer: centre, |c-s|^2,
                              stable argsort, mixed-radix path index)
* ``to_stream_order``      <- detect.py:431-437
* ``true_metrics``         <- detect.py:484-486 (true residual ||y - Hx||^2)
* ``select_best``          <- detect.py:465-470 (lexsort: metric, then labels of
                              stream 0, 1, ...)
* ``detect_rb``            <- cli.py:236-239 / test_acceptance.py:114-117 hard
                              composition, with one plan per resource block tiled
                              over its vectors (bit-identical to per-vector plans).

Pinned against the reference itself: `tests/golden/make_golden.py` imports the
reference in the build container and stores its outputs; `tests/test_oracle.py`
asserts this module reproduces them (labels/best bit-exact, metrics to 1e-12).
"""

from __future__ import annotations

import warnings

import numpy as np


# --------------------------------------------------------------------------
# planning
# --------------------------------------------------------------------------

def _split_budget(budget, slots, cap):
    """Greedy largest-first factorisation of `budget` into <= `slots` factors
    each <= `cap` (non-increasing).  None when impossible.  (detect.py:240-251)"""
    if budget == 1:
        return []
    if slots == 0:
        return None
    d = min(cap, budget)
    while d >= 2:
        if budget % d == 0:
            tail = _split_budget(budget // d, slots - 1, d)
            if tail is not None:
                return [d] + tail
        d -= 1
    return None


def allocate_expansions(n_layers, q, n_paths, n_forced=0):
    """(expansions indexed by tree position, realized path count).

    Position n_layers-1 is the top layer.  detect.py:221-280.
    """
    if n_paths < 1:
        raise ValueError("n_paths must be >= 1")
    n_paths = min(n_paths, q ** n_layers)
    if n_forced > 0 and n_paths < q ** n_forced:
        warnings.warn(f"n_paths={n_paths} < {q}^{n_forced}: cannot fully expand "
                      "all rank-deficient layers", stacklevel=2)
    n_force = min(n_forced, n_layers)
    target = n_paths
    while target >= 1:
        fac, rem, bad = [], target, False
        for _ in range(n_force):
            if rem >= q:
                if rem % q:
                    bad = True
                    break
                fac.append(q)
                rem //= q
            else:
                fac.append(rem)
                rem = 1
        if not bad:
            tail = _split_budget(rem, n_layers - n_force, min(q, fac[-1]) if fac else q)
            if tail is not None:
                fac = sorted(fac + tail + [1] * (n_layers - len(fac) - len(tail)),
                             reverse=True)
                return np.array(fac[::-1], dtype=np.int64), target
        target -= 1
    raise AssertionError("unreachable")


def sorted_qr(a):
    """Column-pivoted MGS over a stack a (B, Ma, N) -> perm, q, r."""
    a = np.array(a, dtype=complex)
    nb, _, n = a.shape
    rows = np.arange(nb)
    perm = np.tile(np.arange(n), (nb, 1))
    r = np.zeros((nb, n, n), dtype=complex)
    colnorm = np.sum(np.abs(a) ** 2, axis=1)
    for k in range(n):
        p = k + np.argmax(colnorm[:, k:], axis=1)
        # exchange column k with the pivot column everywhere it is tracked
        a[rows, :, k], a[rows, :, p] = a[rows, :, p].copy(), a[rows, :, k].copy()
        colnorm[rows, k], colnorm[rows, p] = colnorm[rows, p].copy(), colnorm[rows, k].copy()
        perm[rows, k], perm[rows, p] = perm[rows, p].copy(), perm[rows, k].copy()
        if k:
            r[rows, :k, k], r[rows, :k, p] = r[rows, :k, p].copy(), r[rows, :k, k].copy()
        diag = np.maximum(np.sqrt(np.sum(np.abs(a[:, :, k]) ** 2, axis=1)), 1e-300)
        r[:, k, k] = diag
        qk = a[:, :, k] / diag[:, None]
        a[:, :, k] = qk
        if k + 1 < n:
            proj = np.einsum("bm,bmj->bj", qk.conj(), a[:, :, k + 1:])
            r[:, k, k + 1:] = proj
            a[:, :, k + 1:] -= qk[:, :, None] * proj[:, None, :]
            colnorm[:, k + 1:] = np.maximum(colnorm[:, k + 1:] - np.abs(proj) ** 2, 0.0)
    return perm, a, r


class Plan:
    """Per-channel plan: perm (C,N), qh (C,N,M), r (C,N,N), expansions, P."""

    def __init__(self, perm, qh, r, expansions, n_paths, augmented, noise_var):
        self.perm, self.qh, self.r = perm, qh, r
        self.expansions, self.n_paths = expansions, n_paths
        self.augmented, self.noise_var = augmented, noise_var

    def tile(self, reps):
        """One plan row per vector: repeat each channel's plan `reps` times."""
        return Plan(np.repeat(self.perm, reps, 0), np.repeat(self.qh, reps, 0),
                    np.repeat(self.r, reps, 0), self.expansions, self.n_paths,
                    self.augmented, self.noise_var)


def plan_channels(h, noise_var, n_paths, order):
    h = np.asarray(h, dtype=complex)
    if h.ndim == 2:
        h = h[None]
    _, m, n = h.shape
    aug = n > m
    e, p = allocate_expansions(n, order, n_paths, n_forced=max(0, n - m))
    a = h
    if aug:
        eye = np.broadcast_to(np.eye(n), (h.shape[0], n, n))
        a = np.concatenate([h, np.sqrt(noise_var) * eye], axis=1)
    perm, q, r = sorted_qr(a)
    qh = np.ascontiguousarray(q[:, :m, :].conj().transpose(0, 2, 1))
    return Plan(perm, qh, r, e, p, aug, noise_var)


# --------------------------------------------------------------------------
# detection
# --------------------------------------------------------------------------

def expand_tree(z, r, expansions, points):
    """Labels (B, P, N) in tree-position order; path index is mixed radix
    with the top layer most significant (detect.py:403-428)."""
    nb, n = z.shape
    lab = np.zeros((nb, 1, n), dtype=np.int64)
    interf = np.zeros((nb, 1, n), dtype=complex)
    for pos in range(n - 1, -1, -1):
        e = int(expansions[pos])
        centre = (z[:, None, pos] - interf[:, :, pos]) / r[:, None, pos, pos].real
        d2 = np.abs(centre[:, :, None] - points) ** 2
        kids = np.argsort(d2, axis=-1, kind="stable")[:, :, :e]
        lab = np.repeat(lab, e, axis=1)
        lab[:, :, pos] = kids.reshape(nb, -1)
        if pos:
            sym = points[kids]
            interf = (interf[:, :, None, :] + r[:, None, None, :, pos] * sym[..., None]
                      ).reshape(nb, -1, n)
    return lab


def to_stream_order(lab_pos, perm):
    nb, npth, _ = lab_pos.shape
    out = np.empty_like(lab_pos)
    out[np.arange(nb)[:, None, None], np.arange(npth)[None, :, None],
        perm[:, None, :]] = lab_pos
    return out


def true_metrics(h, y, labels, points):
    cand = points[labels]
    res = y[:, None, :] - np.einsum("bmn,bpn->bpm", h, cand)
    return np.sum(np.abs(res) ** 2, axis=2)


def select_best(labels, metrics):
    n = labels.shape[2]
    keys = tuple(labels[:, :, j] for j in range(n - 1, -1, -1)) + (metrics,)
    return np.lexsort(keys, axis=1)[:, 0]


def detect_batch(plan, h, y, points):
    """Per-vector plan rows -> (labels (B,P,N), metrics (B,P), best (B,))."""
    z = np.einsum("bnm,bm->bn", plan.qh, y)
    lab = to_stream_order(expand_tree(z, plan.r, plan.expansions, points), plan.perm)
    met = true_metrics(h, y, lab, points)
    return lab, met, select_best(lab, met)


def detect_rb(h_rb, y_rb, noise_var, n_paths, order, points):
    """Hard output for resource blocks.

    h_rb (C, M, N) one channel per RB, y_rb (C, V, M).  Returns
    hard labels (C, V, N) int64, winning metric (C, V), second-lowest
    metric (C, V) (inf when P == 1).
    """
    h_rb = np.asarray(h_rb, dtype=complex)
    y_rb = np.asarray(y_rb, dtype=complex)
    c, v, m = y_rb.shape
    n = h_rb.shape[2]
    plan = plan_channels(h_rb, noise_var, n_paths, order).tile(v)
    h = np.repeat(h_rb, v, axis=0)
    y = y_rb.reshape(c * v, m)
    lab, met, best = detect_batch(plan, h, y, points)
    rows = np.arange(c * v)
    hard = lab[rows, best]
    m1 = met[rows, best]
    if met.shape[1] > 1:
        m2 = np.partition(met, 1, axis=1)[:, 1]
    else:
        m2 = np.full(c * v, np.inf)
    return hard.reshape(c, v, n), m1.reshape(c, v), m2.reshape(c, v)


def _chunk_worker(args):
    h_rb, y_rb, noise_var, n_paths, order = args
    from paper_2409_14355_b200.core import constellation_for
    return detect_rb(h_rb, y_rb, noise_var, n_paths, order,
                     constellation_for(order).points)


def detect_rb_parallel(h_rb, y_rb, noise_var, n_paths, order, workers=None,
                       rbs_per_task=2):
    """`detect_rb` over whole-RB chunks in a process pool (cli.py:250-263
    pattern).  Worker count never changes the result."""
    import os
    from concurrent.futures import ProcessPoolExecutor

    workers = workers or len(os.sched_getaffinity(0))
    c = h_rb.shape[0]
    tasks = [(h_rb[i:i + rbs_per_task], y_rb[i:i + rbs_per_task], noise_var,
              n_paths, order) for i in range(0, c, rbs_per_task)]
    if workers == 1:
        parts = [_chunk_worker(t) for t in tasks]
    else:
        with ProcessPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(_chunk_worker, tasks))
    return tuple(np.concatenate([p[i] for p in parts]) for i in range(3))


# --------------------------------------------------------------------------
# list max-log LLRs
# --------------------------------------------------------------------------

def candidate_llrs(labels, metrics, noise_var, order, clip=20.0):
    """Max-log LLRs over candidate lists (detect.py:439-453): labels (B,P,N),
    metrics (B,P) -> (B,N,bps) float64.  Bits MSB first as bits_from_labels
    (core.py:209-213); clip = LLR_CLIP (core.py:21); noise_var scalar or (B,)."""
    bps = int(order).bit_length() - 1
    lab = np.asarray(labels, dtype=np.int64)
    bits = ((lab[..., None] >> np.arange(bps - 1, -1, -1)) & 1).astype(bool)
    mm = np.asarray(metrics, dtype=np.float64)[:, :, None, None]
    min1 = np.where(bits, mm, np.inf).min(axis=1)
    min0 = np.where(~bits, mm, np.inf).min(axis=1)
    nv = np.asarray(noise_var, dtype=np.float64)
    if nv.ndim:
        nv = nv.reshape((-1,) + (1,) * (min0.ndim - 1))
    with np.errstate(invalid="ignore"):
        llr = (min1 - min0) / nv
    return np.clip(llr, -clip, clip)


def _points(order):
    """Unit-energy Gray QAM points indexed by label (core.py:56-76)."""
    half = (int(order).bit_length() - 1) // 2
    n = 1 << half
    lv = np.empty(n)
    for pos in range(n):
        lv[pos ^ (pos >> 1)] = n - 1 - 2 * pos
    lab = np.arange(order)
    return (lv[lab >> half] + 1j * lv[lab & (n - 1)]) / np.sqrt(2.0 * (4 ** half - 1) / 3.0)


def linear_detect(h, y, noise_var, order, mode, clip=20.0):
    """Batched ZF / MMSE (detect.py:528-557) with the max-log demapper
    (core.py:191-206): h (B,M,N), y (B,M) -> (labels (B,N), llrs (B,N,bps),
    raw soft A^-1 H^H y (B,N)).  np.linalg.inv raises LinAlgError on a singular A, as there."""
    b, m, n = h.shape
    hh = h.conj().transpose(0, 2, 1)
    gram = hh @ h
    hy = np.einsum("bnm,bm->bn", hh, y)
    nv = np.broadcast_to(np.asarray(noise_var, dtype=float), (b,))
    if mode == "zf":
        a = gram
    elif mode == "mmse":
        a = gram + nv[:, None, None] * np.eye(n)
    else:
        raise ValueError(f"unknown linear mode {mode!r}")
    a_inv = np.linalg.inv(a)
    soft = np.einsum("bij,bj->bi", a_inv, hy)
    diag = np.real(np.einsum("bii->bi", a_inv))
    if mode == "zf":
        est, nv_eff = soft, nv[:, None] * diag
    else:
        beta = np.clip(1.0 - nv[:, None] * diag, 1e-12, None)
        est = soft / beta
        nv_eff = np.clip((1.0 - beta) / beta, 1e-15, None)
    pts = _points(order)
    bps = int(order).bit_length() - 1
    d = np.abs(est[..., None] - pts) ** 2                          # (B,N,Q)
    labels = np.argmin(d, axis=-1)
    bits = ((np.arange(order)[:, None] >> np.arange(bps - 1, -1, -1)) & 1).astype(bool)
    d1 = np.where(bits.T, d[..., None, :], np.inf).min(axis=-1)    # (B,N,bps)
    d0 = np.where(~bits.T, d[..., None, :], np.inf).min(axis=-1)
    llrs = (d1 - d0) / nv_eff[..., None]
    return labels, np.clip(llrs, -clip, clip), soft
