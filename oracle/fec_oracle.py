"""CPU oracle for the LDPC stage after detection — TEST INFRASTRUCTURE ONLY
(SURVEY §8f row 3).

Only `tests/` (and the bench's CPU legs) may import this module, as a checker;
the product path (`paper_2409_14355_b200.fec`) runs the CUDA library.

A numpy restatement of the reference's `mpnlsim.fec`
(`/root/reference/pkg/src/mpnlsim/fec.py`), written per codeword so the
arithmetic order is explicit (the GPU kernel must reproduce it bit for bit):

* ``expand_base_matrix``  <- fec.py:44-57   (circulant right shifts)
* ``parity_solver``       <- fec.py:60-81   (GF(2) elimination on the parity columns)
* ``graph``               <- fec.py:107-133 (check-major edges, var-major edge lists)
* ``encode``              <- fec.py:136-148 (systematic: parity = E @ info mod 2)
* ``decode``              <- fec.py:156-220 (flooding normalized min-sum):
    m_vc[e]  = total[v(e)] - m_cv[e]          (first iteration: the channel LLR)
    per check: parity of the signs, first argmin of |m_vc|, second minimum;
    m_cv[e]  = +-(alpha * (e == argmin ? min2 : min1)), sign = parity xor own;
    total[v] = llr[v] + sum_e m_cv[e] over the variable's padded edge row,
               summed in numpy's order for an add-reduce over a contiguous
               row of length max_dv (sequential below 8 terms, 8-way pairwise
               blocks from 8 on: ``np_sum_order``);
    hard = total < 0; converged when the syndrome of the hard decision is 0
    (checked first on the channel LLRs, then after every iteration).
* ``decode_rate_matched`` <- fec.py:307-326 (shortened bits = SHORTENED_LLR,
                              punctured = 0), ``design_rate_match`` <- fec.py:244-275.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

ALPHA = 0.8125
SHORTENED_LLR = 1e7
LIFT = 54


def expand_base_matrix(base, lift=LIFT):
    base = np.asarray(base)
    mb, nb = base.shape
    h = np.zeros((mb * lift, nb * lift), dtype=np.uint8)
    for i in range(mb):
        for j in range(nb):
            s = int(base[i, j])
            if s >= 0:
                rows = np.arange(lift)
                h[i * lift + rows, j * lift + (rows - s) % lift] = 1
    return h


def parity_solver(h):
    """E (m, k) with parity = E @ info (mod 2)."""
    m, n = h.shape
    k = n - m
    w = h.astype(np.uint8).copy()
    for r, c in enumerate(range(k, n)):
        piv = np.nonzero(w[r:, c])[0]
        if piv.size == 0:
            raise ValueError("parity submatrix is singular")
        p = piv[0] + r
        if p != r:
            w[[r, p]] = w[[p, r]]
        mask = w[:, c].astype(bool)
        mask[r] = False
        w[mask] ^= w[r]
    return w[:, :k].copy()


def graph(h):
    """check_vars (m, dc) var index or -1, var_edges (n, dv) flat edge index
    (check * dc + slot) or -1; edges enumerated row-major as np.nonzero."""
    m, n = h.shape
    rows, cols = np.nonzero(h)
    dc = int(np.bincount(rows, minlength=m).max())
    dv = int(np.bincount(cols, minlength=n).max())
    cv = np.full((m, dc), -1, np.int64)
    ve = np.full((n, dv), -1, np.int64)
    sc = np.zeros(m, np.int64)
    sv = np.zeros(n, np.int64)
    for r, c in zip(rows, cols):
        cv[r, sc[r]] = c
        ve[c, sv[c]] = r * dc + sc[r]
        sc[r] += 1
        sv[c] += 1
    return cv, ve


def encode(h, info):
    e = parity_solver(h)
    info = np.atleast_2d(np.asarray(info, np.uint8))
    par = (info.astype(np.int64) @ e.T.astype(np.int64)) % 2
    return np.concatenate([info, par.astype(np.uint8)], axis=1)


def syndrome(h, bits):
    return (np.asarray(bits, np.int64) @ h.T.astype(np.int64)) % 2


def np_sum_order(vals):
    """numpy's add.reduce of one contiguous row (float64): 0 + pairwise."""
    d = len(vals)
    if d < 8:
        s = 0.0
        for x in vals:
            s = s + x
        return s
    r = list(vals[:8])
    i = 8
    while i + 8 <= d:
        for j in range(8):
            r[j] = r[j] + vals[i + j]
        i += 8
    s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < d:
        s = s + vals[i]
        i += 1
    return 0.0 + s


def decode_one(cv, ve, llr, max_iter=10, alpha=ALPHA):
    """One codeword -> (hard decision (n,) uint8, converged, iterations)."""
    m, dc = cv.shape
    n, dv = ve.shape
    llr = np.asarray(llr, np.float64)
    valid = cv >= 0
    mcv = np.zeros(m * dc)
    total = llr.copy()

    def synd_zero(bits):
        return not np.any(np.bitwise_xor.reduce(np.where(valid, bits[np.maximum(cv, 0)], 0),
                                                axis=1))

    it = 0
    while True:
        bits = (total < 0).astype(np.uint8)
        if synd_zero(bits):
            return bits, True, it
        if it == max_iter:
            return bits, False, it
        for r in range(m):
            mvc = [total[cv[r, s]] - mcv[r * dc + s] if valid[r, s] else np.inf
                   for s in range(dc)]
            neg = [x < 0 for x in mvc]
            par = False
            for x in neg:
                par ^= x
            mag = [abs(x) for x in mvc]
            amin = int(np.argmin(mag))
            min1 = mag[amin]
            min2 = min([mag[s] for s in range(dc) if s != amin], default=np.inf)
            a1, a2 = alpha * min1, alpha * min2
            for s in range(dc):
                if valid[r, s]:
                    ext = a2 if s == amin else a1
                    mcv[r * dc + s] = -ext if (par ^ neg[s]) else ext
        for v in range(n):
            vals = [mcv[e] if e >= 0 else 0.0 for e in ve[v]]
            total[v] = llr[v] + np_sum_order(vals)
        it += 1


def decode(h, llrs, max_iter=10, alpha=ALPHA):
    """(info bits (B, k), converged (B,)) as fec.ldpc_decode on a batch:
    `decode_one` vectorised over the words (same elementwise arithmetic; the
    slot loops keep the per-element order)."""
    cv, ve = graph(h)
    llrs = np.atleast_2d(np.asarray(llrs, np.float64))
    if not np.all(np.isfinite(llrs)):
        raise ValueError("LLRs must be finite")
    b, n = llrs.shape
    m, dc = cv.shape
    dv = ve.shape[1]
    k = n - m
    valid = cv >= 0
    cvi = np.maximum(cv, 0)
    mcv = np.zeros((b, m, dc))
    total = llrs.copy()
    out = np.zeros((b, n), np.uint8)
    done = np.zeros(b, bool)
    for it in range(max_iter + 1):
        bits = (total < 0).astype(np.uint8)
        synd = np.bitwise_xor.reduce(np.where(valid, bits[:, cvi], 0), axis=2).any(axis=1)
        newly = ~done & ~synd
        out[newly] = bits[newly]
        done |= newly
        if it == max_iter or done.all():
            break
        mvc = np.where(valid, total[:, cvi] - mcv, np.inf)          # (B, m, dc)
        neg = mvc < 0
        par = np.logical_xor.reduce(neg, axis=2)
        mag = np.abs(mvc)
        amin = np.argmin(mag, axis=2)
        min1 = np.take_along_axis(mag, amin[..., None], axis=2)[..., 0]
        rest = mag.copy()
        np.put_along_axis(rest, amin[..., None], np.inf, axis=2)
        min2 = rest.min(axis=2)
        a1, a2 = alpha * min1, alpha * min2
        ext = np.where(np.arange(dc) == amin[..., None], a2[..., None], a1[..., None])
        mcv = np.where(valid, np.where(par[..., None] ^ neg, -ext, ext), 0.0)
        flat = np.concatenate([mcv.reshape(b, -1), np.zeros((b, 1))], axis=1)
        vals = flat[:, np.where(ve >= 0, ve, m * dc)]                # (B, n, dv)
        total = llrs + np_sum_order([vals[:, :, j] for j in range(dv)])
    out[~done] = (total[~done] < 0)
    return out[:, :k], done


def design_rate_match(n, k, target_rate, n_tx):
    """(k_tb, n_shortened, n_punctured) or ValueError (fec.py:244-275)."""
    target = Fraction(target_rate)
    if not 0 < target < 1:
        raise ValueError("target rate must be in (0, 1)")
    k_tb = max(1, round(n_tx * target))
    p = n_tx - k_tb
    if k_tb > k or p > n - k or p < 1:
        raise ValueError("infeasible rate match")
    if abs(k_tb / n_tx - float(target)) > 0.02 * float(target):
        raise ValueError("effective rate misses the target by more than 2%")
    return k_tb, k - k_tb, (n - k) - p


def full_llrs(n, k, k_tb, llrs_tx):
    """Mother-code LLRs of a rate-matched word (fec.py:316-321)."""
    llrs_tx = np.atleast_2d(np.asarray(llrs_tx, np.float64))
    p = llrs_tx.shape[1] - k_tb
    full = np.zeros((llrs_tx.shape[0], n))
    full[:, :k_tb] = llrs_tx[:, :k_tb]
    full[:, k_tb:k] = SHORTENED_LLR
    full[:, k:k + p] = llrs_tx[:, k_tb:]
    return full
