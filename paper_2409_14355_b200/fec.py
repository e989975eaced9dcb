"""LDPC stage after detection on the B200 kernels.

Mirrors the reference module `mpnlsim.fec` (`/root/reference/pkg/src/mpnlsim/fec.py`):
same names, argument order, return types and errors, backed by the C ABI of
`include/mpnl_b200.h` (`mpnl_ldpc_*`, ctypes) — no CPU fallback.

=======================  =====================================  ==============================
this module              reference                              kernels
=======================  =====================================  ==============================
expand_base_matrix       fec.py:44-57                           host (code construction)
LdpcCode                 fec.py:84-133                          host C++ graph + GF(2) encoder
ldpc_encode              fec.py:136-148                         ldpc_encode_kernel
ldpc_syndrome            fec.py:151-153                         ldpc_syndrome_kernel
ldpc_decode              fec.py:156-220 (normalized min-sum)    ldpc_decode_kernel (fp64,
                                                                bit-identical)
design_rate_match        fec.py:237-275                         host arithmetic
encode_rate_matched      fec.py:278-293                         ldpc_encode_kernel
decode_rate_matched      fec.py:296-326                         ldpc_decode_kernel (rate match
                                                                fused into the LLR load)
load_alist / save_alist  fec.py:333-368                         host file I/O
=======================  =====================================  ==============================

numpy inputs give numpy results (uint8 bits, bool flags) like the reference;
CUDA torch tensors stay on the device (uint8 bits, uint8 flags).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib

MIN_SUM_NORMALIZATION = 0.8125
DEFAULT_MAX_ITER = 10
SHORTENED_LLR = 1e7          # decoder LLR of shortened (known-zero) bits
LIFT = 54

# the shipped rate-1/2 mother code (fec.py:27-40): circulant shift per
# 54x54 block, -1 = all-zero block (code data, not logic)
BASE_MATRIX = (
    (-1, -1, -1, -1, -1, -1, 47, -1, -1, 16, -1, 45, 1, 0, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1),
    (-1, -1, -1, -1, -1, -1, 24, -1, 29, -1, 8, -1, -1, 0, 0, -1, -1, -1, -1, -1, -1, -1, -1, -1),
    (-1, -1, 20, 46, -1, -1, -1, 0, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1, -1, -1, -1, -1, -1),
    (-1, -1, -1, 0, 13, -1, -1, 53, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1, -1, -1, -1, -1),
    (-1, -1, -1, -1, 4, -1, -1, 9, -1, -1, 23, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1, -1, -1, -1),
    (14, -1, -1, -1, -1, 52, -1, -1, -1, -1, -1, 11, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1, -1, -1),
    (-1, -1, -1, -1, -1, 13, -1, -1, 37, -1, 24, -1, 0, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1, -1),
    (-1, -1, -1, -1, 7, 4, -1, -1, -1, 26, -1, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1, -1),
    (-1, 34, -1, -1, -1, -1, -1, -1, 39, -1, -1, 29, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1),
    (22, 43, 28, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1),
    (35, -1, -1, 26, -1, -1, -1, -1, -1, 50, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0),
    (-1, 48, 10, -1, -1, -1, 31, -1, -1, -1, -1, -1, 1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 0),
)


def expand_base_matrix(base=BASE_MATRIX, lift: int = LIFT) -> np.ndarray:
    """Dense binary H from a base matrix of circulant shifts (block (i, j)
    with shift s has ones at (r, (r - s) mod lift): the identity rolled by -s
    along the columns, as fec.py:53-55)."""
    base = np.asarray(base)
    mb, nb = base.shape
    h = np.zeros((mb * lift, nb * lift), dtype=np.uint8)
    r = np.arange(lift)
    for i, j in zip(*np.nonzero(base >= 0)):
        h[i * lift + r, j * lift + (r - int(base[i, j])) % lift] = 1
    return h


def _device():
    if not torch.cuda.is_available():
        raise _lib.MpnlError("LDPC kernels need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return torch.cuda.current_stream().cuda_stream


class LdpcCode:
    """Binary LDPC code defined by its parity-check matrix (fec.py:84-133).
    The decoder graph and the systematic encoder are built once by the C++
    host port (`mpnl_ldpc_build`) and kept on each device used."""

    def __init__(self, parity_check):
        h = np.asarray(parity_check, dtype=np.uint8)
        if h.ndim != 2 or h.shape[0] >= h.shape[1]:
            raise ValueError("parity-check matrix must be m x n with m < n")
        self.parity_check = np.ascontiguousarray(h)
        self._host = None
        self._dev = {}

    @property
    def n(self) -> int:
        return self.parity_check.shape[1]

    @property
    def k(self) -> int:
        return self.n - self.parity_check.shape[0]

    @property
    def rate(self) -> Fraction:
        return Fraction(self.k, self.n)

    def _tables(self):
        if self._host is None:
            lib = _lib.load()
            m, n = self.parity_check.shape
            dc, dv = np.zeros(1, np.int32), np.zeros(1, np.int32)
            _lib.check(lib.mpnl_ldpc_graph_dims(self.parity_check.ctypes.data, m, n,
                                                dc.ctypes.data, dv.ctypes.data), "LdpcCode")
            dc, dv = int(dc[0]), int(dv[0])
            cv = np.empty(m * dc, np.uint16)
            ve = np.empty(n * dv, np.uint16)
            enc = np.empty(m * ((self.k + 31) // 32), np.uint32)
            rc = lib.mpnl_ldpc_build(self.parity_check.ctypes.data, m, n, dc, dv,
                                     cv.ctypes.data, ve.ctypes.data, enc.ctypes.data)
            if rc == _lib.MPNL_EINVAL:
                raise ValueError(_lib.last_error())
            _lib.check(rc, "LdpcCode")
            self._host = (dc, dv, cv, ve, enc)
        return self._host

    def device_tables(self, dev):
        """(max_dc, max_dv, check_vars, var_edges, encoder) on `dev`."""
        t = self._dev.get(dev)
        if t is None:
            dc, dv, cv, ve, enc = self._tables()
            t = (dc, dv, torch.from_numpy(cv.view(np.int16)).to(dev),
                 torch.from_numpy(ve.view(np.int16)).to(dev),
                 torch.from_numpy(enc.view(np.int32)).to(dev))
            self._dev[dev] = t
        return t

    @property
    def _encoder(self) -> np.ndarray:
        """E (m, k) with parity = E @ info mod 2 (fec.py:104-105)."""
        enc = self._tables()[4].reshape(self.n - self.k, -1)
        bits = np.unpackbits(enc.view(np.uint8), axis=1, bitorder="little")
        return bits[:, :self.k].copy()


_DEFAULT_CODE = None


def default_code() -> LdpcCode:
    global _DEFAULT_CODE
    if _DEFAULT_CODE is None:
        _DEFAULT_CODE = LdpcCode(expand_base_matrix())
    return _DEFAULT_CODE


def _as_dev(a, dtype):
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(_device())
        return t.to(dtype).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a))).to(_device()).to(dtype), True


def _encode(code: LdpcCode, info, k_tb: int, n_tx: int):
    lib = _lib.load()
    t, was_np = _as_dev(info, torch.uint8)
    single = t.dim() == 1
    if single:
        t = t.unsqueeze(0)
    dev = t.device
    _, _, _, _, enc = code.device_tables(dev)
    out = torch.empty((t.shape[0], n_tx), dtype=torch.uint8, device=dev)
    m = code.n - code.k
    _lib.check(lib.mpnl_ldpc_encode(enc.data_ptr(), m, code.n, t.data_ptr(), t.shape[0], k_tb,
                                    n_tx, out.data_ptr(), _stream()), "ldpc_encode")
    if single:
        out = out[0]
    return out.cpu().numpy() if was_np else out


def ldpc_encode(code: LdpcCode, info) -> np.ndarray:
    """Systematic encoding of (k,) or (B, k) bits (fec.py:136-148)."""
    shape = info.shape if isinstance(info, torch.Tensor) else np.asarray(info).shape
    if shape[-1] != code.k:
        raise ValueError(f"info length {shape[-1]} != k = {code.k}")
    return _encode(code, info, code.k, code.n)


def ldpc_syndrome(code: LdpcCode, bits):
    """(B, m) parity checks of (B, n) bits (fec.py:151-153)."""
    lib = _lib.load()
    t, was_np = _as_dev(bits, torch.uint8)
    single = t.dim() == 1
    if single:
        t = t.unsqueeze(0)
    dc, _, cv, _, _ = code.device_tables(t.device)
    m = code.n - code.k
    out = torch.empty((t.shape[0], m), dtype=torch.uint8, device=t.device)
    _lib.check(lib.mpnl_ldpc_syndrome(cv.data_ptr(), m, dc, t.data_ptr(), t.shape[0], code.n,
                                      out.data_ptr(), _stream()), "ldpc_syndrome")
    if single:
        out = out[0]
    return out.cpu().numpy() if was_np else out


def _decode(code: LdpcCode, llrs, k_tb: int, n_tx: int, max_iter: int, alpha: float,
            return_iterations=False):
    lib = _lib.load()
    t, was_np = _as_dev(llrs, torch.float64)
    single = t.dim() == 1
    if single:
        t = t.unsqueeze(0)
    dev = t.device
    dc, dv, cv, ve, _ = code.device_tables(dev)
    b = t.shape[0]
    info = torch.empty((b, k_tb), dtype=torch.uint8, device=dev)
    conv = torch.empty(b, dtype=torch.uint8, device=dev)
    iters = torch.empty(b, dtype=torch.int32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    m = code.n - code.k
    _lib.check(lib.mpnl_ldpc_decode(cv.data_ptr(), ve.data_ptr(), m, code.n, dc, dv,
                                    t.data_ptr(), b, n_tx, k_tb, int(max_iter), float(alpha),
                                    float(SHORTENED_LLR), info.data_ptr(), conv.data_ptr(),
                                    iters.data_ptr(), bad.data_ptr(), _stream()), "ldpc_decode")
    if int(bad.item()):
        raise ValueError("LLRs must be finite")
    outs = [info, conv.bool() if not was_np else conv, iters]
    if was_np:
        outs = [info.cpu().numpy(), conv.cpu().numpy().astype(bool), iters.cpu().numpy()]
    if single:
        outs = [outs[0][0], bool(outs[1][0]), int(outs[2][0])]
    return tuple(outs) if return_iterations else tuple(outs[:2])


def ldpc_decode(code: LdpcCode, llrs, max_iter: int = DEFAULT_MAX_ITER,
                alpha: float = MIN_SUM_NORMALIZATION, *, return_iterations=False):
    """Normalized min-sum decoding (fec.py:156-220): llrs (n,) or (B, n),
    positive = bit 0.  Returns (info bits, converged) — bit-identical to the
    reference (fp64 kernel, same arithmetic order)."""
    shape = llrs.shape if isinstance(llrs, torch.Tensor) else np.asarray(llrs).shape
    if shape[-1] != code.n:
        raise ValueError(f"LLR length {shape[-1]} != codeword length {code.n}")
    return _decode(code, llrs, code.k, code.n, max_iter, alpha, return_iterations)


# ---------------------------------------------------------------------------
# rate matching (fec.py:223-326)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class RateMatch:
    target_rate: Fraction
    n_tx: int
    k_tb: int
    n_shortened: int
    n_punctured: int

    @property
    def method(self) -> str:
        parts = [p for p, on in (("shorten", self.n_shortened), ("puncture", self.n_punctured))
                 if on]
        return "+".join(parts) or "none"

    @property
    def effective_rate(self) -> float:
        return self.k_tb / self.n_tx


def design_rate_match(code: LdpcCode, target_rate, n_tx: int) -> RateMatch:
    """Shorten trailing info bits / puncture trailing parity bits so k_tb
    info bits ride on n_tx transmitted bits (fec.py:244-275, same errors)."""
    target = Fraction(target_rate)
    if not 0 < target < 1:
        raise ValueError("target rate must be in (0, 1)")
    k_tb = max(1, round(n_tx * target))
    p = n_tx - k_tb
    if k_tb > code.k:
        raise ValueError(f"needs {k_tb} info bits; mother code has {code.k}")
    if p > code.n - code.k:
        raise ValueError(f"needs {p} parity bits; mother code has {code.n - code.k}")
    if p < 1:
        raise ValueError("allocation leaves no parity bits")
    rm = RateMatch(target_rate=target, n_tx=n_tx, k_tb=k_tb, n_shortened=code.k - k_tb,
                   n_punctured=(code.n - code.k) - p)
    if abs(rm.effective_rate - float(target)) > 0.02 * float(target):
        raise ValueError(f"effective rate {rm.effective_rate:.4f} misses target "
                         f"{float(target):.4f} by more than 2%")
    return rm


def encode_rate_matched(code: LdpcCode, rm: RateMatch, info):
    """k_tb info bits -> n_tx transmitted bits (fec.py:278-293)."""
    shape = info.shape if isinstance(info, torch.Tensor) else np.asarray(info).shape
    if shape[-1] != rm.k_tb:
        raise ValueError(f"info length {shape[-1]} != k_tb = {rm.k_tb}")
    return _encode(code, info, rm.k_tb, rm.n_tx)


def decode_rate_matched(code: LdpcCode, rm: RateMatch, llrs_tx,
                        max_iter: int = DEFAULT_MAX_ITER, *, return_iterations=False):
    """Transmitted-bit LLRs -> k_tb info bits (fec.py:296-326)."""
    shape = llrs_tx.shape if isinstance(llrs_tx, torch.Tensor) else np.asarray(llrs_tx).shape
    if shape[-1] != rm.n_tx:
        raise ValueError(f"LLR length {shape[-1]} != n_tx = {rm.n_tx}")
    return _decode(code, llrs_tx, rm.k_tb, rm.n_tx, max_iter, MIN_SUM_NORMALIZATION,
                   return_iterations)


# ---------------------------------------------------------------------------
# alist I/O (fec.py:333-368): plain text, host only
# ---------------------------------------------------------------------------

def load_alist(path) -> LdpcCode:
    with open(path) as f:
        tok = [int(t) for t in f.read().split()]
    n, m, max_dv = tok[0], tok[1], tok[2]
    pos = 4 + n + m                                   # skip the degree lists
    h = np.zeros((m, n), dtype=np.uint8)
    for col in range(n):
        rows = [r for r in tok[pos:pos + max_dv] if r > 0]
        h[np.asarray(rows, dtype=np.int64) - 1, col] = 1
        pos += max_dv
    return LdpcCode(h)


def save_alist(code: LdpcCode, path) -> None:
    h = code.parity_check
    m, n = h.shape
    dv, dc = h.sum(axis=0), h.sum(axis=1)
    out = [f"{n} {m}", f"{dv.max()} {dc.max()}", " ".join(map(str, dv)),
           " ".join(map(str, dc))]
    for col in range(n):
        rows = list(np.nonzero(h[:, col])[0] + 1)
        out.append(" ".join(map(str, rows + [0] * (int(dv.max()) - len(rows)))))
    for row in range(m):
        cols = list(np.nonzero(h[row])[0] + 1)
        out.append(" ".join(map(str, cols + [0] * (int(dc.max()) - len(cols)))))
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
