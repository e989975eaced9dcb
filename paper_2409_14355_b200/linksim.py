"""Slot I/O around the detector on the B200 kernels.

Mirrors the grid-level pieces of the reference link simulator
(`/root/reference/pkg/src/mpnlsim/linksim.py`) that sit either side of the
detection path, backed by the C ABI (`mpnl_slot_receive`,
`mpnl_dmrs_ls_estimate`, `mpnl_select_symbols`) — no CPU fallback:

=======================  =============================================  =========================
this module              reference                                      kernel
=======================  =============================================  =========================
dmrs_pattern             linksim.py:103-114 (_dmrs_pattern)             host (port table)
receive_grid             linksim.py:207 (einsum "tfmn,btfn->btfm" + n)  slot_receive_kernel
estimate_channel_ls      linksim.py:117-137                             dmrs_ls_kernel (bit-exact)
data_re_batch            linksim.py:211-216 (h[data_syms], y[:, ds])    select_rows_kernel
=======================  =============================================  =========================

numpy inputs give numpy outputs; CUDA torch tensors stay on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DMRS_COMBS = 6   # disjoint subcarrier combs; 6 combs x 2 symbols = 12 ports


def dmrs_pattern(num, n_streams: int, n_sc: int):
    """(DMRS symbols, [(symbol, pilot subcarriers)] per stream) — the
    reference's comb assignment (linksim.py:103-114), same ValueError."""
    if n_streams > DMRS_COMBS * num.dmrs_symbols:
        raise ValueError("too many streams for the pilot book")
    dmrs_syms = (3, 12)[:num.dmrs_symbols]
    ports = []
    for v in range(n_streams):
        ports.append((dmrs_syms[v // DMRS_COMBS], np.arange(v % DMRS_COMBS, n_sc, DMRS_COMBS)))
    return dmrs_syms, ports


def data_symbols(num, n_streams: int, n_sc: int):
    dmrs = dmrs_pattern(num, n_streams, n_sc)[0]
    return [s for s in range(num.symbols_per_slot) if s not in dmrs]


def _dev():
    if not torch.cuda.is_available():
        raise _lib.MpnlError("slot kernels need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _c128(a):
    """-> (contiguous complex128 CUDA tensor, was_numpy)."""
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(_dev())
        return t.to(torch.complex128).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128))).to(_dev()), True


def _stream():
    return torch.cuda.current_stream().cuda_stream


def receive_grid(h, x, noise=None):
    """y (F, S, SC, M) = einsum("tfmn,btfn->btfm", h, x) + noise: the slot's
    received grid (linksim.py:207).  h (S, SC, M, N), x (F, S, SC, N),
    noise (F, S, SC, M) or None."""
    lib = _lib.load()
    ht, was_np = _c128(h)
    xt, _ = _c128(x)
    if ht.dim() != 4 or xt.dim() != 4 or xt.shape[1:3] != ht.shape[:2] or xt.shape[3] != ht.shape[3]:
        raise ValueError("h must be (S, SC, M, N) and x (F, S, SC, N)")
    s, sc, m, n = ht.shape
    f = xt.shape[0]
    nt = None
    if noise is not None:
        nt, _ = _c128(noise)
        if tuple(nt.shape) != (f, s, sc, m):
            raise ValueError("noise must be (F, S, SC, M)")
    y = torch.empty((f, s, sc, m), dtype=torch.complex128, device=ht.device)
    _lib.check(lib.mpnl_slot_receive(ht.data_ptr(), xt.data_ptr(),
                                     nt.data_ptr() if nt is not None else None, f, s, sc, m, n,
                                     y.data_ptr(), _stream()), "receive_grid")
    return y.cpu().numpy() if was_np else y


def estimate_channel_ls(grid_obs, pilots, cfg):
    """LS channel estimate from DMRS observations (linksim.py:117-137):
    grid_obs (symbols, subcarriers, M), pilots (n_streams, n_pilot_sc) ->
    (symbols, subcarriers, M, N) by nearest-pilot interpolation, constant
    across symbols.  `cfg` needs numerology, n_subcarriers, m_antennas and
    n_streams (the reference's LinkConfig fields).  Bit-identical."""
    lib = _lib.load()
    num = cfg.numerology
    n_sc, m, n = cfg.n_subcarriers, cfg.m_antennas, cfg.n_streams
    _, ports = dmrs_pattern(num, n, n_sc)
    ot, was_np = _c128(grid_obs)
    pt, _ = _c128(pilots)
    s = num.symbols_per_slot
    if tuple(ot.shape) != (s, n_sc, m):
        raise ValueError("grid_obs must be (symbols, subcarriers, M)")
    n_pilot = len(ports[0][1])
    if tuple(pt.shape) != (n, n_pilot):
        raise ValueError("pilots must be (n_streams, n_pilot_sc)")
    dev = ot.device
    sym = torch.tensor([p[0] for p in ports], dtype=torch.int32, device=dev)
    scs = torch.from_numpy(np.stack([p[1] for p in ports]).astype(np.int32)).to(dev)
    h_est = torch.empty((s, n_sc, m, n), dtype=torch.complex128, device=dev)
    _lib.check(lib.mpnl_dmrs_ls_estimate(ot.data_ptr(), pt.data_ptr(), sym.data_ptr(),
                                         scs.data_ptr(), s, n_sc, m, n, n_pilot,
                                         h_est.data_ptr(), _stream()), "estimate_channel_ls")
    return h_est.cpu().numpy() if was_np else h_est


def _select(src, rows, batch_dims):
    lib = _lib.load()
    t, was_np = _c128(src)
    s = t.shape[batch_dims]
    lead = t.shape[:batch_dims]
    rest = t.shape[batch_dims + 1:]
    batch = int(np.prod(lead)) if lead else 1
    row_bytes = int(np.prod(rest)) * 16
    r = torch.tensor(list(rows), dtype=torch.int32, device=t.device)
    out = torch.empty(tuple(lead) + (len(rows),) + tuple(rest), dtype=torch.complex128,
                      device=t.device)
    _lib.check(lib.mpnl_select_symbols(t.data_ptr(), batch, s, row_bytes, r.data_ptr(),
                                       len(rows), out.data_ptr(), _stream()), "data_re_batch")
    return out, was_np


def data_re_batch(h_grid, y_grid, data_syms):
    """Per-RE detector batch of the data symbols (linksim.py:211-216):
    h (S, SC, M, N) -> h_flat (n_re, M, N); y (F, S, SC, M) -> y_flat (F, n_re, M),
    n_re = len(data_syms) * SC, RE order = (symbol, subcarrier)."""
    h_sel, was_np = _select(h_grid, data_syms, 0)
    y_sel, _ = _select(y_grid, data_syms, 1)
    s_, sc, m, n = h_sel.shape
    h_flat = h_sel.reshape(s_ * sc, m, n)
    y_flat = y_sel.reshape(y_sel.shape[0], s_ * sc, m)
    if was_np:
        return h_flat.cpu().numpy(), y_flat.cpu().numpy()
    return h_flat, y_flat
