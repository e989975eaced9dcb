"""Slot I/O around the detector on the B200 kernels.

Mirrors the grid-level pieces of the reference link simulator
(`/root/reference/pkg/src/mpnlsim/linksim.py`) that sit either side of the
detection path, backed by the C ABI (`mpnl_slot_receive`,
`mpnl_dmrs_ls_estimate`, `mpnl_select_symbols`) — no CPU fallback:

=======================  =============================================  =========================
this module              reference                                      kernel
=======================  =============================================  =========================
dmrs_pattern             linksim.py:103-114 (_dmrs_pattern)             host (port table)
receive_grid             linksim.py:207 (einsum "tfmn,btfn->btfm" + n)  slot_receive_kernel (bit-exact)
estimate_channel_ls      linksim.py:117-137                             dmrs_ls_kernel (bit-exact)
data_re_batch            linksim.py:211-216 (h[data_syms], y[:, ds])    select_rows_kernel
simulate_frames          linksim.py:159-232 (one channel, many frames)  all of the above + LDPC
                                                                        encode / decode + MPNL
                                                                        soft output / linear
LinkConfig               linksim.py:31-65 (fields the frames use)       host
PerResult, measure_per   linksim.py:83-96, 241-271 (PER + early stop)   simulate_frames
=======================  =============================================  =========================

`simulate_frames` keeps the reference's per-frame random streams (info bits and
noise drawn on the host from SeedSequence((seed, chan_idx, frame)), exactly as
linksim.py:97-99, 186-190) and runs everything else on the GPU.  Encoding,
modulation, the receive grid, the LS estimate, the gathers and the decoder are
bit-identical to the reference; the MPNL list metrics are the plan's fp64 PED
(the reference's einsum residual differs by rounding, ~1e-15 relative), so the
LLRs agree to rounding and the decode outcomes match (tested on reference
goldens).

numpy inputs give numpy outputs; CUDA torch tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib
from . import detect as _det
from . import fec as _fec

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


# ---------------------------------------------------------------------------
# frame simulation (linksim.py:159-232)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Numerology:
    """The slot fields simulate_frames uses (core.py:133-152 defaults)."""
    symbols_per_slot: int = 14
    data_symbols: int = 12
    dmrs_symbols: int = 2
    sc_per_rb: int = 12


@dataclass(frozen=True)
class LinkConfig:
    """The LinkConfig fields simulate_frames uses (linksim.py:31-65).  `mcs`
    needs `.constellation` and `.code_rate` (the reference's McsEntry works,
    and so does the reference's own LinkConfig in place of this one)."""
    n_streams: int
    m_antennas: int
    mcs: object
    rb_per_vehicle: int
    detector: str = "mpnl"
    n_paths: int = 32
    csi: str = "genie"
    numerology: Numerology = Numerology()
    seed: int = 0

    def __post_init__(self):
        if not 1 <= self.n_streams <= 12:
            raise ValueError("n_streams must be in [1, 12]")
        if not 1 <= self.m_antennas <= 32:
            raise ValueError("m_antennas must be in [1, 32]")
        if self.detector not in ("zf", "mmse", "mpnl"):
            raise ValueError(f"unknown detector {self.detector!r}")
        if self.csi not in ("genie", "ls_dmrs"):
            raise ValueError("csi must be 'genie' or 'ls_dmrs'")

    @property
    def n_subcarriers(self) -> int:
        return self.rb_per_vehicle * self.numerology.sc_per_rb

    @property
    def bits_per_block(self) -> int:
        return (self.n_subcarriers * self.numerology.data_symbols
                * self.mcs.constellation.bits_per_symbol)


def _frame_rng(seed: int, chan_idx: int, frame_idx: int):
    """The reference's per-frame stream (linksim.py:97-99)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=(seed, chan_idx, frame_idx)))


def _detect_llrs(cfg, c, h_flat, y_rc, noise_var, plan=None, precision="fp64"):
    """LLRs (n_re, V, N, bps) of y_rc (n_re, V, M) against the n_re per-RE
    channels h_flat (linksim.py:140-156, the V frames batched per channel)."""
    if cfg.detector in ("zf", "mmse"):
        n_re, v, m = y_rc.shape
        hb = h_flat.unsqueeze(1).expand(n_re, v, m, h_flat.shape[2]).reshape(n_re * v, m, -1)
        _, llr = _det.linear_detect_batch(hb.contiguous(), y_rc.reshape(n_re * v, m).contiguous(),
                                          noise_var, c, cfg.detector)
        return llr.reshape(n_re, v, h_flat.shape[2], c.bits_per_symbol)
    if plan is None:
        plan = _det.mpnl_plan_batch(h_flat, noise_var, cfg.n_paths, c)
    return _det.mpnl_detect_llrs(plan, h_flat, y_rc, c, noise_var, precision=precision)


def simulate_frames(cfg, grid, noise_var: float, chan_idx: int, frame_indices, *,
                    soft_precision: str = "fp64") -> np.ndarray:
    """Frames on one channel realisation (linksim.py:159-232): boolean
    (n_frames, n_streams), True = transport block decoded correctly.
    `grid` has `.h` (symbols, subcarriers, >= M, >= N) (the reference's
    ChannelGrid) or is that array.  `soft_precision` selects the MPNL soft
    output: "fp64" (the reference's arithmetic; outcomes identical to the
    reference's) or "fp32" (`detect.mpnl_detect_llrs(precision="fp32")`: LLRs
    within ~1e-6 of the metrics / noise_var of the reference's)."""
    num = cfg.numerology
    n_sc = cfg.n_subcarriers
    n, m = cfg.n_streams, cfg.m_antennas
    h_all = np.asarray(getattr(grid, "h", grid))
    if h_all.shape[2] < m or h_all.shape[3] < n or h_all.shape[1] < n_sc:
        raise ValueError("channel grid is smaller than the configuration")
    c = cfg.mcs.constellation
    bps = c.bits_per_symbol
    code = _fec.default_code()
    rm = _fec.design_rate_match(code, cfg.mcs.code_rate, cfg.bits_per_block)
    dmrs_syms, ports = dmrs_pattern(num, n, n_sc)
    data_syms = [s for s in range(num.symbols_per_slot) if s not in dmrs_syms]
    n_re = len(data_syms) * n_sc
    frames = list(frame_indices)
    f = len(frames)
    s_all = num.symbols_per_slot
    # per-frame payloads and noise from the reference's streams (host RNG)
    info = np.empty((f, n, rm.k_tb), dtype=np.uint8)
    noise = np.empty((f, s_all, n_sc, m), dtype=complex)
    for i, fi in enumerate(frames):
        rng = _frame_rng(cfg.seed, chan_idx, fi)
        info[i] = rng.integers(0, 2, (n, rm.k_tb))
        noise[i] = np.sqrt(noise_var / 2) * (rng.standard_normal((s_all, n_sc, m))
                                             + 1j * rng.standard_normal((s_all, n_sc, m)))
    dev = _dev()
    h = torch.from_numpy(np.array(h_all[:, :n_sc, :m, :n], dtype=complex)).to(dev)
    info_d = torch.from_numpy(info.reshape(f * n, rm.k_tb)).to(dev)
    noise_d = torch.from_numpy(noise).to(dev)
    # encode + modulate (MSB-first bit groups -> Gray labels -> points, core.py:180-188)
    tx = _fec.encode_rate_matched(code, rm, info_d)                       # (f n, n_tx) u8
    w = (1 << torch.arange(bps - 1, -1, -1, device=dev, dtype=torch.int64))
    lab = (tx.reshape(f, n, len(data_syms), n_sc, bps).to(torch.int64) * w).sum(-1)
    pts = torch.from_numpy(np.asarray(c.points, dtype=complex)).to(dev)
    x = torch.zeros((f, s_all, n_sc, n), dtype=torch.complex128, device=dev)
    x[:, data_syms] = pts[lab].permute(0, 2, 3, 1)                        # (f, ds, sc, n)
    pilots = []
    for v, (sym, sc_idx) in enumerate(ports):
        x[:, sym, torch.from_numpy(sc_idx).to(dev), v] = 1.0
        pilots.append(np.ones(sc_idx.size, dtype=complex))
    pilots = np.array(pilots)
    y = receive_grid(h, x, noise_d)                                       # (f, s, sc, m)
    if cfg.csi == "genie":
        h_flat, y_flat = data_re_batch(h, y, data_syms)                  # (n_re,m,n), (f,n_re,m)
        llrs = _detect_llrs(cfg, c, h_flat, y_flat.permute(1, 0, 2).contiguous(), noise_var,
                            precision=soft_precision)
        llrs = llrs.permute(1, 0, 2, 3)                                   # (f, n_re, n, bps)
    else:
        llrs = torch.empty((f, n_re, n, bps), dtype=torch.float64, device=dev)
        pil = torch.from_numpy(pilots).to(dev)
        for i in range(f):
            h_est = estimate_channel_ls(y[i], pil, cfg)
            h_flat, y_flat = data_re_batch(h_est, y[i:i + 1], data_syms)
            llrs[i] = _detect_llrs(cfg, c, h_flat, y_flat.permute(1, 0, 2).contiguous(),
                                   noise_var, precision=soft_precision)[:, 0]
    # per-vehicle LLR concatenation in RE order -> rate-matched LDPC decoding
    llrs_v = llrs.permute(0, 2, 1, 3).reshape(f * n, n_re * bps).contiguous()
    dec, conv = _fec.decode_rate_matched(code, rm, llrs_v)
    ok = conv.bool() & ~torch.any(dec != info_d, dim=1)
    return ok.reshape(f, n).cpu().numpy()


@dataclass(frozen=True)
class PerResult:
    """Transport-block error count (linksim.py:83-96)."""
    frames: int
    errors: int

    @property
    def per(self) -> float:
        return self.errors / self.frames

    @property
    def ci95_halfwidth(self) -> float:
        p = self.per
        return 1.96 * np.sqrt(max(p * (1 - p), 1e-12) / self.frames)


def measure_per(cfg, channels, noise_vars, frames_per_channel: int = 200,
                stop_threshold: float | None = None, min_frames: int = 400) -> PerResult:
    """Average transport-block error rate over a channel set (linksim.py:241-271):
    the reference's loop — 25-frame batches per channel, optional early stop
    once the 95% interval excludes `stop_threshold` — over the GPU
    `simulate_frames`; same frame indices, so the same outcomes."""
    if frames_per_channel < 1:
        raise ValueError("need at least one frame per channel")
    frames = errors = 0
    batch = 25
    for chan_idx, (grid, nv) in enumerate(zip(channels, noise_vars)):
        done = 0
        while done < frames_per_channel:
            take = min(batch, frames_per_channel - done)
            ok = simulate_frames(cfg, grid, nv, chan_idx, range(done, done + take))
            errors += int((~ok).sum())
            frames += ok.size
            done += take
            if stop_threshold is not None and frames >= min_frames:
                res = PerResult(frames=frames, errors=errors)
                if (res.per - res.ci95_halfwidth > stop_threshold
                        or res.per + res.ci95_halfwidth < stop_threshold):
                    return res
    return PerResult(frames=frames, errors=errors)
