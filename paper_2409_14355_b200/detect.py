"""Drop-in MPNL detector API on the B200 kernels.

Mirrors the MPNL part of the reference module `mpnlsim.detect`
(`/root/reference/pkg/src/mpnlsim/detect.py`): same names, argument order,
return types and error behaviour, backed by the C ABI of
`include/mpnl_b200.h` (ctypes) — there is no CPU fallback.

=========================  ==========================================  =====================
this module                reference                                   kernels
=========================  ==========================================  =====================
allocate_expansions        detect.py:221-280                           host C++ port
mpnl_plan_batch            detect.py:361-388 (+ _sorted_qr_batch)      K1 plan (fp64 QR)
mpnl_detect_batch          detect.py:473-488 (full candidate list)     K5 exact (fp64)
_candidate_llrs_batch      detect.py:439-453 (list max-log LLRs)       K6 candidate LLR
mpnl_detect_llrs           linksim.py:151-155 (the "mpnl" branch)      K5 + K6 on device
mpnl_detect_hard           hard composition cli.py:236-239,            K3 fp32 traversal +
                           test_acceptance.py:114-117                  K5 fix-up of flags
mpnl_hard_output           plan + hard composition from HOST arrays    K1-K5, pipelined
                           (the cli._bench_chunk call, cli.py:236-239) host<->device copies
mpnl_hard_output_device    the same from DEVICE arrays, channel        K1-K5 on forked
                           groups overlapped                           streams
mpnl_preprocess            detect.py:391-400                           K1
mpnl_detect                detect.py:491-506                           K5
detect("mpnl", ...)        detect.py:563-576                           K1 + K5
=========================  ==========================================  =====================

Inputs may be numpy arrays (results come back as numpy, int64 labels /
float64 metrics, like the reference) or CUDA torch tensors (results stay on
the device: uint8 labels, float32/float64 metrics).  Extension over the
reference: `y` may be (B, V, M) against a plan of B channels (V vectors per
channel, e.g. the 168 REs of a resource block), equal to tiling the plan.
"""

from __future__ import annotations

import hashlib
import warnings
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .core import LLR_CLIP, Constellation, bits_from_labels

__all__ = [
    "allocate_expansions", "BatchPathPlan", "PathPlan", "mpnl_plan_batch",
    "mpnl_preprocess", "mpnl_detect_batch", "mpnl_detect_hard", "mpnl_hard_output",
    "mpnl_hard_output_device", "mpnl_detect",
    "detect", "DetectorInput", "CandidateList", "DetectionOutput",
    "llr_from_candidates", "mpnl_detect_llrs", "DETECTOR_NAMES", "SingularChannelError",
    "linear_detect_batch", "zf_detect", "mmse_detect",
]


class SingularChannelError(ValueError):
    pass


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def _stream():
    return torch.cuda.current_stream().cuda_stream


def _device():
    if not torch.cuda.is_available():
        raise _lib.MpnlError("MPNL kernels need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev_complex(a, name):
    """-> (contiguous CUDA complex tensor, is_f64, was_numpy)."""
    if isinstance(a, torch.Tensor):
        t = a
        if not t.is_cuda:
            t = t.to(_device())
        if t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        return t.contiguous(), t.dtype == torch.complex128, False
    arr = np.asarray(a)
    if arr.dtype != np.complex64:
        arr = arr.astype(np.complex128)
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(_device())
    return t, arr.dtype == np.complex128, True


def _ptr(t):
    return t.data_ptr() if t is not None else None


# ---------------------------------------------------------------------------
# planning
# ---------------------------------------------------------------------------

def allocate_expansions(n_layers: int, q: int, n_paths: int,
                        n_forced: int = 0) -> tuple[np.ndarray, int]:
    """Per-layer expansion counts (tree position order) and realized paths.

    Same rule and errors as detect.py:221-280 (computed by the C++ port)."""
    lib = _lib.load()
    out = np.zeros(max(int(n_layers), 1), dtype=np.int64)
    realized = np.zeros(1, dtype=np.int64)
    warned = np.zeros(1, dtype=np.int32)
    rc = lib.mpnl_alloc_expansions(int(n_layers), int(q), int(n_paths), int(n_forced),
                                   out.ctypes.data, realized.ctypes.data, warned.ctypes.data)
    if warned[0]:
        capped = min(int(n_paths), q ** n_layers)
        warnings.warn(f"n_paths={capped} < {q}^{n_forced}: cannot fully expand all "
                      "rank-deficient layers", UserWarning, stacklevel=2)
    _lib.check(rc, "allocate_expansions")
    return out[:n_layers], int(realized[0])


@dataclass(frozen=True)
class BatchPathPlan:
    """Candidate-tree plans for a stack of channels (device resident).

    Fields of the reference's BatchPathPlan (detect.py:283-302) are exposed
    as numpy properties (`perm`, `qh`, `r`), materialised on first access."""

    perm_dev: torch.Tensor = field(repr=False)     # (B, N) int32
    r_dev: torch.Tensor = field(repr=False)        # (B, N, N) complex128
    qh_dev: torch.Tensor = field(repr=False)       # (B, N, M) complex128
    tables: torch.Tensor = field(repr=False)       # (B, T) float32, fast-path tables
    expansions: np.ndarray = field(repr=False)     # (N,) int64
    n_paths: int = 0
    augmented: bool = False
    noise_var: float = 0.0
    order: int = 0
    h_dev: torch.Tensor = field(default=None, repr=False)
    h_src: object = field(default=None, repr=False, compare=False)   # the planned h object

    @property
    def batch(self) -> int:
        return self.perm_dev.shape[0]

    @property
    def n(self) -> int:
        return self.perm_dev.shape[1]

    @property
    def m(self) -> int:
        return self.qh_dev.shape[2]

    @cached_property
    def perm(self) -> np.ndarray:
        return self.perm_dev.cpu().numpy().astype(np.int64)

    @cached_property
    def qh(self) -> np.ndarray:
        return self.qh_dev.cpu().numpy()

    @cached_property
    def r(self) -> np.ndarray:
        return self.r_dev.cpu().numpy()

    @cached_property
    def fingerprint(self) -> bytes:
        h = self.h_dev.cpu().numpy().astype(np.complex128)
        return hashlib.sha1(h.tobytes()).digest()


@dataclass(frozen=True)
class PathPlan:
    """Single-channel view (detect.py:305-318)."""

    ordering: np.ndarray
    q_factor: np.ndarray = field(repr=False)
    r_factor: np.ndarray = field(repr=False)
    expansions: np.ndarray
    n_paths: int
    requested_paths: int
    channel: np.ndarray = field(repr=False)
    noise_var: float = 0.0
    fingerprint: bytes = b""
    _batch: BatchPathPlan = field(default=None, repr=False)


def mpnl_plan_batch(h, noise_var: float, n_paths: int, c: Constellation) -> BatchPathPlan:
    """Plan candidate trees for a (B, M, N) channel stack (detect.py:361-388).

    Sorted QR in fp64 on the GPU (K1).  Overloaded channels (N > M) are
    planned on [H; sqrt(nv) I] with the top N - M layers forced full."""
    lib = _lib.load()
    hd, h64, _ = _to_dev_complex(h, "h")
    if hd.dim() == 2:
        hd = hd.unsqueeze(0)
    b, m, n = hd.shape
    expansions, realized = allocate_expansions(n, c.order, n_paths, n_forced=max(0, n - m))
    dev = hd.device
    perm = torch.empty((b, n), dtype=torch.int32, device=dev)
    r = torch.empty((b, n, n), dtype=torch.complex128, device=dev)
    qh = torch.empty((b, n, m), dtype=torch.complex128, device=dev)
    tables = torch.empty((b, int(lib.mpnl_tables_floats(m, n))), dtype=torch.float32, device=dev)
    rc = lib.mpnl_plan(hd.data_ptr(), int(h64), b, m, n, c.order, float(noise_var),
                       perm.data_ptr(), r.data_ptr(), qh.data_ptr(), tables.data_ptr(), _stream())
    _lib.check(rc, "mpnl_plan")
    return BatchPathPlan(perm_dev=perm, r_dev=r, qh_dev=qh, tables=tables,
                         expansions=expansions, n_paths=realized, augmented=n > m,
                         noise_var=float(noise_var), order=c.order, h_dev=hd, h_src=h)


def mpnl_preprocess(h, noise_var: float, n_paths: int, c: Constellation) -> PathPlan:
    """Channel-time planning for a single matrix (detect.py:391-400)."""
    h = np.asarray(h, dtype=complex)
    bp = mpnl_plan_batch(h[None], noise_var, n_paths, c)
    return PathPlan(ordering=bp.perm[0], q_factor=bp.qh[0].conj().T, r_factor=bp.r[0],
                    expansions=bp.expansions, n_paths=bp.n_paths, requested_paths=n_paths,
                    channel=h, noise_var=noise_var,
                    fingerprint=hashlib.sha1(h.tobytes()).digest(), _batch=bp)


# ---------------------------------------------------------------------------
# detection
# ---------------------------------------------------------------------------

def _check_h(plan: BatchPathPlan, h):
    """The reference scores paths by ||y - H x||^2 with the `h` passed to
    mpnl_detect_batch (detect.py:484-486); here the metric is the plan's PED,
    which equals it exactly for the planned channel.  `h` must therefore be the
    planned channel: the same object (free), or equal data (one device
    comparison); another channel raises instead of silently mixing the two."""
    if h is None or h is plan.h_src or h is plan.h_dev:
        return
    if isinstance(h, torch.Tensor):
        t = h.to(plan.h_dev.device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(h))).to(plan.h_dev.device)
    if t.dim() == 2:
        t = t.unsqueeze(0)
    ref = plan.h_dev
    if tuple(t.shape) != tuple(ref.shape):
        raise ValueError("inconsistent channel/observation dimensions")
    if not torch.equal(t.to(torch.complex128), ref.to(torch.complex128)):
        raise ValueError("h differs from the channel the plan was made for: "
                         "re-plan with mpnl_plan_batch(h, ...)")


def _shape_y(plan: BatchPathPlan, y):
    yd, y64, was_np = _to_dev_complex(y, "y")
    if yd.dim() == 1:
        yd = yd.reshape(1, 1, -1)
        squeeze = "vec"
    elif yd.dim() == 2:
        yd = yd.reshape(yd.shape[0], 1, yd.shape[1])
        squeeze = "batch"
    else:
        squeeze = None
    if yd.shape[0] != plan.batch or yd.shape[2] != plan.m:
        raise ValueError("inconsistent channel/observation dimensions")
    return yd.contiguous(), y64, was_np, squeeze


def workspace_stats(ws: torch.Tensor) -> dict:
    """The diagnostic counters a mpnl_detect_hard call left in its workspace."""
    off = int(_lib.load().mpnl_workspace_stats_offset())
    v = ws[off:off + 32].view(torch.int32).tolist()
    keys = ("events", "redecided_fp64", "ties_settled_fp64", "sent_to_fp64", "three_way_ties",
            "fp64_level_ties", "fp64_disagreements", "event_overflows")
    return dict(zip(keys, v))


def mpnl_detect_hard(plan: BatchPathPlan, h, y, c: Constellation, *, return_flags=False,
                     workspace: torch.Tensor | None = None):
    """Hard-output MPNL: (hard labels (..., N), min_metric (...)).

    Equals `take_along_axis(labels, best)` / `metrics[best]` of
    `mpnl_detect_batch` (cli.py:236-239).  fp32 traversal kernel with an
    in-kernel guard; guarded vectors are recomputed in fp64 on the GPU.
    `h` must be the planned channel (`_check_h`: the metric is the plan's PED,
    equal to the reference's true residual for that channel).
    `workspace`: optional caller-owned uint8 device buffer (reused across calls
    on one stream; `workspace_stats` reads its counters); by default a fresh
    one comes from the stream's caching allocator, so concurrent calls on
    different streams never share scratch."""
    lib = _lib.load()
    if c.order != plan.order:
        raise ValueError("constellation does not match the plan")
    _check_h(plan, h)
    yd, y64, was_np, squeeze = _shape_y(plan, y)
    nch, v, m = yd.shape
    n = plan.n
    dev = yd.device
    hard = torch.empty((nch, v, n), dtype=torch.uint8, device=dev)
    metric = torch.empty((nch, v), dtype=torch.float32, device=dev)
    flags = torch.empty((nch, v), dtype=torch.uint8, device=dev) if return_flags else None
    nb = int(lib.mpnl_workspace_bytes(nch * v, n, c.order, plan.expansions.ctypes.data))
    if nb < 0:
        raise ValueError("unsupported configuration")
    ws = workspace
    if ws is None:
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    elif ws.numel() < nb or ws.device != dev or ws.dtype != torch.uint8:
        raise ValueError(f"workspace must be a uint8 tensor of >= {nb} bytes on {dev}")
    rc = lib.mpnl_detect_hard(plan.perm_dev.data_ptr(), plan.r_dev.data_ptr(),
                              plan.qh_dev.data_ptr(), plan.tables.data_ptr(), yd.data_ptr(),
                              int(y64), nch, v, m, n, c.order, plan.expansions.ctypes.data,
                              plan.noise_var, hard.data_ptr(), metric.data_ptr(), _ptr(flags),
                              ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "mpnl_detect_hard")
    outs = [hard, metric] + ([flags] if return_flags else [])
    if squeeze == "batch":
        outs = [o[:, 0] for o in outs]
    elif squeeze == "vec":
        outs = [o[0, 0] for o in outs]
    if was_np:
        outs = [outs[0].cpu().numpy().astype(np.int64), outs[1].cpu().numpy().astype(np.float64)
                ] + ([outs[2].cpu().numpy().astype(bool)] if return_flags else [])
    return tuple(outs)


def _host_complex(a, name):
    """-> (contiguous CPU complex tensor (pinned if it was a torch tensor), is_f64)."""
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.is_cuda:
            raise ValueError(f"{name} must be a host array for mpnl_hard_output")
        if t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        return t.contiguous(), t.dtype == torch.complex128
    arr = np.asarray(a)
    if arr.dtype != np.complex64:
        arr = arr.astype(np.complex128)
    return torch.from_numpy(np.ascontiguousarray(arr)), arr.dtype == np.complex128


def mpnl_hard_output(h, y, noise_var: float, n_paths: int, c: Constellation, *,
                     chunk_channels: int | None = None, out=None):
    """Plan + hard-output detection straight from HOST arrays, one call.

    The reference's hard-output loop `mpnl_plan_batch` -> `mpnl_detect_batch`
    -> `take_along_axis(labels, best)` (cli.py:236-239) with numpy inputs:
    h (n_ch, M, N), y (n_ch, V, M) (one channel per resource block).  Runs
    the C-ABI host pipeline (`mpnl_detect_hard_host`): uploads, kernels and
    downloads of consecutive channel chunks overlap.  Pinned torch CPU
    tensors give asynchronous copies.  Returns host (hard (n_ch, V, N) uint8
    point labels in stream order, min_metric (n_ch, V) float32), complete on
    return (the call synchronises the current stream)."""
    lib = _lib.load()
    ht, h64 = _host_complex(h, "h")
    yt, y64 = _host_complex(y, "y")
    if ht.dim() != 3 or yt.dim() != 3 or yt.shape[0] != ht.shape[0] or yt.shape[2] != ht.shape[1]:
        raise ValueError("inconsistent channel/observation dimensions")
    n_ch, m, n = ht.shape
    v = yt.shape[1]
    ex, _ = allocate_expansions(n, c.order, n_paths, max(0, n - m))
    if chunk_channels is None:
        # >= 4 chunks, <= ~12 MB of observations each: enough to overlap the
        # transfers with the kernels, few enough that per-chunk latency stays small
        ybytes = yt.numel() * yt.element_size()
        chunks = max(4, -(-ybytes // (12 << 20)))
        chunk_channels = max(1, -(-n_ch // chunks))
    if out is None:
        hard = torch.empty((n_ch, v, n), dtype=torch.uint8).pin_memory()
        metric = torch.empty((n_ch, v), dtype=torch.float32).pin_memory()
    else:
        hard, metric = out
    nb = int(lib.mpnl_host_workspace_bytes(n_ch, chunk_channels, v, m, n, c.order, int(h64),
                                           int(y64), ex.ctypes.data))
    if nb < 0:
        raise ValueError("unsupported configuration")
    # per-call scratch from the caching allocator (the call synchronises below,
    # so nothing outlives it; concurrent callers never share it)
    ws = torch.empty(nb, dtype=torch.uint8, device=_device())
    rc = lib.mpnl_detect_hard_host(ht.data_ptr(), int(h64), yt.data_ptr(), int(y64), n_ch, v, m,
                                   n, c.order, ex.ctypes.data, float(noise_var), hard.data_ptr(),
                                   metric.data_ptr(), chunk_channels, ws.data_ptr(), ws.numel(),
                                   _stream())
    _lib.check(rc, "mpnl_hard_output")
    torch.cuda.current_stream().synchronize()
    return hard, metric


def mpnl_hard_output_device(h, y, noise_var: float, n_paths: int, c: Constellation, *,
                            groups: int = 1, out=None):
    """Plan + hard-output detection of DEVICE-resident h (n_ch, M, N) and
    y (n_ch, V, M), one C-ABI call (`mpnl_plan_detect_hard`): the channels
    run as `groups` contiguous groups on forked streams so one group's
    latency-bound stages overlap another's traversal.  Same results as
    mpnl_plan_batch + mpnl_detect_hard.  Returns device (hard (n_ch, V, N)
    uint8, min_metric (n_ch, V) float32), stream-ordered (no sync)."""
    lib = _lib.load()
    hd, h64, _ = _to_dev_complex(h, "h")
    yd, y64, _ = _to_dev_complex(y, "y")
    if hd.dim() != 3 or yd.dim() != 3 or yd.shape[0] != hd.shape[0] or yd.shape[2] != hd.shape[1]:
        raise ValueError("inconsistent channel/observation dimensions")
    n_ch, m, n = hd.shape
    v = yd.shape[1]
    ex, _ = allocate_expansions(n, c.order, n_paths, max(0, n - m))
    if out is None:
        hard = torch.empty((n_ch, v, n), dtype=torch.uint8, device=yd.device)
        metric = torch.empty((n_ch, v), dtype=torch.float32, device=yd.device)
    else:
        hard, metric = out
    nb = int(lib.mpnl_group_workspace_bytes(n_ch, v, m, n, c.order, ex.ctypes.data, int(groups)))
    if nb < 0:
        raise ValueError("unsupported configuration")
    # per-call scratch on the current stream: the forked group streams join back
    # into it before the call returns, so the caching allocator's stream order
    # protects the block when it is reused
    ws = torch.empty(nb, dtype=torch.uint8, device=yd.device)
    rc = lib.mpnl_plan_detect_hard(hd.data_ptr(), int(h64), yd.data_ptr(), int(y64), n_ch, v, m,
                                   n, c.order, ex.ctypes.data, float(noise_var), hard.data_ptr(),
                                   metric.data_ptr(), int(groups), ws.data_ptr(), ws.numel(),
                                   _stream())
    _lib.check(rc, "mpnl_hard_output_device")
    return hard, metric


def mpnl_detect_batch(plan: BatchPathPlan, h, y, c: Constellation):
    """Full parallel-path search (detect.py:473-488).

    Returns (labels (B, P, N), metrics (B, P), best (B,)): labels in path
    order (mixed radix, top layer most significant) and stream order,
    metrics = ||y - Hx||^2, best by (metric, labels) total order.  fp64
    kernel with the reference's decision rules."""
    lib = _lib.load()
    if c.order != plan.order:
        raise ValueError("constellation does not match the plan")
    _check_h(plan, h)
    yd, y64, was_np, squeeze = _shape_y(plan, y)
    nch, v, m = yd.shape
    n, p = plan.n, plan.n_paths
    dev = yd.device
    labels = torch.empty((nch, v, p, n), dtype=torch.uint8, device=dev)
    metrics = torch.empty((nch, v, p), dtype=torch.float64, device=dev)
    best = torch.empty((nch, v), dtype=torch.int64, device=dev)
    rc = lib.mpnl_detect_full(plan.perm_dev.data_ptr(), plan.r_dev.data_ptr(),
                              plan.qh_dev.data_ptr(), yd.data_ptr(), int(y64), nch, v, m, n,
                              c.order, plan.expansions.ctypes.data, plan.noise_var,
                              labels.data_ptr(), metrics.data_ptr(), best.data_ptr(), _stream())
    _lib.check(rc, "mpnl_detect_batch")
    outs = [labels, metrics, best]
    if squeeze == "batch":
        outs = [o[:, 0] for o in outs]
    elif squeeze == "vec":
        outs = [o[0, 0] for o in outs]
    if was_np:
        outs = [outs[0].cpu().numpy().astype(np.int64), outs[1].cpu().numpy(),
                outs[2].cpu().numpy()]
    return tuple(outs)


# ---------------------------------------------------------------------------
# linear ZF / MMSE batch detector
# ---------------------------------------------------------------------------

_LINEAR_MODES = {"zf": 0, "mmse": 1}


def linear_detect_batch(h, y, noise_var, c: Constellation, mode: str, *, return_est=False):
    """Batched ZF / MMSE detection (detect.py:528-557) on the GPU.

    h (B, M, N), y (B, M) numpy or CUDA tensors; noise_var scalar or (B,).
    Returns (hard labels (B, N) int64, llrs (B, N, log2 Q) float64) as numpy
    for numpy inputs (device tensors — labels uint8 — for CUDA inputs), plus
    the raw equalised symbols A^-1 H^H y (B, N) — the biased MMSE output, as
    the reference's single-instance `soft` — when return_est.  Same errors as the
    reference: unknown mode -> ValueError, singular A -> np.linalg.LinAlgError.
    Soft values and LLRs agree with the reference to fp64 rounding (Cholesky
    here, LAPACK inverse there); tests pin the tolerance."""
    if mode not in _LINEAR_MODES:
        raise ValueError(f"unknown linear mode {mode!r}")
    lib = _lib.load()
    ht, _, was_np = _to_dev_complex(h, "h")
    yt, _, _ = _to_dev_complex(y, "y")
    ht, yt = ht.to(torch.complex128).contiguous(), yt.to(torch.complex128).contiguous()
    if ht.dim() != 3 or yt.shape != ht.shape[:2]:
        raise ValueError("h must be (B, M, N) and y (B, M)")
    b, m, n = ht.shape
    dev = ht.device
    nv_arr = np.asarray(noise_var.cpu() if isinstance(noise_var, torch.Tensor) else noise_var,
                        dtype=np.float64)
    nv_t = None
    if nv_arr.ndim:
        nv_t = torch.from_numpy(np.broadcast_to(nv_arr, (b,)).copy()).to(dev)
    labels = torch.empty((b, n), dtype=torch.uint8, device=dev)
    llr = torch.empty((b, n, c.bits_per_symbol), dtype=torch.float64, device=dev)
    est = torch.empty((b, n), dtype=torch.complex128, device=dev) if return_est else None
    n_sing = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = lib.mpnl_linear_detect(ht.data_ptr(), yt.data_ptr(), b, m, n, c.order,
                                _LINEAR_MODES[mode], float(nv_arr) if nv_t is None else 0.0,
                                _ptr(nv_t), float(LLR_CLIP), labels.data_ptr(), llr.data_ptr(),
                                _ptr(est), n_sing.data_ptr(), _stream())
    _lib.check(rc, "linear_detect_batch")
    if int(n_sing.item()):
        raise np.linalg.LinAlgError("Singular matrix")
    if was_np:
        out = (labels.cpu().numpy().astype(np.int64), llr.cpu().numpy())
        return out + (est.cpu().numpy(),) if return_est else out
    return (labels, llr, est) if return_est else (labels, llr)


def zf_detect(inp: "DetectorInput") -> "DetectionOutput":
    """Zero-forcing, single instance (detect.py:100-119) through the batch
    kernel (B = 1).  Same SingularChannelError cases: M < N, singular Gram
    matrix, condition number above 1e12."""
    if inp.m < inp.n:
        raise SingularChannelError("ZF requires M >= N")
    h = np.asarray(inp.h, dtype=complex)
    if not np.isfinite(c := np.linalg.cond(h)) or c * c > 1e12:   # cond(H^H H) = cond(H)^2
        raise SingularChannelError("rank-deficient channel")
    return _linear_single(inp, "zf")


def mmse_detect(inp: "DetectorInput") -> "DetectionOutput":
    """MMSE, single instance (detect.py:122-145) through the batch kernel:
    `soft` is the raw (biased) MMSE output, slicing and LLRs use the unbiased
    estimate with the effective noise variance."""
    return _linear_single(inp, "mmse")


def _linear_single(inp, mode):
    c = inp.constellation
    try:
        lab, llr, soft = linear_detect_batch(np.asarray(inp.h)[None], np.asarray(inp.y)[None],
                                             float(inp.noise_var), c, mode, return_est=True)
    except np.linalg.LinAlgError:
        raise SingularChannelError("rank-deficient channel") from None
    labels = lab[0]
    hard = c.points[labels]
    return DetectionOutput(hard=hard, hard_labels=labels, llrs=llr[0],
                           min_metric=_residual_metric(np.asarray(inp.h), np.asarray(inp.y), hard),
                           soft=soft[0])


# ---------------------------------------------------------------------------
# single-instance API (detect.py:30-77, 456-506, 560-576)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DetectorInput:
    h: np.ndarray
    y: np.ndarray
    noise_var: float
    constellation: Constellation

    def __post_init__(self):
        h = np.asarray(self.h, dtype=complex)
        y = np.asarray(self.y, dtype=complex).ravel()
        if h.ndim != 2 or y.size != h.shape[0]:
            raise ValueError("inconsistent channel/observation dimensions")
        if self.noise_var <= 0:
            raise ValueError("noise_var must be positive")
        object.__setattr__(self, "h", h)
        object.__setattr__(self, "y", y)

    @property
    def m(self) -> int:
        return self.h.shape[0]

    @property
    def n(self) -> int:
        return self.h.shape[1]


@dataclass(frozen=True)
class CandidateList:
    candidates: np.ndarray = field(repr=False)
    labels: np.ndarray = field(repr=False)
    metrics: np.ndarray = field(repr=False)

    @property
    def n_paths(self) -> int:
        return self.candidates.shape[0]


@dataclass(frozen=True)
class DetectionOutput:
    hard: np.ndarray = field(repr=False)
    hard_labels: np.ndarray = field(repr=False)
    llrs: np.ndarray = field(repr=False)
    min_metric: float
    soft: np.ndarray | None = field(default=None, repr=False)


def _residual_metric(h, y, x):
    r = y - h @ x
    return float(np.real(np.vdot(r, r)))


def _candidate_llrs_batch(labels, metrics, noise_var, c: Constellation,
                          clip: float = LLR_CLIP):
    """Max-log LLRs over candidate lists (detect.py:439-453) on the GPU.

    labels (B, P, N) and metrics (B, P) — numpy (result numpy float64) or CUDA
    tensors (uint8 / float64; result stays on the device).  `noise_var` is a
    scalar or a per-row (B,) array, as in the reference.  Returns
    (B, N, log2 Q) float64, bit-identical to the reference."""
    lib = _lib.load()
    was_np = not isinstance(labels, torch.Tensor)
    dev = labels.device if not was_np else _device()
    if was_np:
        lab = np.asarray(labels)
        if lab.size and (lab.min() < 0 or lab.max() >= c.order):
            raise ValueError("labels outside the constellation")
        lab_t = torch.from_numpy(np.ascontiguousarray(lab.astype(np.uint8))).to(dev)
    else:
        lab_t = labels.to(dev, torch.uint8).contiguous()
    met_t = (torch.as_tensor(np.asarray(metrics, dtype=np.float64)) if not
             isinstance(metrics, torch.Tensor) else metrics).to(dev, torch.float64).contiguous()
    if lab_t.dim() != 3 or met_t.shape != lab_t.shape[:2]:
        raise ValueError("labels must be (B, P, N) and metrics (B, P)")
    b, p, n = lab_t.shape
    nv_arr = np.asarray(noise_var.cpu() if isinstance(noise_var, torch.Tensor) else noise_var,
                        dtype=np.float64)
    nv_t = None
    if nv_arr.ndim:
        nv_t = torch.from_numpy(np.ascontiguousarray(nv_arr.reshape(-1))).to(dev)
        if nv_t.numel() != b:
            raise ValueError("noise_var must be a scalar or one value per candidate list")
    llr = torch.empty((b, n, c.bits_per_symbol), dtype=torch.float64, device=dev)
    rc = lib.mpnl_candidate_llrs(lab_t.data_ptr(), met_t.data_ptr(), b, p, n, c.order,
                                 float(nv_arr) if nv_t is None else 0.0, _ptr(nv_t),
                                 float(clip), llr.data_ptr(), _stream())
    _lib.check(rc, "_candidate_llrs_batch")
    return llr.cpu().numpy() if was_np else llr


def llr_from_candidates(clist: CandidateList, noise_var: float, c: Constellation,
                        clip: float = LLR_CLIP) -> np.ndarray:
    """List max-log LLRs over one candidate list (detect.py:455-462)."""
    if clist.n_paths < 1:
        raise ValueError("empty candidate list")
    return _candidate_llrs_batch(np.asarray(clist.labels)[None],
                                 np.asarray(clist.metrics)[None], noise_var, c, clip)[0]


def mpnl_detect_llrs(plan: BatchPathPlan, h, y, c: Constellation, noise_var=None,
                     clip: float = LLR_CLIP, *, precision: str = "fp64", return_flags=False):
    """The link simulator's MPNL soft output (linksim.py:151-155):
    `mpnl_detect_batch` then `_candidate_llrs_batch`.  `noise_var` defaults to
    the plan's.  Returns LLRs shaped like y's leading axes + (N, log2 Q).

    precision="fp64" (default): the fp64 full-list kernel, then the list-LLR
    kernel, the candidate list staying on the device in between — bit-identical
    to the reference.
    precision="fp32": the fused fp32 traversal + LLR kernel
    (`mpnl_detect_llrs_fast`; no candidate list), about 30x faster.  Vectors it
    flags (an fp32 decision within the guard bound of a boundary on a path that
    can reach an unclipped LLR) are recomputed by the fp64 path here, so every
    LLR agrees with the reference within the fp32 metric error,
    |d llr| <= 2 ped_tol / noise_var (~1e-6 of the metrics / noise_var).  Needs
    a scalar noise_var; plans without an fp32 path (overloaded channels, more
    than 3 expanded layers) take the fp64 path.  `return_flags` also returns the
    boolean mask of recomputed vectors."""
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"unknown precision {precision!r}")
    was_np = not isinstance(y, torch.Tensor)
    yt = y if not was_np else torch.from_numpy(np.ascontiguousarray(np.asarray(y))).to(_device())
    nv = plan.noise_var if noise_var is None else noise_var
    if isinstance(nv, np.ndarray) and nv.ndim:
        nv = nv.reshape(-1)
    fast = (precision == "fp32" and np.ndim(nv) == 0 and not plan.augmented)
    if fast:
        out = _detect_llrs_fp32(plan, h, yt, c, float(nv), float(clip))
        if out is not None:
            llr, flags = out
            if was_np:
                llr, flags = llr.cpu().numpy(), flags.cpu().numpy()
            return (llr, flags) if return_flags else llr
    labels, metrics, _ = mpnl_detect_batch(plan, h, yt, c)
    lead = labels.shape[:-2]
    n, p = labels.shape[-1], labels.shape[-2]
    llr = _candidate_llrs_batch(labels.reshape(-1, p, n), metrics.reshape(-1, p), nv, c, clip)
    llr = llr.reshape(*lead, n, c.bits_per_symbol)
    llr = llr.cpu().numpy() if was_np else llr
    if return_flags:
        flags = np.ones(lead, bool) if was_np else torch.ones(lead, dtype=torch.bool,
                                                               device=llr.device)
        return llr, flags
    return llr


def _detect_llrs_fp32(plan: BatchPathPlan, h, yt, c: Constellation, nv: float, clip: float):
    """`mpnl_detect_llrs_fast` + the fp64 re-computation of the vectors it
    flags.  Returns (llr, recomputed mask) on the device, or None when the plan
    has no fp32 path."""
    lib = _lib.load()
    if c.order != plan.order:
        raise ValueError("constellation does not match the plan")
    _check_h(plan, h)
    yd, y64, _, squeeze = _shape_y(plan, yt)
    nch, v, m = yd.shape
    n, bps = plan.n, c.bits_per_symbol
    dev = yd.device
    nb = int(lib.mpnl_workspace_bytes(nch * v, n, c.order, plan.expansions.ctypes.data))
    if nb < 0:
        return None
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    llr = torch.empty((nch, v, n, bps), dtype=torch.float64, device=dev)
    flags = torch.empty((nch, v), dtype=torch.uint8, device=dev)
    rc = lib.mpnl_detect_llrs_fast(plan.perm_dev.data_ptr(), plan.r_dev.data_ptr(),
                                   plan.qh_dev.data_ptr(), plan.tables.data_ptr(), yd.data_ptr(),
                                   int(y64), nch, v, m, n, c.order,
                                   plan.expansions.ctypes.data, plan.noise_var, nv, clip,
                                   llr.data_ptr(), flags.data_ptr(), ws.data_ptr(), ws.numel(),
                                   _stream())
    if rc == _lib.MPNL_EUNSUPPORTED:
        return None
    _lib.check(rc, "mpnl_detect_llrs")
    redo = flags.bool()
    idx = redo.reshape(-1).nonzero().reshape(-1)
    if idx.numel():
        # flagged vectors through the fp64 list path: one plan row per vector
        ch = idx // v
        p = plan.n_paths
        yv = yd.reshape(nch * v, 1, m).index_select(0, idx).contiguous()
        perm_g = plan.perm_dev.index_select(0, ch).contiguous()
        r_g = plan.r_dev.index_select(0, ch).contiguous()
        qh_g = plan.qh_dev.index_select(0, ch).contiguous()
        k = int(idx.numel())
        labels = torch.empty((k, p, n), dtype=torch.uint8, device=dev)
        metrics = torch.empty((k, p), dtype=torch.float64, device=dev)
        best = torch.empty((k,), dtype=torch.int64, device=dev)
        rc = lib.mpnl_detect_full(perm_g.data_ptr(), r_g.data_ptr(), qh_g.data_ptr(),
                                  yv.data_ptr(), int(y64), k, 1, m, n, c.order,
                                  plan.expansions.ctypes.data, plan.noise_var,
                                  labels.data_ptr(), metrics.data_ptr(), best.data_ptr(), _stream())
        _lib.check(rc, "mpnl_detect_llrs (fp64 recomputation)")
        fix = _candidate_llrs_batch(labels, metrics, nv, c, clip)
        llr.reshape(nch * v, n, bps).index_copy_(0, idx, fix)
    if squeeze == "batch":
        llr, redo = llr[:, 0], redo[:, 0]
    elif squeeze == "vec":
        llr, redo = llr[0, 0], redo[0, 0]
    return llr, redo


def mpnl_detect(plan: PathPlan, inp: DetectorInput):
    """Evaluate the planned candidate paths for one observation."""
    fp = hashlib.sha1(np.asarray(inp.h, dtype=complex).tobytes()).digest()
    if fp != plan.fingerprint:
        raise ValueError("plan/channel fingerprint mismatch")
    c = inp.constellation
    labels, metrics, best = mpnl_detect_batch(plan._batch, inp.h[None], inp.y[None], c)
    labels, metrics, b = labels[0], metrics[0], int(best[0])
    cands = c.points[labels]
    clist = CandidateList(candidates=cands, labels=labels, metrics=metrics)
    llrs = llr_from_candidates(clist, inp.noise_var, c)
    hard = cands[b]
    out = DetectionOutput(hard=hard, hard_labels=labels[b], llrs=llrs,
                          min_metric=_residual_metric(inp.h, inp.y, hard))
    return clist, out


DETECTOR_NAMES = ("zf", "mmse", "mpnl")


def detect(name: str, inp: DetectorInput, n_paths: int = 32) -> DetectionOutput:
    """Name dispatch (detect.py:563-576).  Only the MPNL path is in scope for
    this library, plus the linear ZF / MMSE detectors; the
    reference's ml / sphere stay in the reference."""
    if name == "mpnl":
        plan = mpnl_preprocess(inp.h, inp.noise_var, n_paths, inp.constellation)
        return mpnl_detect(plan, inp)[1]
    if name == "zf":
        return zf_detect(inp)
    if name == "mmse":
        return mmse_detect(inp)
    if name in ("ml", "sphere"):
        raise NotImplementedError(f"detector {name!r} is outside the MPNL hot path")
    raise ValueError(f"unknown detector {name!r}")
