"""ctypes binding of the C ABI in `include/mpnl_b200.h`.

The library is built in-tree by `paper_2409_14355_b200/build.py`
(`__graft_entry__.build()`).  There is no fallback: if it is missing or the
machine has no CUDA device, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_LIB_PATH = Path(os.environ.get("MPNL_LIB") or
                 Path(__file__).resolve().parent / "_lib" / "libmpnl_b200.so")
_lock = threading.Lock()
_lib = None

MPNL_OK, MPNL_EINVAL, MPNL_EUNSUPPORTED, MPNL_ECUDA = 0, -1, -2, -3

_vp, _i32, _i64, _f64 = C.c_void_p, C.c_int, C.c_int64, C.c_double
_SIGS = {
    "mpnl_last_error": ([], C.c_char_p),
    "mpnl_version": ([], _i32),
    "mpnl_alloc_expansions": ([_i32, _i32, _i64, _i32, _vp, _vp, _vp], _i32),
    "mpnl_tables_floats": ([_i32, _i32], _i64),
    "mpnl_plan": ([_vp, _i32, _i64, _i32, _i32, _i32, _f64, _vp, _vp, _vp, _vp, _vp], _i32),
    "mpnl_workspace_bytes": ([_i64, _i32, _i32, _vp], _i64),
    "mpnl_detect_hard": ([_vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp,
                          _f64, _vp, _vp, _vp, _vp, _i64, _vp], _i32),
    "mpnl_detect_hard_stage": ([_i32, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i32, _i32,
                                _i32, _vp, _f64, _vp, _vp, _vp, _vp, _i64, _vp], _i32),
    "mpnl_host_workspace_bytes": ([_i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp], _i64),
    "mpnl_detect_hard_host": ([_vp, _i32, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp, _f64,
                               _vp, _vp, _i64, _vp, _i64, _vp], _i32),
    "mpnl_detect_full": ([_vp, _vp, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp, _f64,
                          _vp, _vp, _vp, _vp], _i32),
    "mpnl_detect_llrs_fast": ([_vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp,
                               _f64, _f64, _f64, _vp, _vp, _vp, _i64, _vp], _i32),
    "mpnl_group_workspace_bytes": ([_i64, _i64, _i32, _i32, _i32, _vp, _i32], _i64),
    "mpnl_plan_detect_hard": ([_vp, _i32, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp, _f64,
                               _vp, _vp, _i32, _vp, _i64, _vp], _i32),
    "mpnl_candidate_llrs": ([_vp, _vp, _i64, _i64, _i32, _i32, _f64, _vp, _f64, _vp, _vp],
                            _i32),
    "mpnl_linear_detect": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _f64, _vp, _f64, _vp, _vp,
                            _vp, _vp, _vp], _i32),
    "mpnl_workspace_stats_offset": ([], _i64),
    "mpnl_slot_receive": ([_vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp], _i32),
    "mpnl_dmrs_ls_estimate": ([_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp], _i32),
    "mpnl_select_symbols": ([_vp, _i64, _i32, _i64, _vp, _i32, _vp, _vp], _i32),
    "mpnl_ldpc_graph_dims": ([_vp, _i32, _i32, _vp, _vp], _i32),
    "mpnl_ldpc_build": ([_vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp], _i32),
    "mpnl_ldpc_decode": ([_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i64, _i32, _i32, _i32, _f64,
                          _f64, _vp, _vp, _vp, _vp, _vp], _i32),
    "mpnl_ldpc_encode": ([_vp, _i32, _i32, _vp, _i64, _i32, _i32, _vp, _vp], _i32),
    "mpnl_ldpc_syndrome": ([_vp, _i32, _i32, _vp, _i64, _i32, _vp, _vp], _i32),
    "mpnl_ffma_probe": ([_vp, _i32, _i32, _i32, _vp], _i64),
    "mpnl_ffma2_probe": ([_vp, _i32, _i32, _i32, _vp], _i64),
}


class MpnlError(RuntimeError):
    pass


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes library; raises if not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise MpnlError(f"MPNL CUDA library not built ({_LIB_PATH}); run "
                                "`python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(str(_LIB_PATH))
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def last_error() -> str:
    return load().mpnl_last_error().decode()


def check(rc: int, where: str):
    if rc == MPNL_OK:
        return
    msg = last_error()
    if rc == MPNL_EINVAL:
        raise ValueError(msg)
    if rc == MPNL_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise MpnlError(f"{where}: {msg}")
