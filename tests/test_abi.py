"""CPU: the C-ABI library loads, exports every symbol include/mpnl_b200.h
declares, and its host-only entry points (the allocator port) match the
reference.  No GPU compute here."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2409_14355_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def header_symbols():
    text = (ROOT / "include" / "mpnl_b200.h").read_text()
    return sorted(set(re.findall(r"\b(mpnl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert lib.mpnl_version() == 0x000100


def test_alloc_port_matches_reference_grid():
    lib = _lib.load()
    g = np.load(GOLD / "alloc.npz")
    out = np.zeros(32, np.int64)
    real = np.zeros(1, np.int64)
    warned = np.zeros(1, np.int32)
    for i in range(len(g["n"])):
        n = int(g["n"][i])
        rc = lib.mpnl_alloc_expansions(n, int(g["q"][i]), int(g["p"][i]), int(g["nf"][i]),
                                       out.ctypes.data, real.ctypes.data, warned.ctypes.data)
        assert rc == 0
        assert real[0] == g["realized"][i]
        assert np.array_equal(out[:n], g["expansions"][i, :n]), (n, g["q"][i], g["p"][i])
        assert warned[0] == g["warned"][i]


def test_alloc_error_behaviour():
    lib = _lib.load()
    out = np.zeros(4, np.int64)
    real = np.zeros(1, np.int64)
    rc = lib.mpnl_alloc_expansions(3, 4, 0, 0, out.ctypes.data, real.ctypes.data, None)
    assert rc == _lib.MPNL_EINVAL
    assert _lib.last_error() == "n_paths must be >= 1"
    with pytest.raises(ValueError, match="n_paths must be >= 1"):
        _lib.check(rc, "x")


def test_shim_allocate_expansions_warns():
    from paper_2409_14355_b200 import detect
    with pytest.warns(UserWarning, match="rank-deficient"):
        e, r = detect.allocate_expansions(3, 4, 8, 2)
    assert r == 8 and int(np.prod(e)) == 8


def test_tables_and_workspace_sizes():
    lib = _lib.load()
    assert lib.mpnl_tables_floats(12, 12) % 4 == 0
    ex = np.array([1] * 10 + [4, 16], dtype=np.int64)
    assert lib.mpnl_workspace_bytes(1000, 12, 16, ex.ctypes.data) >= 1000 * (8 + 4 + 16 + 8 + 64)
