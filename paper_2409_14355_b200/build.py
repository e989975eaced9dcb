"""Build the in-tree CUDA library `paper_2409_14355_b200/_lib/libmpnl_b200.so`.

Every `.cu` under `csrc/` is compiled for sm_100a with nvcc (in parallel, one
process per translation unit; up to date objects are reused), then linked into
one shared library with the CUDA runtime linked statically, so the library
only needs the driver on the GPU box.  The Python package loads it with
ctypes through the C ABI in `include/mpnl_b200.h`.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# MPNL_VARIANT=<name> MPNL_EXTRA_FLAGS="-D..." builds an experimental variant
# into _lib/libmpnl_b200_<name>.so (load it with MPNL_LIB=<path>)
_VARIANT = os.environ.get("MPNL_VARIANT", "")
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / (f"libmpnl_b200_{_VARIANT}.so" if _VARIANT else "libmpnl_b200.so")
OBJ_DIR = PKG.parent / "build" / (f"obj_{_VARIANT}" if _VARIANT else "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-I", str(PKG.parent / "include")] + os.environ.get("MPNL_EXTRA_FLAGS", "").split()


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def _stale(obj: Path, src: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *deps])


def build(jobs: int | None = None, verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    deps = sorted(CSRC.glob("*.cuh")) + sorted((PKG.parent / "include").glob("*.h"))
    nvcc = _nvcc()

    def compile_one(src: Path) -> Path:
        obj = OBJ_DIR / (src.stem + ".o")
        if _stale(obj, src, deps):
            cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
        return obj

    jobs = jobs or max(1, os.cpu_count() or 1)
    # biggest units first (the large-N traversal instantiations dominate)
    srcs.sort(key=lambda s: (("_p3" in s.name) * 3 + ("_p2" in s.name) * 2
                             + ("_p1" in s.name)), reverse=True)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(compile_one, srcs))
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB),
               *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
