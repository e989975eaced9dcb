"""Static SASS instruction census of the traversal kernel instance each config
runs (FFMA2 vs slicing / guard / bookkeeping instructions).

    python tools/sass_census.py > profiles/r02/sass_census.txt

For each BASELINE config: the traverse_kernel<N, L, VPI, SH, ONEB> instance
the launcher picks (as in the ncu launch lists), its SASS from the in-tree
objects (cuobjdump -sass), opcode counts over the whole kernel and the
algorithmic FFMA2 count per path (sum over layers of 2 pos + 2), to show how
much of the fma pipe's work is the path arithmetic."""

import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OBJ = ROOT / "build" / "obj"
# config -> (N, L, VPI, SH, ONEB, P, PT)
CFG = {"C1": (8, 4, 1, 0, 0, 32, 4), "C2": (12, 4, 0, 1, 1, 64, 2),
       "C3": (16, 8, 0, 1, 0, 128, 2), "C4": (32, 4, 0, 0, 0, 256, 1),
       "C5P16": (24, 8, 1, 0, 0, 16, 1), "C5P64": (24, 8, 0, 0, 0, 64, 1),
       "C5P256": (24, 8, 0, 0, 0, 256, 1), "C5P1024": (24, 8, 0, 0, 0, 1024, 1)}
GROUPS = {
    "FFMA2 (packed fp32 FMA: path arithmetic + magic rounding + guard)": ["FFMA2"],
    "FADD2 / FMUL2 (packed)": ["FADD2", "FMUL2"],
    "FMUL (slicing, .SAT)": ["FMUL"],
    "FFMA / FADD (scalar fp32)": ["FFMA", "FADD"],
    "FMNMX / FSETP (guard, top-3)": ["FMNMX", "FSETP", "FSEL"],
    "LDS (r'' row pairs, tables)": ["LDS"],
    "integer / logic (LOP3, IMAD, IADD3, ISETP, SHF, ...)": ["LOP3", "IMAD", "IADD3", "ISETP",
                                                             "SHF", "LEA", "SEL", "IABS",
                                                             "VIADD", "IMNMX", "VIMNMX"],
    "warp (SHFL, REDUX, VOTE)": ["SHFL", "REDUX", "VOTE", "MATCH"],
    "memory other (LDG, STG, STS, ATOMS, UBLKCP, SYNCS)": ["LDG", "STG", "STS", "ATOMS", "ATOM",
                                                           "RED", "UBLKCP", "SYNCS", "LDSM"],
}


def mangled(n, l, vpi, sh, oneb):
    b = lambda x: "1" if x else "0"   # noqa: E731
    return (f"_ZN4mpnl15traverse_kernelILi{n}ELi{l}ELb{b(vpi)}ELb{b(sh)}ELb{b(oneb)}EEEv"
            "NS_10DetectArgsENS_10TreeParamsE")


def sass(obj, fun):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, str(obj)], capture_output=True,
                         text=True).stdout
    ops = []
    for ln in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", ln)
        if m:
            ops.append(m.group(2))
    return ops


def main():
    for name, (n, l, vpi, sh, oneb, p, pt) in CFG.items():
        part = (n - 1) // 8
        obj = OBJ / f"traverse_l{l}_p{part}.o"
        ops = sass(obj, mangled(n, l, vpi, sh, oneb))
        c = Counter(ops)
        tot = sum(c.values())
        alg = sum(2 * pos + 2 for pos in range(n))    # FFMA2 of one path
        print(f"== {name}: traverse_kernel<{n}, {l}, {vpi}, {sh}, {oneb}> "
              f"(P = {p}, {pt} path(s) per lane) -- {tot} SASS instructions")
        for g, keys in GROUPS.items():
            k = sum(c[x] for x in keys)
            print(f"   {k:6d}  {100.0 * k / max(tot, 1):5.1f}%  {g}")
        print(f"   algorithmic FFMA2 per path {alg} (x {pt} paths per lane in the unrolled "
              f"body = {alg * pt}); FFMA2 in the binary {c['FFMA2']}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
