"""Attribute an ncu SASS-level source page to CUDA source lines.

    python tools/sass_lines.py build/obj/<unit>.o <kernel-substring> <ncu_sass.csv> [top]

The ncu CSV (``--page source --csv --print-source=sass``) lists the kernel's
instructions in program order; ``nvdisasm -g`` of the same object gives each
instruction's source line.  Prints instructions executed and stall samples
per source line (the object must be the one that was profiled)."""

from __future__ import annotations

import csv
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path


def sass_lines(obj: str, kernel: str):
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=tmp,
                   capture_output=True)
    cubin = next(tmp.glob("*.cubin"))
    out = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True,
                         text=True).stdout
    funcs, cur, line = {}, None, None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = f"{Path(m.group(1)).name}:{m.group(2)}"
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            funcs[cur].append(line)
    names = [f for f in funcs if kernel in f]
    if not names:
        raise SystemExit(f"no function matching {kernel!r}; have {list(funcs)[:10]}")
    return funcs[names[0]], names[0]


def main():
    obj, kernel, csvf = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lines, name = sass_lines(obj, kernel)
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    smp = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ie]
    if len(data) != len(lines):
        print(f"warning: {len(data)} profiled vs {len(lines)} disassembled instructions",
              file=sys.stderr)
    ins, sam = defaultdict(int), defaultdict(int)
    for i, r in enumerate(data):
        key = lines[i] if i < len(lines) else "?"
        ins[key] += int(r[ie] or 0)
        sam[key] += int(r[smp] or 0)
    ts = sum(sam.values()) or 1
    ti = sum(ins.values()) or 1
    print(f"{name}: {ti} instructions, {ts} samples")
    for k in sorted(sam, key=lambda k: -sam[k])[:top]:
        print(f"{100 * sam[k] / ts:5.1f}% smp {100 * ins[k] / ti:5.1f}% ins  {k}")


if __name__ == "__main__":
    main()
