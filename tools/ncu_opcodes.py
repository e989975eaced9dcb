"""Dynamic instruction mix (executed warp instructions per SASS opcode) of the
first kernel in an ncu --set full report.

    python tools/ncu_opcodes.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys

csv.field_size_limit(1 << 30)
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-metric-instances",
                      "details"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
kern = d.get("Kernel Name", "?")
for metric in ("sass__inst_executed_per_opcode", "sass__inst_executed_per_opcode_category"):
    raw = d[metric]
    total, _, rest = raw.partition(" ")
    items = []
    for part in rest.strip("()").split(";"):
        part = part.strip()
        if ":" in part:
            k, x = part.rsplit(":", 1)
            items.append((k.strip(), float(x)))
    tot = float(total)
    print(f"{metric} for {kern[:70]}: {tot:.4g} warp instructions")
    for k, x in sorted(items, key=lambda t: -t[1])[:top]:
        print(f"   {x:16.0f}  {100 * x / tot:5.1f}%  {k}")
