"""Summarise ncu captures for profiles/.

    python tools/ncu_summary.py full REPORT.ncu-rep      # key metrics of a --set full capture
    python tools/ncu_summary.py launches LAUNCHES.csv    # per-kernel time shares
    python tools/ncu_summary.py traffic r01              # profiles/traffic.json + per-config summaries

Prints plain text (commit the output under profiles/)."""

from __future__ import annotations

import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")]
        stalls = sorted(((k, float(v.replace(",", "") or 0)) for k, v in stalls),
                        key=lambda x: -x[1])
        print("  top stall reasons (warps per issue-active cycle):")
        for k, v in stalls[:8]:
            name = k.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", "")
            print(f"    {name:30s} {v:6.3f}")


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def _bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                        "Gbyte": 1e9}.get(unit, 1)


def traffic(tag, outdir="profiles"):
    """<outdir>/traffic.json from gpurun_out/<tag>_trav_<cfg>.ncu-rep captures."""
    import glob
    import json
    import os
    res = {}
    for p in sorted(glob.glob(f"gpurun_out/{tag}_trav_*.ncu-rep")):
        cfg = p.rsplit("_trav_", 1)[1].split(".")[0]
        rows, units = _raw(p)
        d = rows[0]
        rd = _bytes(d["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
        wr = _bytes(d["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
        res[cfg] = {"dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr),
                    "kernel": d["Kernel Name"].split("(")[0],
                    "source": f"profiles/{tag}_ncu_traverse_{cfg}.txt (ncu --set full)"}
        os.makedirs(outdir, exist_ok=True)
        with open(f"{outdir}/{tag}_ncu_traverse_{cfg}.txt", "w") as f:
            import contextlib
            import io
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                full(p)
            f.write(f"# ncu --set full --clock-control none, {cfg} full size, from {os.path.basename(p)}\n")
            f.write(buf.getvalue())
    with open(f"{outdir}/traffic.json", "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launches(path):
    tot, cnt = defaultdict(float), defaultdict(int)
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0][:70]
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                  "ms": 1e3}.get(unit, 1.0)
            tot[k] += v
            cnt[k] += 1
    s = sum(tot.values()) or 1.0
    print(f"{'total us':>10s} {'share':>6s} {'n':>4s}  kernel   (cold-cache, serialised by ncu)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.1f} {100 * v / s:5.1f}% {cnt[k]:4d}  {k}")


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
