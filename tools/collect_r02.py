"""Copy one evidence run (tools/gpu_r02_evidence.sh -> gpurun_out/e_*) into the
committed profiles/r02/ files, with the ncu summaries extended by the pipe /
shared-memory / occupancy metrics the DESIGN analysis quotes.

    python tools/collect_r02.py"""
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles" / "r02"
P.mkdir(parents=True, exist_ok=True)

COPY = {
    "e_bench_default.json": "bench_default.json", "e_bench_reference.json": "bench_reference_arm.json",
    "e_bench_C1.json": "bench_C1.json", "e_bench_C2.json": "bench_C2.json",
    "e_bench_C3.json": "bench_C3.json", "e_bench_C4.json": "bench_C4.json",
    "e_stage_times.txt": "stage_times.txt", "e_smoke.log": "smoke.log",
    "e_c1_steady_and_per_vector.jsonl": "c1_steady_and_per_vector.jsonl",
    "e_soft_C2.json": "soft_C2.json", "e_soft_C5P64.json": "soft_C5P64.json",
    "e_soft_kernel_times.txt": "soft_kernel_times.txt", "e_linksim_bench.jsonl": "linksim_bench.jsonl",
    "e_ffma2_forms.txt": "ffma2_forms.txt",
}
for src, dst in COPY.items():
    if (G / src).exists():
        lines = [l for l in (G / src).read_text().splitlines() if not l.startswith("[gpurun]")]
        (P / dst).write_text("\n".join(lines) + "\n")
if (G / "e_gpu_tests.log").exists():
    (P / "gpu_tests_summary.txt").write_text(
        "\n".join((G / "e_gpu_tests.log").read_text().splitlines()[-8:]) + "\n")
if (G / "e_launches_default.csv").exists():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), "launches",
                          str(G / "e_launches_default.csv")], capture_output=True, text=True).stdout
    (P / "launches_default.txt").write_text(
        "# ncu --metrics gpu__time_duration.sum --clock-control none of\n"
        "#   python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline\n"
        "# (cold cache, serialised launches: shares, not absolute times; ns)\n" + out)

EXTRA = [
    "sm__cycles_elapsed.max",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__sass_inst_executed_op_shared_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.per_cycle_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block", "launch__waves_per_multiprocessor",
    "sass__inst_executed_register_spilling",
]


def ncu(tag, dst, title):
    txt, raw = G / f"{tag}.txt", G / f"{tag}_raw.csv"
    if not txt.exists():
        return
    out = [f"# {title}", txt.read_text().rstrip()]
    if raw.exists():
        rows = list(csv.reader(open(raw)))
        d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
        out.append("  further metrics (same capture):")
        for k in EXTRA:
            if k in d:
                out.append(f"    {k:82s} {d[k]:>16s} {u.get(k, '')}")
    sass = G / f"{tag}_sass.csv"
    if sass.exists():
        rows = list(csv.reader(open(sass)))
        hdr = rows[1]
        si, ie = hdr.index("Source"), hdr.index("Instructions Executed")
        tot, ops = 0, {}
        for r in rows[2:]:
            t = r[si].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            n = int(r[ie])
            ops[op] = ops.get(op, 0) + n
            tot += n
        out.append(f"  executed warp instructions by opcode (source page): total {tot:,}")
        for op, n in sorted(ops.items(), key=lambda x: -x[1])[:12]:
            out.append(f"    {op:10s} {n:>16,d} {100 * n / tot:5.1f}%")
    (P / dst).write_text("\n".join(out) + "\n")


ncu("e_ncu_traverse_C5P1024", "ncu_traverse_C5P1024.txt",
    "ncu --set full --clock-control none, C5P1024 full size (tools/prof_full.sh), headline traversal")
ncu("e_ncu_plan_C5", "ncu_plan_qr_reg_C5.txt",
    "ncu --set full --clock-control none, plan kernel on C5's 2,048 24x24 channels")
ncu("e_ncu_soft_C2", "ncu_soft_llr_C2.txt",
    "ncu --set full --clock-control none, fp32 soft-output kernel on C2 (273 RB x 168 RE)")
ncu("e_ncu_select_C5P1024", "ncu_select_C5P1024.txt",
    "ncu --set full --clock-control none, 64-QAM partial-layer selection (E = 16) on C5P1024")
ncu("e_ncu_check_C5P1024", "ncu_check_C5P1024.txt",
    "ncu --set full --clock-control none, event checks on C5P1024")
ncu("e_ncu_check_C5P16", "ncu_check_C5P16.txt",
    "ncu --set full --clock-control none, event checks on C5P16")
ncu("e_ncu_prep2_C5P16", "ncu_prep2_C5P16.txt",
    "ncu --set full --clock-control none, fp64 rotation + guard bounds on C5 (344,064 vectors)")
ncu("e_ncu_verify_C5P16", "ncu_verify_C5P16.txt",
    "ncu --set full --clock-control none, winner re-trace on C5 (344,064 vectors)")

# roofline.traffic of the headline config from this round's capture
raw = G / "e_ncu_traverse_C5P1024_raw.csv"
if raw.exists():
    rows = list(csv.reader(open(raw)))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * mul[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * mul[u["dram__bytes_write.sum"]]
    tj = ROOT / "profiles" / "traffic.json"
    t = json.loads(tj.read_text())
    t["C5P1024"] = {"dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr),
                    "kernel": d["Kernel Name"].split("(")[0],
                    "source": "profiles/r02/ncu_traverse_C5P1024.txt (ncu --set full)"}
    tj.write_text(json.dumps(t, indent=1) + "\n")
print("profiles/r02 updated:", sorted(p.name for p in P.iterdir()))
