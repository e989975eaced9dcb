# Round-2 evidence on one B200 (run through gpurun from the repo root); outputs
# land in gpurun_out/ and the committed copies in profiles/r02/.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_r02_evidence.sh'
set -u
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/e_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/e_gpu_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/e_bench_default.json 2> gpurun_out/e_bench_default.err; echo bench rc=$?
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/e_bench_reference.json 2>&1; echo ref rc=$?
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-sweep > gpurun_out/e_bench_$c.json 2>/dev/null; echo $c rc=$?
done
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4 C1; do python tools/stage_times.py $c 10; done > gpurun_out/e_stage_times.txt 2>&1
python tools/stage_times.py C1 10 8192 >> gpurun_out/e_stage_times.txt 2>&1
python tools/c1_steady.py > gpurun_out/e_c1_steady_and_per_vector.jsonl 2>gpurun_out/e_c1.err; echo c1 rc=$?
python tools/soft_bench.py C2 273 2 > gpurun_out/e_soft_C2.json 2>/dev/null; echo soft rc=$?
python tools/soft_bench.py C5P64 64 1 > gpurun_out/e_soft_C5P64.json 2>/dev/null
python tools/soft_time.py C2 273 > gpurun_out/e_soft_kernel_times.txt 2>/dev/null
for a in "C3 273" "C4 64" "C5P64 64" "C5P256 32" "C5P1024 16"; do python tools/soft_time.py $a >> gpurun_out/e_soft_kernel_times.txt 2>/dev/null; done
(python tools/linksim_bench.py 25 mpnl; python tools/linksim_bench.py 100 mpnl; python tools/linksim_bench.py 25 mmse) > gpurun_out/e_linksim_bench.jsonl 2>/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_forms tools/probes/ffma2_forms.cu && /tmp/ffma2_forms > gpurun_out/e_ffma2_forms.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches_default.csv \
    python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
bash tools/prof_full.sh e_ncu_traverse_C5P1024 C5P1024 traverse_kernel
bash tools/prof_full.sh e_ncu_plan_C5 C5P16 plan_qr_reg
bash tools/prof_full.sh e_ncu_soft_C2 C2 soft_llr 0 soft
bash tools/prof_full.sh e_ncu_select_C5P1024 C5P1024 select_kernel
bash tools/prof_full.sh e_ncu_check_C5P1024 C5P1024 check_kernel
bash tools/prof_full.sh e_ncu_prep2_C5P16 C5P16 prep2_kernel
bash tools/prof_full.sh e_ncu_verify_C5P16 C5P16 verify_kernel
bash tools/prof_full.sh e_ncu_check_C5P16 C5P16 check_kernel
rm -f gpurun_out/e_ncu_*_sass.csv.bak
