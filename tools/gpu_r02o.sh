timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/o_api.log 2>&1; echo api rc=$?; tail -1 gpurun_out/o_api.log
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-sweep > gpurun_out/o_bench_$c.json 2>gpurun_out/o_bench_$c.err; echo $c rc=$?; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/o_bench_reference.json 2>&1; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/o_launches_default.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
ncu --set full --clock-control none -k regex:traverse_kernel -c 1 -o gpurun_out/o_trav_C5P1024 python tools/profile_one.py C5P1024 0 1 > /dev/null 2>&1; echo ncu2 rc=$?
cat gpurun_out/o_bench_*.json | cut -c1-400
