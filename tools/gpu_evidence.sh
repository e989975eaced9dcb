# round evidence: default bench (+cpu baseline), reference arm, launch list, ncu full of the hot kernel
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
python tools/profile_one.py C2 0 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:traverse -c 1 -o gpurun_out/traverse_C2_full python tools/profile_one.py C2 0 1 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
cat gpurun_out/bench_default.json gpurun_out/bench_reference.json
