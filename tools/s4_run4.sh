set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4d_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s4d_gpu_tests.log
for c in C5P1024 C5P256 C3; do python tools/stage_times.py $c 10; done > gpurun_out/s4d_stage_times.txt 2>&1
cat gpurun_out/s4d_stage_times.txt
python tools/profile_one.py C5P1024 0 1 > gpurun_out/s4d_stats.txt 2>&1; tail -1 gpurun_out/s4d_stats.txt
