# session-4 check: GPU suite + stage split + event statistics after the flush-time event filter
set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4b_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s4b_gpu_tests.log
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4 C1; do python tools/stage_times.py $c 10; done > gpurun_out/s4b_stage_times.txt 2>&1
cat gpurun_out/s4b_stage_times.txt
for c in C5P1024 C5P256 C4 C3 C2; do python tools/profile_one.py $c 0 1; done > gpurun_out/s4b_stats.txt 2>&1
cat gpurun_out/s4b_stats.txt
