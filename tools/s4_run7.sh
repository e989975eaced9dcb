set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4g_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s4g_gpu_tests.log
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/stage_times.py $c 10; done
