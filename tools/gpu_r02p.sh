for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/profile_one.py $c 0 1 | cut -c1-400; done
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/stage_times.py $c 10; done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q > gpurun_out/p_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/p_tests.log
