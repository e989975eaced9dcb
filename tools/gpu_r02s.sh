timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/s_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s_tests.log; grep -E "^E |FAILED" gpurun_out/s_tests.log | head -5
for c in C2 C3 C1; do python tools/stage_times.py $c 10; done
python tools/stage_times.py C1 10 8192
python tools/stage_times.py C1 10 65536
python tools/c1_steady.py 256 8192
