timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/gpu_parity.log 2>&1; echo parity rc=$?
tail -3 gpurun_out/gpu_parity.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "not C5P1024" > gpurun_out/fullsize.log 2>&1; echo full rc=$?
tail -3 gpurun_out/fullsize.log
for c in C5P16 C2 C4; do python tools/stage_times.py $c 10; done
