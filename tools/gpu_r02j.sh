timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/gpu_parity.log 2>&1; echo parity rc=$?
tail -2 gpurun_out/gpu_parity.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "not C5P1024" > gpurun_out/fullsize.log 2>&1; echo full rc=$?
grep -E "vectors,|passed|failed|^E " gpurun_out/fullsize.log | head
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/stage_times.py $c 10; done
