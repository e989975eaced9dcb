timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -k "C4" > gpurun_out/fullsize.log 2>&1; echo fullsize rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/gpu_parity.log 2>&1; echo parity rc=$?
grep -E "vectors|Error|passed|failed" gpurun_out/fullsize.log gpurun_out/gpu_parity.log
