python tools/diag_rb.py C4 60 > gpurun_out/diag_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -k "not C5P1024" > gpurun_out/fullsize.log 2>&1; echo fullsize rc=$?
cat gpurun_out/diag_c4.log; grep -E "vectors|Error|passed|failed" gpurun_out/fullsize.log
