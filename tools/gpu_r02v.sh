timeout 1200 python -m pytest tests/test_gpu_linksim.py tests/test_slot.py -q > gpurun_out/v_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/v_tests.log; grep -E "^E |FAILED" gpurun_out/v_tests.log | head -8
python tools/linksim_bench.py 25 mpnl 4 8 2
python tools/linksim_bench.py 25 mmse 4 8 2
python tools/linksim_bench.py 100 mpnl 4 8 2
