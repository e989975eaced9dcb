timeout 900 python -m pytest tests/test_llr.py tests/test_gpu_api.py -q > gpurun_out/t_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_tests.log; grep -E "^E |FAILED" gpurun_out/t_tests.log | head -5
python tools/llr_bench.py 45864 64 12 16
python tools/llr_bench.py 45864 256 32 16
python tools/llr_bench.py 45864 64 24 64
python tools/soft_bench.py C2 273 2
ncu --set full --clock-control none -k regex:traverse_kernel -c 1 -o gpurun_out/t_trav_C2 python tools/profile_one.py C2 0 1 > /dev/null 2>&1; echo ncu rc=$?
