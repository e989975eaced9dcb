python tools/soft_bench.py C2 273 2
python tools/soft_bench.py C3 64 1
for c in C2 C3 C1; do python tools/stage_times.py $c 10; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_llr.py -q -x 2>&1 | tail -2
