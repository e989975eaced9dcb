for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/stage_times.py $c 8; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_edges.py -q > gpurun_out/x_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/x_tests.log
