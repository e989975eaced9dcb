set -u
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/e_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/e_gpu_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/e_bench_default.json 2> gpurun_out/e_bench_default.err; echo bench rc=$?
tail -c 1500 gpurun_out/e_bench_default.json
