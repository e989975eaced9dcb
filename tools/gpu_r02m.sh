python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m_gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/m_gpu_tests.log
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo bench rc=$?
cat gpurun_out/m_bench.json
