timeout 900 python -m pytest tests/test_gpu_fec.py -q -x > gpurun_out/gpu_fec.log 2>&1; echo fec rc=$?
tail -30 gpurun_out/gpu_fec.log
timeout 600 python tools/ldpc_bench.py > gpurun_out/ldpc_bench.jsonl 2>&1; echo bench rc=$?
cat gpurun_out/ldpc_bench.jsonl
