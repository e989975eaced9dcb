timeout 900 python -m pytest tests/test_linear.py tests/test_slot.py tests/test_gpu_api.py -q > gpurun_out/lin.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/lin.log; grep -E "^E |FAILED" gpurun_out/lin.log | head
for a in "12 12 16 mmse" "12 12 16 zf" "4 4 64 mmse" "2 2 4 mmse" "16 16 64 mmse" "8 8 16 mmse" "24 24 64 mmse 344064" "32 32 16 mmse 45864"; do python tools/linear_bench.py $a; done > gpurun_out/linear_bench.jsonl 2>&1
cat gpurun_out/linear_bench.jsonl
