python tools/soft_bench.py C2 273 2 > gpurun_out/soft_C2.json 2>&1; echo soft rc=$?
python tools/soft_bench.py C5P64 256 1 > gpurun_out/soft_C5P64.json 2>&1; echo soft2 rc=$?
python tools/c1_steady.py 256 8192 > gpurun_out/c1_steady.jsonl 2>&1; echo c1 rc=$?
cat gpurun_out/soft_C2.json gpurun_out/soft_C5P64.json gpurun_out/c1_steady.jsonl
