set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "C1 or C2 or C3 or C4 or C5P16 or C5P64" -s > gpurun_out/fullsize.log 2>&1; echo fullsize rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/fullsize.log; cat gpurun_out/bench.log
