set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4i_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s4i_gpu_tests.log
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4 C1; do python tools/stage_times.py $c 10; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
