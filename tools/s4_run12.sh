set -u
export MPNL_LIB=$PWD/paper_2409_14355_b200/_lib/libmpnl_b200_xt.so
for c in C5P1024 C5P256 C5P64 C3 C4; do python tools/stage_times.py $c 10; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -3
