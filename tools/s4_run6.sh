set -u
export MPNL_LIB=$PWD/paper_2409_14355_b200/_lib/libmpnl_b200_sk2.so
python tools/stage_times.py C5P1024 10
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_soft.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -3
python tools/profile_one.py C5P1024 0 1 2>&1 | tail -1
