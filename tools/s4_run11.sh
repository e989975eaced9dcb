set -u
export MPNL_LIB=$PWD/paper_2409_14355_b200/_lib/libmpnl_b200_xs.so
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4 C1; do python tools/stage_times.py $c 10; done
