for c in C5P1024 C5P256 C5P64 C5P16 C4; do python tools/stage_times.py $c 8; done
echo "--- minb3"
for c in C5P1024 C5P256 C5P64 C5P16 C4; do MPNL_LIB=paper_2409_14355_b200/_lib/libmpnl_b200_minb3.so python tools/stage_times.py $c 8; done
