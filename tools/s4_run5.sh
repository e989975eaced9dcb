set -u
python tools/stage_times.py C5P1024 10
MPNL_LIB=$PWD/paper_2409_14355_b200/_lib/libmpnl_b200_mb12.so python tools/stage_times.py C5P1024 10
bash tools/prof_full.sh s4e_ncu_select_C5P1024 C5P1024 select_kernel
cat gpurun_out/s4e_ncu_select_C5P1024.txt
