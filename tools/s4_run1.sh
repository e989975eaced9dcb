set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s4_gpu_tests.log
for c in C5P1024 C5P16 C2; do python tools/stage_times.py $c 10; done > gpurun_out/s4_stage_times.txt 2>&1
cat gpurun_out/s4_stage_times.txt
bash tools/prof_full.sh s4_ncu_check_C5P1024 C5P1024 check_kernel
bash tools/prof_full.sh s4_ncu_check_C5P16 C5P16 check_kernel
bash tools/prof_full.sh s4_ncu_select_C5P1024 C5P1024 select_kernel
bash tools/prof_full.sh s4_ncu_prep2_C5P16 C5P16 prep2_kernel
bash tools/prof_full.sh s4_ncu_verify_C5P16 C5P16 verify_kernel
ls -la gpurun_out | tail -30
