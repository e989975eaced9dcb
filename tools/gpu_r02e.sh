ncu --set full --clock-control none -k regex:ldpc_decode -c 1 -o gpurun_out/ncu_ldpc python tools/ldpc_bench.py --words 16384 --snr 2.5 --reps 1 --ref-words 1 > gpurun_out/ncu_ldpc.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_ldpc.log
