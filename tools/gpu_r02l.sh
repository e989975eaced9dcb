ncu --set full --clock-control none -k regex:linear_detect -c 1 -o gpurun_out/ncu_lin12 python tools/linear_bench.py 12 12 16 mmse > gpurun_out/ncu_lin.log 2>&1; echo rc=$?
