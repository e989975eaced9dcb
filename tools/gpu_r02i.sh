ncu --set full --clock-control none -k regex:plan_qr -c 1 -o gpurun_out/ncu_plan python tools/profile_one.py C5P16 0 1 > gpurun_out/ncu_plan.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_plan.log
