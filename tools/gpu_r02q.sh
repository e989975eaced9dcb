python tools/stage_times.py C1 10 8192
python tools/stage_times.py C1 10 65536
python tools/stage_times.py C2 10 65536
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_pv.csv python tools/stage_times.py C1 1 8192 > /dev/null 2>&1
python tools/launches.py gpurun_out/q_pv.csv
