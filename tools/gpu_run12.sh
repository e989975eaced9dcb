for c in C3 C4 C5P256 C5P1024; do timeout 300 python tools/profile_one.py $c 64 1; done
python tools/profile_one.py C5P1024 0 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_C5P1024.csv python tools/profile_one.py C5P1024 0 1 > /dev/null 2>&1
