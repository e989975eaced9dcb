for c in C2 C5P64; do
python tools/profile_one.py $c 0 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python tools/profile_one.py $c 0 1 > /dev/null 2>&1
done
python tools/profile_one.py C2 64 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:traverse -c 1 -o gpurun_out/trav_c2d python tools/profile_one.py C2 64 1 > gpurun_out/ncu6.log 2>&1; tail -1 gpurun_out/ncu6.log
