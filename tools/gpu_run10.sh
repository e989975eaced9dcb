for c in C2 C4; do
python tools/profile_one.py $c 128 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:traverse -c 1 -o gpurun_out/trav_${c}_e python tools/profile_one.py $c 128 1 > gpurun_out/ncu10.log 2>&1; tail -1 gpurun_out/ncu10.log
done
