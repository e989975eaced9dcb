# usage: bash tools/launch_lists.sh "C2 C5P1024" -> gpurun_out/l_<cfg>.csv + stats
for c in $1; do
  timeout 300 python tools/profile_one.py $c 0 1 > gpurun_out/stats_$c.txt 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$c.csv python tools/profile_one.py $c 0 1 > /dev/null 2>&1
  tail -1 gpurun_out/stats_$c.txt
done
