# per-kernel durations (ncu launch list, cold) of stage_times.py runs (3 reps each)
# usage (via gpurun): bash tools/gpu_launches_cfg.sh "C2 C4" TAG
for c in $1; do
  timeout 300 python tools/stage_times.py $c 1 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${2}_launch_$c.csv python tools/stage_times.py $c 1 > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/${2}_launch_$c.csv | head -14
done
