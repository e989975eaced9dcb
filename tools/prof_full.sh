# Full ncu capture of one kernel of one config, with the complete raw metric page
# and the per-instruction SASS page brought back as CSV (the .ncu-rep stays on the box).
# usage: bash tools/prof_full.sh TAG CFG [kernel-regex] [n_rb] [soft]
TAG=$1; C=$2; K=${3:-traverse_kernel}; NRB=${4:-0}; X=${5:-}
python tools/profile_one.py $C $NRB 1 $X > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${TAG} python tools/profile_one.py $C $NRB 1 $X > gpurun_out/${TAG}.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py full gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}.txt
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
