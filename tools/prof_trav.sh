# usage: bash tools/prof_trav.sh TAG CFG [kernel-regex]
TAG=$1; C=$2; K=${3:-traverse_kernel}
python tools/profile_one.py $C 0 1 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${TAG} python tools/profile_one.py $C 0 1 > gpurun_out/${TAG}.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py full gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}.txt
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
