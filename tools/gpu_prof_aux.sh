# ncu --set full of the auxiliary kernels of one config: bash tools/gpu_prof_aux.sh TAG CFG "prep_kernel select_kernel check_kernel"
TAG=$1; C=$2
python tools/profile_one.py $C 0 1 > /dev/null 2>&1
for k in $3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_$k python tools/profile_one.py $C 0 1 > gpurun_out/${TAG}_$k.log 2>&1; echo ncu $k rc=$?
  python tools/ncu_summary.py full gpurun_out/${TAG}_$k.ncu-rep > gpurun_out/${TAG}_$k.txt
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_${k}_sass.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_$k.ncu-rep; cat gpurun_out/${TAG}_$k.txt
done
