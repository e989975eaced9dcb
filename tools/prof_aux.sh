O=gpurun_out
python tools/profile_one.py C2 0 1 > $O/stats_C2.txt 2>&1
for k in select_kernel exact_kernel prep_kernel check_kernel verify_kernel plan_qr; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/aux_$k python tools/profile_one.py C2 0 1 > $O/ncu_aux_$k.log 2>&1; echo $k rc=$?
  python tools/ncu_summary.py full $O/aux_$k.ncu-rep > $O/aux_$k.txt
done
du -sh $O
