bash tools/launch_lists.sh "C5P16 C2 C5P1024"
for c in C5P16 C2 C5P1024; do echo "== $c"; python tools/launches.py gpurun_out/l_$c.csv; done > gpurun_out/launch_summary.txt
cat gpurun_out/launch_summary.txt
