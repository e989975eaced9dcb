for c in C2 C3 C4 C5P16 C5P1024; do timeout 300 python tools/stage_times.py $c 10; done
bash tools/variants.sh "a pt4m3 pt4m2" "C2 C3"
bash tools/prof_trav.sh r01c_trav_C2 C2
cat gpurun_out/r01c_trav_C2.txt
