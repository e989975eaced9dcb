for c in C5P1024 C5P256 C5P64 C5P16 C2 C3 C4; do python tools/stage_times.py $c 10; done > gpurun_out/stages.txt 2>&1
cat gpurun_out/stages.txt
