timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024; do timeout 300 python tools/profile_one.py $c 64 2; done
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
python -c "import json;d=json.load(open('gpurun_out/bench_C2.json'));print('C2', d['value'], d['ms_per_step'], d['roofline'], d['flag_rate'])"
python tools/profile_one.py C2 64 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:traverse -c 1 -o gpurun_out/trav_c2b python tools/profile_one.py C2 64 1 > gpurun_out/ncu3.log 2>&1; tail -1 gpurun_out/ncu3.log
