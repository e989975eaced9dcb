timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for c in C2 C5P64; do
python tools/profile_one.py $c 0 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python tools/profile_one.py $c 0 1 > /dev/null 2>&1
done
for c in C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', '%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], '%.2g'%d['flag_rate'], d['clocks']['sm_mhz'])"
done
