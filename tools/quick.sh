timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
  python -c "import json;d=json.load(open('gpurun_out/q_$c.json'));print('$c', '%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['flag_rate'])" || tail -3 gpurun_out/q_$c.err
done
