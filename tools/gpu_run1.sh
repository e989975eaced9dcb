set -x
timeout 900 python -m pytest tests -x -q -m gpu -rA 2>&1 | grep -E "passed|failed|flagged|Error|error" | tail -30
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
for c in C1 C3 C4 C5P16 C5P64 C5P256 C5P1024; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['flag_rate'], d['e2e']['value'], d['clocks'])"
done
