# usage: bash tools/variants.sh "a b c" "C2 C3 C5P64"
for v in $1; do
  if [ "$v" = "a" ]; then lib=""; else lib=$PWD/paper_2409_14355_b200/_lib/libmpnl_b200_$v.so; fi
  for c in $2; do
    MPNL_LIB=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_${v}_$c.json 2> gpurun_out/var_${v}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/var_${v}_$c.json'));print('$v $c', '%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['flag_rate'])" || tail -2 gpurun_out/var_${v}_$c.err
  done
done
