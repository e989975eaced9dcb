# quick GPU check: gpu tests, per-config bench lines (no cpu baseline), guard stats
# usage (via gpurun): bash tools/gpu_quick.sh "C2 C4" [tag]
CFGS=${1:-"C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024"}
TAG=${2:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in $CFGS; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_$c.json'));r=d['roofline'];print('$c', '%.4g'%d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['flag_rate'], '%.4g'%d['e2e']['value'])" || tail -3 gpurun_out/${TAG}_$c.err
  timeout 300 python tools/profile_one.py $c 0 1 2>&1 | tail -1
done
