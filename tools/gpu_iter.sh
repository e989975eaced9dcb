# quick iteration on one B200: gpu tests, stage times for a few configs
# usage: bash tools/gpu_iter.sh "C2 C3 C5P16"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in ${1:-C2 C3 C5P16}; do timeout 200 python tools/stage_times.py $c 20 2>&1 | tail -1; done
