# Round evidence on one B200: gpu tests, default bench (+cpu baseline), reference arm,
# per-config bench lines, launch list of the default bench, ncu --set full of the
# traversal kernel per config (dram traffic), all into gpurun_out/$TAG_*.
# usage (via gpurun): bash tools/gpu_round_evidence.sh r01
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > $O/${TAG}_bench_default.json 2> $O/${TAG}_bench_default.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err; echo ref_rc=$?
for c in C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; echo $c rc=$?
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${TAG}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${TAG}_ncu_launch.log 2>&1; echo launch_rc=$?
for c in C1 C2 C3 C4 C5P16 C5P64 C5P256 C5P1024; do
  timeout 300 python tools/profile_one.py $c 0 1 > $O/${TAG}_stats_$c.txt 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:traverse_kernel -c 1 -o $O/${TAG}_trav_$c \
    python tools/profile_one.py $c 0 1 > $O/${TAG}_ncu_$c.log 2>&1; echo ncu_$c rc=$?
done
python tools/ncu_summary.py traffic $TAG $O/profiles_$TAG > /dev/null; echo traffic_rc=$?
python tools/ncu_summary.py launches $O/${TAG}_launches_default.csv > $O/profiles_$TAG/${TAG}_launches_default.txt
for c in C1 C3 C4 C5P16 C5P64 C5P256 C5P1024; do rm -f $O/${TAG}_trav_$c.ncu-rep; done
du -sh $O
cat $O/${TAG}_bench_default.json $O/${TAG}_bench_reference.json
