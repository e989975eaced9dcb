#!/bin/bash
# A/B of a compile-time variant without a full rebuild: compile only the named csrc units
# with extra flags and link them with the base build's other objects.
# usage: bash tools/variant_unit.sh NAME "FLAGS" unit [unit ...]   (unit = file stem under csrc/)
#   -> paper_2409_14355_b200/_lib/libmpnl_b200_NAME.so   (load it with MPNL_LIB=<path>)
set -e
NAME=$1; FLAGS=$2; shift 2
cd "$(dirname "$0")/.."
OD=build/obj_$NAME; mkdir -p $OD
for u in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include $FLAGS \
       -c paper_2409_14355_b200/csrc/$u.cu -o $OD/$u.o &
done
wait
objs=""
for o in build/obj/*.o; do b=$(basename $o); if [ -f $OD/$b ]; then objs="$objs $OD/$b"; else objs="$objs $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2409_14355_b200/_lib/libmpnl_b200_$NAME.so $objs
ls -la paper_2409_14355_b200/_lib/libmpnl_b200_$NAME.so
