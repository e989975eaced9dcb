#!/bin/bash
# build locally (abort on failure), then run the given command on the GPU box
# usage: bash tools/bgpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python -c "from paper_2409_14355_b200.build import build; print(build())" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; echo BUILD FAILED; exit 1; }
test -f paper_2409_14355_b200/_lib/libmpnl_b200.so || { echo NO LIB; exit 1; }
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
