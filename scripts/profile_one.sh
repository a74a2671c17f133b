#!/bin/bash
# One --set full capture of kernel $1 (regex) from the bench command, after
# the same command exited 0 without ncu (B200_PROFILING.md).  Out: gpurun_out/r2/prof_$2.ncu-rep
set -u
K=$1; NAME=$2; SKIP=${3:-2}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-extras --no-log ${EXTRA:-}"
mkdir -p gpurun_out/r2
$CMD > gpurun_out/r2/plain_$NAME.log 2>&1 || { echo "plain run failed"; tail gpurun_out/r2/plain_$NAME.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/r2/prof_$NAME $CMD > gpurun_out/r2/ncu_$NAME.log 2>&1
echo "$NAME rc=$?"
