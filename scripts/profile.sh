#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench command, run under
# gpurun on ONE GPU.  Each ncu pass runs only after the same command exited 0
# without ncu.  Outputs land in gpurun_out/$R (summaries: NCU_OUT=gpurun_out/$R
# python scripts/summarize_ncu.py $R -> profiles/).
set -u
R=${1:-r02}
O=gpurun_out/$R
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-extras"
mkdir -p $O
$CMD > $O/plain.log 2>&1 || { echo "plain run failed"; tail $O/plain.log; exit 1; }
echo "plain ok"
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
# full sections of the hot kernels, one launch each (after warm-up launches)
for k in fnv_kernel pack_kernel replay_kernel fnv_witness_tc_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/prof_$k $CMD > $O/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
