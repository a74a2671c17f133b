#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench command, run under
# gpurun on ONE GPU.  Each ncu pass runs only after the same command exited 0
# without ncu.  Outputs land in gpurun_out/ (summaries are copied to profiles/).
set -u
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
echo "plain ok"
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
# full sections of the hot kernels, one launch each (after warm-up launches)
for k in fnv_kernel pack_kernel replay_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
