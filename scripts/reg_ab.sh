#!/bin/bash
# Development A/B: FNV register cap (variants/regNN) x async hash, N=1 step
mkdir -p gpurun_out/r2
for v in base reg80 reg72; do
  if [ "$v" != base ] && [ ! -f variants/$v/libmlck_b200.so ]; then echo "$v: not built (scripts/build_variant.sh $v -D...)"; continue; fi
  for a in 0 1; do
    if [ $v = base ]; then unset MLCK_B200_LIB; else export MLCK_B200_LIB=variants/$v/libmlck_b200.so; fi
    L=gpurun_out/r2/rab_${v}_$a.log
    timeout 300 python bench.py --no-cpu --no-log --no-extras --no-convert --steps 12 --hash-async $a > $L 2>&1
    python -c "
import json; j=json.loads(open('$L').read().strip().splitlines()[-1]); k=j['kernels']
print('$v async $a', 'step', round(j['ms_per_step'],3), 'GB/s', round(j['value'],1), 'pack', round(k['pack']['ms_avg'],3), 'fnv', round(k['fnv']['ms_avg'],3), 'parity', j['parity_trailer_ok'])" || tail -3 $L
  done
done
