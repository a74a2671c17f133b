#!/bin/bash
# Development A/B of the fused snapshot kernel: variants/<name> builds
# (wrong bytes by design) against the product build, transport 2, N=1.
mkdir -p gpurun_out/r2
for v in base ${VARIANTS:-}; do
  if [ "$v" != base ] && [ ! -f variants/$v/libmlck_b200.so ]; then echo "$v: not built (scripts/build_variant.sh $v -D...)"; continue; fi
  if [ $v = base ]; then unset MLCK_B200_LIB; else export MLCK_B200_LIB=variants/$v/libmlck_b200.so; fi
  L=gpurun_out/r2/fv_$v.log
  timeout 300 python bench.py --no-cpu --no-log --no-extras --no-convert --no-parity --steps 12 --replica-mode 2 > $L 2>&1
  python -c "
import json; j=json.loads(open('$L').read().strip().splitlines()[-1]); k=j['kernels']
print('$v', 'step', round(j['ms_per_step'],3), 'kernel', round(k['pack_fnv']['ms_avg'],3))" || tail -3 $L
done
