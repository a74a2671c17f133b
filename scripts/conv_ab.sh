#!/bin/bash
# A/B of library variants (scripts/build_variant.sh) on the conversion:
#   bash scripts/conv_ab.sh base minb8 ...   (base = the in-tree build)
mkdir -p gpurun_out/r2
for v in "$@"; do
  if [ "$v" != base ] && [ ! -f variants/$v/libmlck_b200.so ]; then echo "$v: not built (scripts/build_variant.sh $v -D...)"; continue; fi
  if [ "$v" = base ]; then unset MLCK_B200_LIB; else export MLCK_B200_LIB=variants/$v/libmlck_b200.so; fi
  timeout 300 python bench.py --no-cpu --no-log --no-extras --steps 3 > gpurun_out/r2/cab_$v.log 2>&1
  python -c "
import json; j=json.loads(open('gpurun_out/r2/cab_$v.log').read().strip().splitlines()[-1]); c=j['conversion']; k=c['kernels']
print('$v', 'conv', round(c['ms'],3), 'cold', round(c['ms_cold_records'],3), 'replay', round(k['replay']['ms_total'],3), 'witness', round(k.get('fnv_witness',{}).get('ms_total',0),3), 'step', round(j['ms_per_step'],3))"
done
