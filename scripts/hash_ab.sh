#!/bin/bash
# N=1 snapshot step under hash settings: async on/off x SMs left to the pack
mkdir -p gpurun_out/r2
for cfg in "0 0" "1 0" "1 16" "1 32" "1 48"; do
  set -- $cfg
  timeout 300 python bench.py --no-cpu --no-log --no-extras --no-convert --steps 12 --hash-async $1 --hash-reserve $2 > gpurun_out/r2/hab_$1_$2.log 2>&1
  python -c "
import json; j=json.loads(open('gpurun_out/r2/hab_$1_$2.log').read().strip().splitlines()[-1]); k=j['kernels']
print('async $1 reserve $2', 'step', round(j['ms_per_step'],3), 'GB/s', round(j['value'],1), 'pack', round(k['pack']['ms_avg'],3), 'fnv', round(k['fnv']['ms_avg'],3), 'parity', j['parity_trailer_ok'])"
done
