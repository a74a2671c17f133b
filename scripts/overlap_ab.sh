#!/bin/bash
# conversion: witnessed verification beside the replay on N SMs (0 = sequential)
mkdir -p gpurun_out/r2
for n in ${OVERLAPS:-0 24 37 48 74}; do
  timeout 300 python bench.py --no-cpu --no-log --no-extras --steps 3 --convert-overlap $n > gpurun_out/r2/oab_$n.log 2>&1
  python -c "
import json; j=json.loads(open('gpurun_out/r2/oab_$n.log').read().strip().splitlines()[-1]); c=j['conversion']; k=c['kernels']
print('overlap $n', 'conv', round(c['ms'],3), 'replay', round(k['replay']['ms_total'],3), 'witness', round(k.get('fnv_witness',{}).get('ms_total',0),3), 'loc', round(c['localized_recovery']['ms'],3))"
done
