#!/bin/bash
# Development: fused-snapshot (transport 2) and TMA-store (transport 5)
# parity, then the N=1 step under transports 0 / 2 / 5.
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "snapshot" > gpurun_out/r2/fab_tests.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r2/fab_tests.log
timeout 600 python -m pytest tests/test_gpu_witness.py -x -q > gpurun_out/r2/fab_wit.log 2>&1
echo "witness rc=$?"; tail -2 gpurun_out/r2/fab_wit.log
for m in ${MODES:-0 2 5}; do
  L=gpurun_out/r2/fab_$m.log
  timeout 300 python bench.py --no-cpu --no-log --no-extras --no-convert --steps 12 --replica-mode $m > $L 2>&1
  python -c "
import json; j=json.loads(open('$L').read().strip().splitlines()[-1])
print('mode $m', 'step', round(j['ms_per_step'],3), 'GB/s', round(j['value'],1), 'parity', j['parity_trailer_ok'])" || tail -5 $L
done
