#!/bin/bash
# Development: the tcgen05 witness verifier -- parity (witness, conversion,
# localized recovery) and the conversion A/B against the mma.sync verifier.
mkdir -p gpurun_out/r2
timeout 300 python -m pytest tests/test_gpu_witness.py -x -q > gpurun_out/r2/tc_wit.log 2>&1
echo "witness rc=$?"; tail -3 gpurun_out/r2/tc_wit.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -x -q -k "conver or recover or parse" > gpurun_out/r2/tc_par.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/r2/tc_par.log
bash scripts/conv_ab.sh base notc base notc
