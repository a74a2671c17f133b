export MLCK_B200_LIB=scratch_libs/tma/libmlck_b200.so
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "fnv" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 60 python scripts/fnv_probe.py 2>&1 | grep -A1 "^1024 MB"; done
