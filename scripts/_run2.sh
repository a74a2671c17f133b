timeout 100 python -m pytest tests/test_gpu_parity.py -q -x -k "fnv" 2>&1 | tail -1
timeout 200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
echo "== default"; timeout 60 python scripts/fnv_probe.py 2>&1 | grep -vE "^[0-9]+ \[|detail|np.float"
