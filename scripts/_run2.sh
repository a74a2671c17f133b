timeout 200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for v in default k3w16 k3w18 k2w26; do
  w=${v#*w}; [ $v = default ] && w=14
  L=$PWD/scratch_libs/$v/libmlck_b200.so; [ $v = default ] && L=""
  echo "== $v"; MLCK_B200_LIB=$L FNV_CHUNK=$(( w * 32 * 128 )) timeout 60 python scripts/fnv_probe.py 2>&1 | grep -E "MB|wait median"
  MLCK_B200_LIB=$L timeout 100 python -m pytest tests/test_gpu_parity.py -q -x -k fnv 2>&1 | tail -1
done
