for v in default s8; do
  L=$PWD/scratch_libs/$v/libmlck_b200.so; [ $v = default ] && L=""
  echo "== $v"; MLCK_B200_LIB=$L timeout 60 python scripts/fnv_probe.py 2>&1 | grep -E "MB|wait median"
done
