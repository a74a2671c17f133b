# Development: FNV throughput of scratch_libs variants (A/B), 3 alternations.
for rep in 1 2 3; do
for v in "$@"; do
  echo -n "$v: "; MLCK_B200_LIB=scratch_libs/$v/libmlck_b200.so timeout 60 python scripts/fnv_probe.py 2>&1 | grep "^1024 MB" | cut -c1-40
done; done
