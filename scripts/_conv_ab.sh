for v in "$@"; do
  MLCK_B200_LIB=scratch_libs/$v/libmlck_b200.so timeout 300 python bench.py --no-cpu --no-log --steps 3 > gpurun_out/cab_$v.log 2>&1
  python -c "
import json; j=json.loads(open('gpurun_out/cab_$v.log').read().strip().splitlines()[-1]); c=j['conversion']; print('$v', round(c['ms'],2), round(c['kernels']['replay']['ms_total'],3))"
done
