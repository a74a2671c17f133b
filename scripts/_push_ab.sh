for v in "$@"; do
  MLCK_B200_LIB=scratch_libs/$v/libmlck_b200.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 8 --warmup 3 --no-cpu --no-log --no-convert > gpurun_out/pab_$v.log 2>&1
  python -c "
import json; j=json.loads(open('gpurun_out/pab_$v.log').read().strip().splitlines()[-1]); print('$v', round(j['value'],1), round(j['ms_per_step'],3))"
done
