SECONDS=0; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/bench4.log 2>gpurun_out/bench4.err; echo rc=$? wall=$SECONDS
tail -3 gpurun_out/bench4.err
SECONDS=0; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 4 > gpurun_out/ref4.log 2>gpurun_out/ref4.err; echo rc=$? wall=$SECONDS
