timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/bench4.log 2>gpurun_out/bench4.err; echo rc=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/bench2.log 2>gpurun_out/bench2.err; echo rc=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference > gpurun_out/ref2.log 2>gpurun_out/ref2.err; echo rc=$?
bash scripts/profile.sh
