timeout 500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 8 --warmup 3 --no-convert --no-cpu > gpurun_out/bench4.log 2>gpurun_out/bench4.err; echo rc=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 8 --warmup 3 --no-convert --no-cpu > gpurun_out/bench2.log 2>gpurun_out/bench2.err; echo rc=$?
timeout 300 python bench.py > gpurun_out/bench1.log 2>gpurun_out/bench1.err; echo rc=$?
