python bench.py --steps 2 --warmup 3 --no-cpu --no-log --no-convert --no-parity > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fnv_kernel -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 2 --warmup 3 --no-cpu --no-log --no-convert --no-parity > gpurun_out/ncu_fused.log 2>&1
echo ncu rc=$?
