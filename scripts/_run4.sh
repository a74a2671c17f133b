python scripts/fnv_once.py 256 > gpurun_out/once.log 2>&1 || exit 1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fnv_kernel -s 2 -c 1 -o gpurun_out/prof_fnv3 python scripts/fnv_once.py 256 > gpurun_out/ncu_fnv3.log 2>&1
echo ncu rc=$?
