mkdir -p gpurun_out/r2/san
python scripts/sanitize.py > gpurun_out/r2/san/plain.log 2>&1 || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/r2/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2/san/summary.txt
done
