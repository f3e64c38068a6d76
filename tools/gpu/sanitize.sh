# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_subset.py
O=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_subset.py > $O/san_$tool.log 2>&1
  echo "rc=$?" >> $O/san_$tool.log
done
