# compute-sanitizer on the small end-to-end workload (every hot kernel).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py 3 \
    > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
  tail -n 6 gpurun_out/san_$tool.log
done
