mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool exit=$?" >> gpurun_out/sanitizer_$tool.log
  tail -5 gpurun_out/sanitizer_$tool.log
done
