for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc $?"; tail -4 gpurun_out/sanitize_$tool.log
done
