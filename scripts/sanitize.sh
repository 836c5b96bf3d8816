# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_case.py (one GPU).
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/r02_sanitize_$tool.log \
    python scripts/sanitize_case.py > gpurun_out/r02_sanitize_${tool}_stdout.log 2>&1
  echo "$tool rc=$?"
  tail -3 gpurun_out/r02_sanitize_$tool.log
done
