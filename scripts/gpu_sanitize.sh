# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py (small shapes)
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; tail -6 gpurun_out/sanitize_$tool.log
done
