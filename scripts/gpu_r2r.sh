# round 2 (session 3) check of the current build: GPU suite, sanitizers (small + many-item shapes), C3 kernels, bench
mkdir -p gpurun_out/r2r
timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/r2r/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/r2r/sanitize_$tool.log
done
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py --many > gpurun_out/r2r/sanitize_${tool}_many.log 2>&1
  echo "$tool many rc=$?"; tail -2 gpurun_out/r2r/sanitize_${tool}_many.log
done
for i in 1 2; do python scripts/time_kernels.py c3 20 | tail -1; done
timeout 600 python bench.py > gpurun_out/r2r/bench.json 2> gpurun_out/r2r/bench.err; tail -3 gpurun_out/r2r/bench.err; cut -c1-250 gpurun_out/r2r/bench.json
