mkdir -p gpurun_out
set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k c3 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; tail -5 gpurun_out/bench_r1.err; cat gpurun_out/bench_r1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1; wc -l gpurun_out/launches_r1.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sigattn_(fwd|bwd)_kernel" -s 6 -c 2 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_full_r1.log 2>&1; tail -3 gpurun_out/ncu_full_r1.log
