# ncu --set full capture (SASS source counters) of the d=64 backward kernel on C3 (bench launch config)
mkdir -p gpurun_out
TAG=${1:-run}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sigattn_bwd_kernel" -s 3 -c 1 -o gpurun_out/prof_bwd_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_bwd_$TAG.log 2>&1; tail -2 gpurun_out/ncu_bwd_$TAG.log
