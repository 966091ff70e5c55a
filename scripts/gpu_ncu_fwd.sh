# usage: bash scripts/gpu_ncu_fwd.sh TAG -- one ncu --set full capture (with SASS source counters) of the fwd kernel
mkdir -p gpurun_out
TAG=${1:-run}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sigattn_fwd_kernel" -s 3 -c 1 -o gpurun_out/proffwd_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_fwd_$TAG.log 2>&1; tail -2 gpurun_out/ncu_fwd_$TAG.log
