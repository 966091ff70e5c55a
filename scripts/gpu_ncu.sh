# usage: bash scripts/gpu_ncu.sh TAG  -- launch list + one ncu --set full capture of the fwd and bwd kernels (C3 bench step)
mkdir -p gpurun_out
TAG=${1:-run}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sigattn_(fwd|bwd)_kernel" -s 6 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_full_$TAG.log 2>&1; tail -2 gpurun_out/ncu_full_$TAG.log
