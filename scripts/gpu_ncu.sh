# usage: bash scripts/gpu_ncu.sh TAG [WORKLOAD] -- launch list + one ncu --set full capture of the fwd and bwd
# kernels of one bench step (bench.py --workload WORKLOAD, default c3)
mkdir -p gpurun_out
TAG=${1:-run}
WL=${2:-c3}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sigattn_(fwd2?|bwd(128)?)_kernel" -s 6 -c 2 -o gpurun_out/prof_$TAG python bench.py --workload $WL --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_full_$TAG.log 2>&1; tail -2 gpurun_out/ncu_full_$TAG.log
