# round 2 evidence of the current build: GPU tests, bench (default line), ncu c3 + c5, kernel grid
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -3 gpurun_out/r2_bench.err; cut -c1-300 gpurun_out/r2_bench.json
for w in c4 "c5 --cp fused" "c5 --cp nccl"; do timeout 600 python bench.py --workload $w --steps 10 >> gpurun_out/r2_bench_other.jsonl 2>/dev/null; done
bash scripts/gpu_ncu.sh r2_c3 c3
bash scripts/gpu_ncu.sh r2_c5 c5
timeout 900 python scripts/kernel_grid.py --out gpurun_out/r2_kernel_grid.txt > /dev/null 2>&1; tail -4 gpurun_out/r2_kernel_grid.txt
