# round 2 evidence of the current build: GPU tests, bench (default line), ncu c3 + c5, kernel grid
# usage: bash scripts/gpu_r2_evidence.sh TAG
T=${1:-r2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -3 gpurun_out/${T}_bench.err; cut -c1-300 gpurun_out/${T}_bench.json
for w in c4 "c5 --cp fused" "c5 --cp nccl"; do timeout 600 python bench.py --workload $w --steps 10 >> gpurun_out/${T}_bench_other.jsonl 2>/dev/null; done
bash scripts/gpu_ncu.sh ${T}_c3 c3
bash scripts/gpu_ncu.sh ${T}_c5 c5
timeout 900 python scripts/kernel_grid.py --out gpurun_out/${T}_kernel_grid.txt > /dev/null 2>&1; tail -4 gpurun_out/${T}_kernel_grid.txt
