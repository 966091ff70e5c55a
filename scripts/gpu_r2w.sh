# final evidence without the C3 ncu capture (unchanged kernels; keeps gpurun_out under the copy-back limit)
T=${1:-r2w}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -3 gpurun_out/${T}_bench.err; cut -c1-200 gpurun_out/${T}_bench.json
for w in c4 "c5 --cp fused" "c5 --cp nccl"; do timeout 600 python bench.py --workload $w --steps 10 >> gpurun_out/${T}_bench_other.jsonl 2>/dev/null; done
bash scripts/gpu_ncu.sh ${T}_c5 c5
timeout 900 python scripts/kernel_grid.py --out gpurun_out/${T}_kernel_grid.txt > /dev/null 2>&1; tail -4 gpurun_out/${T}_kernel_grid.txt
du -sh gpurun_out
