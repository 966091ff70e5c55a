# round 2: bench of every workload at world 1 (c3 default line, c4 strong, c5 fused / nccl CP), ncu of c3 and c5
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2m_c3.json 2> gpurun_out/r2m_c3.err; tail -3 gpurun_out/r2m_c3.err; cut -c1-400 gpurun_out/r2m_c3.json
for w in c4 "c5 --cp fused" "c5 --cp nccl"; do
  timeout 600 python bench.py --workload $w --steps 10 > gpurun_out/r2m_tmp.json 2> gpurun_out/r2m_tmp.err || tail -5 gpurun_out/r2m_tmp.err
  python -c "import json; d=json.load(open('gpurun_out/r2m_tmp.json')); print(d['config']['workload'], round(d['value'],1), d['scaling'], 'ms', round(d['ms_per_step'],3), 'fwd', round(d['fwd_tflops'],1), 'bwd', round(d['bwd_tflops'],1))"
  cat gpurun_out/r2m_tmp.json >> gpurun_out/r2m_other.jsonl
done
bash scripts/gpu_ncu.sh r2m_c3 c3
bash scripts/gpu_ncu.sh r2m_c5 c5
