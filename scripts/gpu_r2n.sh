# round 2: A/B single vs two MMA issuers in the d=64 backward (interleaved), then the other workloads
for rep in 1 2; do for lib in libsigattn.so libsigattn_old1.so; do
  printf "%-22s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py c3 20 2>&1 | tail -1
  printf "%-22s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py c2:8192:64 20 2>&1 | tail -1
done; done
for w in c4 "c5 --cp fused" "c5 --cp nccl"; do
  timeout 600 python bench.py --workload $w --steps 10 > gpurun_out/r2m_tmp.json 2> gpurun_out/r2m_tmp.err || tail -5 gpurun_out/r2m_tmp.err
  python -c "import json; d=json.load(open('gpurun_out/r2m_tmp.json')); print(d['config']['workload'], round(d['value'],1), d['scaling'], 'ms', round(d['ms_per_step'],3), 'fwd', round(d['fwd_tflops'],1), 'bwd', round(d['bwd_tflops'],1))"
  cat gpurun_out/r2m_tmp.json >> gpurun_out/r2n_other.jsonl
done
bash scripts/gpu_ncu.sh r2n_c5 c5
