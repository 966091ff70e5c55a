# round 2: single-issuer d=64 backward again; fused CP backward = local L2 sum + push kernel
timeout 900 python -m pytest tests/test_cp_fused_gpu.py tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for w in c3 c2:8192:64; do SIGATTN_LIB=$PWD/paper_2604_27124_b200/libsigattn.so timeout 120 python scripts/time_kernels.py $w 20 2>&1 | tail -1; done
for w in "c5 --cp fused" "c5 --cp nccl"; do
  timeout 600 python bench.py --workload $w --steps 10 > gpurun_out/r2m_tmp.json 2> gpurun_out/r2m_tmp.err || tail -5 gpurun_out/r2m_tmp.err
  python -c "import json; d=json.load(open('gpurun_out/r2m_tmp.json')); print(d['config']['workload'], round(d['value'],1), d['scaling'], 'ms', round(d['ms_per_step'],3), 'fwd', round(d['fwd_tflops'],1), 'bwd', round(d['bwd_tflops'],1))"
done
