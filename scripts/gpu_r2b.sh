# round 2: TMEM bandwidth probe; d=64 forward one-tile vs two-tile kernel on C3
mkdir -p gpurun_out
./scripts/probes/tmem_bw > gpurun_out/r2b_tmem_bw.txt 2>&1; cat gpurun_out/r2b_tmem_bw.txt
for lib in libsigattn.so libsigattn_fwd2_64.so; do
  echo "== $lib"
  SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['fwd_kernel_ms'], d['bwd_kernel_ms'])"
done
SIGATTN_LIB=$PWD/paper_2604_27124_b200/libsigattn_fwd2_64.so timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "c1 or c3 or jag or ragged" 2>&1 | tail -3
