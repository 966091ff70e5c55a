# usage: bash scripts/gpu_sweep.sh TAG -- fwd/bwd TFLOPS over the C2 shapes and C5 (one GPU)
mkdir -p gpurun_out
TAG=${1:-sweep}
for w in c5 c2:16384:128 c2:8192:128 c2:4096:128 c2:2048:128 c2:1024:128 c2:16384:64 c2:8192:64 c2:4096:64 c2:2048:64 c2:1024:64; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-clocks 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-14s fwd %7.1f TFLOPS (%.3f ms)  bwd %7.1f TFLOPS (%.3f ms)  fwd+bwd %7.1f' % ('$w', d['fwd_tflops'], d['fwd_kernel_ms'], d['bwd_tflops'], d['bwd_kernel_ms'], d['value']))
" | tee -a gpurun_out/sweep_$TAG.txt
done
