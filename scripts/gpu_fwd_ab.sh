# usage: bash scripts/gpu_fwd_ab.sh VARIANT... -- fwd TFLOPS on c2 points + c3 for default and variant libs
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L="SIGATTN_LIB=paper_2604_27124_b200/libsigattn_$v.so"; fi
  for w in c3 c2:4096:64 c2:16384:64 c2:4096:128 c2:16384:128; do
    env $L timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-clocks --steps 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-8s %-14s fwd %7.1f TF (%.3f ms)  bwd %7.1f' % ('$v', '$w', d['fwd_tflops'], d['fwd_kernel_ms'], d.get('bwd_tflops') or 0))"
  done
done
