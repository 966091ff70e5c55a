# usage: bash scripts/gpu_ab.sh VARIANT...  -- C3 bench line for the default lib and each libsigattn_<VARIANT>.so
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L="SIGATTN_LIB=paper_2604_27124_b200/libsigattn_$v.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-clocks --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-10s value %6.1f  fwd %6.1f (%.3f ms)  bwd %6.1f (%.3f ms)  step %.3f ms' % ('$v', d['value'], d['fwd_tflops'], d['fwd_kernel_ms'], d['bwd_tflops'], d['bwd_kernel_ms'], d['ms_per_step']))"
done
