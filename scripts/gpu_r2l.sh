# round 2: d=64 backward: compute warps split across query halves (+ two MMA issuers)
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -q -m gpu -x 2>&1 | tail -3
for w in c3 c2:8192:64 c2:1024:64; do
for lib in libsigattn.so libsigattn_spec.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
