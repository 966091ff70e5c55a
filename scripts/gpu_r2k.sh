# round 2: d=64 backward with two MMA issuer warps: parity, timing, trace
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -q -m gpu -x 2>&1 | tail -3
for w in c3 c2:8192:64 c2:1024:64; do
for lib in libsigattn.so libsigattn_mmaonly.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
for w in c3 c2:8192; do SIGATTN_LIB=$PWD/paper_2604_27124_b200/libsigattn_trace.so timeout 120 python scripts/trace_bwd_full.py $w; done
