# round 2: fwd64 with separate S / PV issuer warps
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for w in c2:8192:64 c3; do
for lib in libsigattn_f64_nosig.so libsigattn.so libsigattn_e3.so libsigattn_e4.so libsigattn_e5.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
SIGATTN_LIB=$PWD/paper_2604_27124_b200/libsigattn_trace.so timeout 120 python scripts/trace_fwd64.py c2:8192:64 2>&1 | tail -10
