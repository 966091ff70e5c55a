# round 2: new d=64 forward (fwd64.cuh): parity, then timing vs EMU fractions
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_full_gpu.py -q -m gpu -x 2>&1 | tail -4
for w in c3 c2:8192:64 c2:1024:64; do
for lib in libsigattn.so libsigattn_e2.so libsigattn_e3.so libsigattn_e4.so libsigattn_e6.so libsigattn_f64_nosig.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
