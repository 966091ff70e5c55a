# round 2: fwd64 register split
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "c1 or c3 or ragged or short or pad" 2>&1 | tail -2
for w in c3 c2:8192:64; do
for lib in libsigattn.so libsigattn_r96.so libsigattn_e4.so libsigattn_f64_nosig.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
