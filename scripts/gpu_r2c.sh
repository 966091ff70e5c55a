# round 2: forward limiter matrix (sigma on/off x K/V TMA on/off x one/two q tiles), C3 and N=8K unpadded
for w in c3 c2:8192:64; do
for lib in libsigattn.so libsigattn_nosig.so libsigattn_notma.so libsigattn_nosig_notma.so libsigattn_fwd2_64.so libsigattn_f2_nosig.so libsigattn_f2_notma.so libsigattn_f2_nosig_notma.so; do
  printf "%-32s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
