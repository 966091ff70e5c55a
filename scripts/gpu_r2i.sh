# round 2: fwd64 MMA + TMA pipeline alone (no sigma warps): all MMAs, S only, PV only, no K/V TMA
for w in c2:8192:64; do
for lib in libsigattn_mo1.so libsigattn_mo2.so libsigattn_mo3.so libsigattn_mo1nt.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
