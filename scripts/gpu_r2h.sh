# round 2: fwd64 -- does mbarrier polling by the sigma warps slow the tensor pipe?
for w in c2:8192:64; do
for lib in libsigattn_f64_nosig.so libsigattn_sl_nosig.so libsigattn_nt_nosig.so libsigattn.so libsigattn_sl.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
SIGATTN_LIB=$PWD/paper_2604_27124_b200/libsigattn_tr_sl_nosig.so timeout 120 python scripts/trace_fwd64.py c2:8192:64 2>&1 | tail -9
