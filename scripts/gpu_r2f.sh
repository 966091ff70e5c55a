# round 2: fwd64 skeleton hypotheses (cross-item lookahead, MMA spin)
for w in c3 c2:8192:64; do
for lib in libsigattn_f64_nosig.so libsigattn_nx_nosig.so libsigattn_spin_nosig.so libsigattn_f2_nosig.so libsigattn.so libsigattn_nx.so libsigattn_spin.so; do
  printf "%-28s " $lib; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 2>&1 | tail -1
done; done
