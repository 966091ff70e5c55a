# round 2: fwd64 pipeline trace
for w in c2:8192:64 c3; do
for lib in libsigattn_trace.so libsigattn_trace_nosig.so; do
  echo "== $lib $w"; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/trace_fwd64.py $w 2>&1 | tail -10
done; done
