# probes (TMEM bandwidth, cta_group::2 MMA rate, chunk path with FMA-pipe exp2) + A/B of the direct dS staging
mkdir -p gpurun_out
( cd scripts/probes && for p in tmem_bw mma2sm_probe chunk_probe; do echo "== $p"; timeout 120 ./$p; done ) > gpurun_out/r2q_probes.txt 2>&1
cat gpurun_out/r2q_probes.txt
for lib in libsigattn.so libsigattn_dsold.so libsigattn.so libsigattn_dsold.so; do
  for w in c3 c2:8192:64; do echo -n "$lib "; SIGATTN_LIB=$PWD/paper_2604_27124_b200/$lib timeout 120 python scripts/time_kernels.py $w 20 2>&1 | tail -1; done
done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
