# round 2, first GPU call: full-oracle parity tests, whole GPU suite, TMEM bandwidth probe, bench
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
./scripts/probes/tmem_bw > gpurun_out/r2a_tmem_bw.txt 2>&1; cat gpurun_out/r2a_tmem_bw.txt
timeout 1500 python -m pytest tests/test_parity_full_gpu.py -q -m gpu -x -s 2>&1 | tail -15
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -6
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -3 gpurun_out/r2a_bench.err; cut -c1-600 gpurun_out/r2a_bench.json
