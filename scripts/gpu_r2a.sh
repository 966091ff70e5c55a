# round 2, first GPU call: full-oracle parity tests, whole GPU suite, smoke, bench
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_parity_full_gpu.py -q -m gpu -x -s 2>&1 | tail -25
timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -3 gpurun_out/r2a_bench.err; cut -c1-900 gpurun_out/r2a_bench.json
