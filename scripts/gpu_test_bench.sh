# usage: bash scripts/gpu_test_bench.sh TAG   -- GPU parity tests + one bench line
mkdir -p gpurun_out
TAG=${1:-run}
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --cpu-seconds 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','pct_of_peak','fwd_tflops','bwd_tflops','fwd_kernel_ms','bwd_kernel_ms','ms_per_step','gpu_launches_per_step']}); print(d['clocks'])"
