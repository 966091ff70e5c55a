mkdir -p gpurun_out
TAG=${1:-diag}
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-clocks > gpurun_out/bench_${TAG}_noclk.json 2> gpurun_out/bench_${TAG}_noclk.err; tail -3 gpurun_out/bench_${TAG}_noclk.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_noclk.json')); print('noclk', d['value'], d['ms_per_step'], d['fwd_kernel_ms'], d['bwd_kernel_ms'])"
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -3 gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('clk', d['value'], d['ms_per_step'], d['fwd_kernel_ms'], d['bwd_kernel_ms'], d['clocks'])"
