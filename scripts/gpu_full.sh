# usage: bash scripts/gpu_full.sh TAG -- full GPU tests, smoke, default bench line, reference arm
mkdir -p gpurun_out
TAG=${1:-run}
timeout 900 python -m pytest tests/ -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; cat gpurun_out/ref_$TAG.json
