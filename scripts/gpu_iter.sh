# usage: bash scripts/gpu_iter.sh TAG -- GPU parity tests, bench line, bwd trace timeline
mkdir -p gpurun_out
TAG=${1:-run}
timeout 600 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
bash scripts/gpu_ab.sh
SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so timeout 300 python scripts/trace_bwd_timeline.py 2>&1 | head -16
