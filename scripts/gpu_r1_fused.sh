# usage: bash scripts/gpu_r1_fused.sh -- parity tests for default + nodefer libs, then A/B bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
SIGATTN_LIB=paper_2604_27124_b200/libsigattn_nodefer.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
bash scripts/gpu_ab.sh nodefer nofill
bash scripts/gpu_ab.sh nodefer nofill
