timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -2
bash scripts/gpu_ab.sh "$@"
