for k in 2 3 4; do SIGATTN_LIB=paper_2604_27124_b200/libsigattn_emu$k.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1; done
bash scripts/gpu_ab.sh emu2 emu3 emu4
