#!/usr/bin/env python
"""C3 backward: fused (default) vs deterministic two-pass (Alg. 2 + Alg. 3) timing, CUDA events."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import inputs as I  # noqa: E402

cfg = I.C3 if len(sys.argv) < 2 else getattr(I, sys.argv[1])
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
flops = 10 * cfg.H * cfg.d * sum(a * b for a, b in zip(cfg.nq, cfg.nk))
for det in (False, True, False, True):
    ws = None
    for _ in range(3):
        sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=det)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=det)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{'deterministic' if det else 'fused        '} bwd {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOPS (10d credit)")
