#!/usr/bin/env python
"""Backward timing: fused (default) vs deterministic two-pass (Alg. 2 + Alg. 3), CUDA events.

usage: python scripts/time_bwd_modes.py [C3|c5]   (prints whole-call time and the main
dK/dV kernel's own time from the library's profile events)
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

cfg = I.C3 if len(sys.argv) < 2 else (I.c5(16, 128) if sys.argv[1] == "c5" else getattr(I, sys.argv[1]))
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
flops = 10 * cfg.H * cfg.d * sum(a * b for a, b in zip(cfg.nq, cfg.nk))
lib = _lib.load()
for det in (False, True, False, True):
    for _ in range(3):
        sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=det)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    k1.record()   # torch only times events it has recorded once; the library re-records them
    kern = 0.0
    e0.record()
    for _ in range(10):
        lib.sigattn_set_profile_events(None, None, ctypes.c_void_p(k0.cuda_event), ctypes.c_void_p(k1.cuda_event))
        sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=det)
        lib.sigattn_set_profile_events(None, None, None, None)
        k1.synchronize()
        kern += k0.elapsed_time(k1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{'deterministic' if det else 'fused        '} bwd {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOPS (10d credit);"
          f" main (dK/dV) kernel {kern / 10:.3f} ms")
