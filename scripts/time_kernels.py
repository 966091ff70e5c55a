#!/usr/bin/env python
"""Per-kernel timing (fwd kernel, bwd kernel) of one library build on a workload, CUDA events
recorded by the library around its main kernels (debug tool for A/B of build variants).

usage: SIGATTN_LIB=... python scripts/time_kernels.py [c3 | c5 | c2:N:d] [reps]
prints: <fwd kernel ms> <fwd TFLOPS> <bwd kernel ms> <bwd TFLOPS>
"""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if w == "c3":
    cfg = I.C3
elif w == "c5":
    cfg = I.c5(16, 128)
else:
    _, n_, d_ = w.split(":")
    cfg = I.c2(int(n_), int(d_))
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / math.sqrt(cfg.d), -math.log(cfg.N)
fws = torch.empty(sa.fwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dtype=torch.uint8, device="cuda")
ws = torch.empty(sa.bwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dtype=torch.uint8, device="cuda")
o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
lib = _lib.load()
pairs = sum(a * c for a, c in zip(cfg.nq, cfg.nk)) * cfg.H
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
for e4 in ev:
    for e in e4:
        e.record()
for i in range(3 + reps):
    if i >= 3:
        lib.sigattn_set_profile_events(*[e.cuda_event for e in ev[i - 3]])
    sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=o, workspace=fws)
    sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, dq=dq, dk=dk, dv=dv, workspace=ws)
lib.sigattn_set_profile_events(None, None, None, None)
torch.cuda.synchronize()
f = statistics.median(e[0].elapsed_time(e[1]) for e in ev)
g = statistics.median(e[2].elapsed_time(e[3]) for e in ev)
print(f"{w} fwd {f:.4f} ms {4 * cfg.d * pairs / f / 1e9:.1f} TF | bwd {g:.4f} ms {10 * cfg.d * pairs / g / 1e9:.1f} TF")
