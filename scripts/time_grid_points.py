#!/usr/bin/env python
"""Kernel-only times (library events around the main kernels) of chosen grid points (debug tool for A/B
of build variants).  usage: SIGATTN_LIB=... python scripts/time_grid_points.py d:N:pad [...]"""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib  # noqa: E402

lib = _lib.load()
name = os.path.basename(os.environ.get("SIGATTN_LIB", "libsigattn.so"))
out = []
for spec in sys.argv[1:]:
    d, N, pad = spec.split(":")
    d, N, pad = int(d), int(N), float(pad)
    H = 32 if d == 64 else 16
    B = 16384 // N
    n = int(round(N * (1 - pad)))
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(4))
    lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
    fws = torch.empty(sa.fwd_workspace_bytes(B, H, N, N, d), dtype=torch.uint8, device="cuda")
    ws = torch.empty(sa.bwd_workspace_bytes(B, H, N, N, d), dtype=torch.uint8, device="cuda")
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(10)]
    for e4 in ev:
        for e in e4:
            e.record()
    for i in range(13):
        if i >= 3:
            lib.sigattn_set_profile_events(*[e.cuda_event for e in ev[i - 3]])
        sa.sigattn_fwd(q, k, v, lens, lens, out=o, workspace=fws)
        sa.sigattn_bwd(q, k, v, do, lens, lens, dq=dq, dk=dk, dv=dv, workspace=ws)
    lib.sigattn_set_profile_events(None, None, None, None)
    torch.cuda.synchronize()
    f = statistics.median(e[0].elapsed_time(e[1]) for e in ev)
    b_ = statistics.median(e[2].elapsed_time(e[3]) for e in ev)
    fl = 4.0 * B * H * n * n * d
    out.append(f"{spec}: fwd {f:.4f} ms {fl / f / 1e9:.0f} TF | bwd {b_:.4f} ms {2.5 * fl / b_ / 1e9:.0f} TF")
print(name + "\n  " + "\n  ".join(out))
