#!/usr/bin/env python
"""Kernel grid points timed three ways (debug tool): per call wall time on the GPU (CUDA events around a
loop of public-API calls, as scripts/kernel_grid.py), the library's events around the main kernel only,
and a CUDA graph of the public call (no host overhead).

usage (GPU box): python scripts/grid_split.py [d ...]
"""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib  # noqa: E402

lib = _lib.load()


def loop_ms(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def kern_ms(fn, fwd, iters=10):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(iters)]
    for e2 in ev:   # torch creates the CUDA events lazily, on the first record
        for e in e2:
            e.record()
    for e in ev:
        if fwd:
            lib.sigattn_set_profile_events(e[0].cuda_event, e[1].cuda_event, None, None)
        else:
            lib.sigattn_set_profile_events(None, None, e[0].cuda_event, e[1].cuda_event)
        fn()
    lib.sigattn_set_profile_events(None, None, None, None)
    torch.cuda.synchronize()
    return statistics.median(e[0].elapsed_time(e[1]) for e in ev)


def graph_ms(fn, iters=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return loop_ms(g.replay, iters)


ds = [int(x) for x in sys.argv[1:]] or [64, 128]
print("d    N      pad | fwd: loop  kernel  graph (ms) | bwd: loop  kernel  graph (ms)")
for d in ds:
    H = 32 if d == 64 else 16
    for N in (512, 1024, 2048, 4096, 8192):
        B = 16384 // N
        for pad in (0.0, 0.25):
            n = int(round(N * (1 - pad)))
            q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
            lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
            bias = torch.full((B,), -math.log(n), dtype=torch.float32, device="cuda")
            fws = torch.empty(sa.fwd_workspace_bytes(B, H, N, N, d), dtype=torch.uint8, device="cuda")
            ws = torch.empty(sa.bwd_workspace_bytes(B, H, N, N, d), dtype=torch.uint8, device="cuda")
            o = torch.empty_like(q)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            f = lambda: sa.sigattn_fwd(q, k, v, lens, lens, bias=bias, out=o, workspace=fws)  # noqa: E731
            g = lambda: sa.sigattn_bwd(q, k, v, do, lens, lens, bias=bias, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa: E731
            r = [loop_ms(f), kern_ms(f, True), graph_ms(f), loop_ms(g), kern_ms(g, False), graph_ms(g)]
            print("%-4d %-6d %3d%% | %9.3f %7.3f %6.3f      | %9.3f %7.3f %6.3f" % (d, N, int(pad * 100), *r), flush=True)
