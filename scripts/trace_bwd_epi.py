#!/usr/bin/env python
"""MMA / compute / epilogue timeline of the d=64 backward, tiles 40..47 (SIGATTN_TRACE build, debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd_epi.py
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

cfg = I.C3
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
for _ in range(3):
    sa.sigattn_bwd(q, k, v, do, nq, nk, 1 / 8, -math.log(8192))
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_bwd(q, k, v, do, nq, nk, 1 / 8, -math.log(8192))
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
T = buf.view(148, 4096).cpu().numpy().astype(np.float64)
T0 = 40
for cta in (0, 77):
    r = T[cta]
    mma = r[:4 * 512].reshape(4, 512)
    cw = r[4 * 512:6 * 512].reshape(16, 8, 8)
    ep = r[3072:3072 + 8 * 16].reshape(8, 16)
    base = mma[0, T0]
    print(f"CTA {cta}: clocks relative to MMA p0ok of tile {T0}")
    print("  t | MMA p0ok S0iss p1ok dQiss | cw0 h0s h0sig h0arr h1s h1sig h1arr | EPI p0 cp0 free st0 p1 cp1 st1 | drain(t-1) dqf dqe bar done")
    for i in range(8):
        t = T0 + i
        m = mma[:, t] - base
        c = cw[0, i] - base
        e = ep[i] - base
        print("%3d | %6d %6d %6d %6d | %6d %6d %6d %6d %6d %6d | %6d %6d %6d %6d %6d %6d %6d | %6d %6d %6d %6d" % (
            t, *m, *c[:6], *e[:7], *e[7:11]))
