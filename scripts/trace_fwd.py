#!/usr/bin/env python
"""Pipeline timeline of the forward kernel from a SIGATTN_TRACE build (debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_fwd.py
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
    sa.sigattn_fwd(q, k, v, nq, nk, 1 / 8, -math.log(8192))
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_fwd(q, k, v, nq, nk, 1 / 8, -math.log(8192))
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
t = buf.view(148, 4096).cpu().numpy()
for cta in (0, 77):
    r = t[cta]
    t0 = r[512]
    n = int((r[512:1024] > 0).sum())
    print(f"CTA {cta}: {n} S tiles traced")
    rows = []
    for si in range(min(n, 512)):
        s_iss, pf, pv = r[512 + si], r[1024 + si], r[1536 + si]
        wg_s, wg_p, wg_plast = r[2048 + si], r[2560 + si], r[3072 + si]
        rows.append((si, s_iss - t0, wg_s - t0, wg_p - t0, wg_plast - t0, pf - t0, pv - t0))
    print(" si   S_issue  WG4_sfull  WG4_parr  WGlast_parr  MMA_pfull  PV_issue")
    for x in rows[:24]:
        print("%3d " % x[0] + " ".join("%10d" % y for y in x[1:]))
    a = np.array(rows[4:], dtype=np.float64)
    if len(a) > 4:
        d = lambda i, j: np.median(a[:, j] - a[:, i])  # noqa: E731
        print("median: S_issue->WG sfull %.0f | WG sigma (sfull->parr) %.0f | parr first->last WG %.0f | "
              "last parr->MMA pfull %.0f | pfull->PV issued %.0f" % (d(1, 2), d(2, 3), d(3, 4), d(4, 5), d(5, 6)))
        per_tile = np.median(np.diff(a[:, 2]))
        print("median period between consecutive WG s_full: %.0f clk" % per_tile)
