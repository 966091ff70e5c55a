#!/usr/bin/env python
"""Pipeline timeline of the backward kernel from a SIGATTN_TRACE build (debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd.py
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
t = buf.view(148, 4096).cpu().numpy().reshape(148, 8, 512)
names = ["MMA_p0", "MMA_q0iss", "MMA_p1", "MMA_dQiss", "h0_sfull", "h0_parr", "h1_sfull", "h1_parr"]
for cta in (0, 77):
    r = t[cta]
    t0 = r[4, 0]
    n = int((r[0] > 0).sum())
    print(f"CTA {cta}: {n} tiles traced")
    print("  t " + " ".join("%10s" % x for x in names))
    for i in range(min(n, 16)):
        print("%3d " % i + " ".join("%10d" % (r[e, i] - t0) for e in range(8)))
    a = r[:, 4:n].astype(np.float64)
    med = lambda x: float(np.median(x))  # noqa: E731
    print("median period (WG0 sfull->sfull) %.0f" % med(np.diff(a[4])))
    print("h0 compute %.0f, h1 compute %.0f ; h0 parr->MMA p0 %.0f ; p0->q0 issued %.0f ; h1 parr->MMA p1 %.0f ;"
          " p1->dQ issued %.0f" % (med(a[5] - a[4]), med(a[7] - a[6]), med(a[0] - a[5]), med(a[1] - a[0]),
                                    med(a[2] - a[7]), med(a[3] - a[2])))
    print("h0 parr(t) -> h0 sfull(t+1) %.0f ; h1 parr(t) -> h1 sfull(t+1) %.0f"
          % (med(a[4, 1:] - a[5, :-1]), med(a[6, 1:] - a[7, :-1])))
