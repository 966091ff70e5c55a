#!/usr/bin/env python
"""Per-compute-warp phases of the backward kernel (SIGATTN_TRACE build, debug tool)."""
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
t = buf.view(148, 4096).cpu().numpy()
names = ["c0 ld+sigma", "waits", "c0 stores", "c1 ld+sigma+STTM", "c1 STS", "-", "wait_st+fences+arrive"]
for cta in (0, 77):
    r = t[cta]
    ev = r[4 * 512:6 * 512].reshape(16, 8, 8)   # warp, tile, event
    print(f"CTA {cta}: median over tiles 2..7 of phase durations per warp: " + " | ".join(names))
    for w in range(16):
        e2 = ev[w, 2:8, :].copy()
        e2[:, 5] = e2[:, 6]   # event 5 (c1 sigma) now precedes event 4 in time; reorder 3,5,4,6
        order = [0, 1, 2, 3, 4, 6, 7]
        d = np.diff(ev[w, 2:8][:, order], axis=1)
        print(f"  warp {w:2d}: " + " ".join("%6d" % np.median(d[:, e]) for e in range(6)))
