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
for cta in (0, 77):
    r = t[cta]
    ev = r[4 * 512:6 * 512].reshape(16, 8, 8).astype(np.float64)   # warp, tile (8..15), event
    t0 = ev[0, 0, 0]
    print(f"CTA {cta}: per warp median over 8 tiles: h0[ld+compute, STTM+STS+wait_st, fences+arrive] |"
          f" h1 [s_full wait+ld+compute, STTM, STS+wait_st, fences+arrive]")
    for w in range(16):
        e = ev[w]
        m = lambda a, b: np.median(e[:, b] - e[:, a])  # noqa: E731
        print(f"  warp {w:2d}: h0 {m(0,1):5.0f} {m(1,2):5.0f} {m(2,3):5.0f} | h1 {m(3,4):5.0f} {m(4,5):5.0f} {m(5,6):5.0f} "
              f"{m(6,7):5.0f} | next h0 wait {np.median(e[1:, 0] - e[:-1, 7]):5.0f}")
