#!/usr/bin/env python
"""Joint MMA-warp / compute-warp timeline of the d=64 backward (SIGATTN_TRACE build, debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd_timeline.py
Slots: [0..4)*512 + t   MMA warp: p_full0 passed, S/dP(h0 of t+1) issued, p_full1 passed, dQ issued
       4*512 + (warp*8 + t-8)*8 + e, tiles 8..15, compute warp events:
       0 h0 s_full passed, 1 h0 sigma done, 2 h0 arrive, 3 h1 s_full passed, 4 h1 sigma done, 5 h1 arrive
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
for cta in (0, 77, 140):
    r = T[cta]
    mma = r[:4 * 512].reshape(4, 512)
    ev = r[4 * 512:6 * 512].reshape(16, 8, 8)   # warp, tile-8, event
    t0 = mma[0, 8]
    print(f"CTA {cta}  (clocks relative to MMA p_full0 of tile 8)")
    print("  t |  MMA: p0ok  S0iss  p1ok  dQiss | warp0: h0s  h0sig h0arr h1s  h1sig h1arr |"
          " warp15: h0s h0arr h1s h1arr")
    for i in range(8, 16):
        m = mma[:, i] - t0
        w0 = ev[0, i - 8] - t0
        w15 = ev[15, i - 8] - t0
        print("%3d | %6d %6d %6d %6d | %5d %5d %5d %5d %5d %5d | %5d %5d %5d %5d" % (
            i, *m, *w0[:6], w15[0], w15[2], w15[3], w15[5]))
    per = np.median(np.diff(mma[0, 8:40]))
    print("  median tile period %.0f clk" % per)
    d = lambda a, b: np.median(ev[:, :, b] - ev[:, :, a])  # noqa: E731
    print("  all-warp medians: h0 sigma %.0f, h0 st+arrive %.0f, h0->h1 s_full wait %.0f, h1 sigma %.0f, "
          "h1 st+arrive %.0f" % (d(0, 1), d(1, 2), d(2, 3), d(3, 4), d(4, 5)))
    arr0 = ev[:, :, 2].max(0); arr1 = ev[:, :, 5].max(0)
    print("  last-warp arrive -> MMA p0ok: %.0f ; -> p1ok: %.0f" % (
        np.median(mma[0, 8:16] - arr0), np.median(mma[2, 8:16] - arr1)))
    print("  MMA: p0ok->S0iss %.0f ; S0iss->p1ok %.0f ; p1ok->dQiss %.0f ; dQiss->next p0ok %.0f" % (
        np.median(mma[1, 8:40] - mma[0, 8:40]), np.median(mma[2, 8:40] - mma[1, 8:40]),
        np.median(mma[3, 8:40] - mma[2, 8:40]), np.median(mma[0, 9:41] - mma[3, 8:40])))
