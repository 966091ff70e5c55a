#!/usr/bin/env python
"""Joint timeline of the d=64 fused backward's roles for tiles 40..47 of a few CTAs (SIGATTN_TRACE build).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd_full.py [c3|c2:N]
Slots (bwd.cuh): gradient-MMA warp t: p_full0 passed, 1024+t p_full1 passed, 1536+t dQ(t) issued; score-MMA
warp 512+t S/dP(t+1,h0) issued, 3328+t S/dP(t+1,h1) issued (t < 512);
compute 2048+(warp*8+t-40)*8+e (0 S h0 seen, 1 h0 done, 2 h0 arrived, 3 S h1 seen, 4 h1 done, 5 h1 arrived);
epilogue 3072+(t-40)*16+e (0 p h0 seen, 1 h0 copied, 2 ds_free ok, 3 h0 staged, 4 p h1 seen, 5 h1 copied,
6 h1 staged, 7 dQ(t-1) full seen, 8 dQ read, 9 dQ staged, 10 reduce issued).
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = I.C3 if w == "c3" else I.c2(int(w.split(":")[1]), 64)
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / 8, -math.log(cfg.N)
for _ in range(3):
    sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
T = buf.view(148, 4096).cpu().numpy().astype(np.float64)
per = []
agg = {}
for cta in range(148):
    r = T[cta]
    if r[40] <= 0 or r[48] <= 0:
        continue
    per.append(np.median(np.diff(r[40:48])))
    for t in range(41, 47):
        base = r[t]                       # MMA p_full0 passed for tile t
        def put(name, val):
            if val > 0:
                agg.setdefault(name, []).append(val - base)
        put("MMA S/dP(t+1,h0) issued", r[512 + t])
        put("MMA p_full1 passed", r[1024 + t])
        put("MMA S/dP(t+1,h1) issued", r[3328 + t])
        put("MMA dQ issued", r[1536 + t])
        put("MMA next p_full0", r[t + 1])
        ev = r[2048:3072].reshape(16, 8, 8)[:, t - 40, :]
        for e, nm in enumerate(["S h0 seen", "h0 done", "h0 arrived", "S h1 seen", "h1 done", "h1 arrived"]):
            vals = ev[:, e]
            if (vals > 0).all():
                put("compute first " + nm, vals.min())
                put("compute last  " + nm, vals.max())
        ep = r[3072 + (t - 40) * 16: 3072 + (t - 40) * 16 + 11]
        for e, nm in enumerate(["p h0 seen", "h0 copied", "ds_free ok", "h0 staged", "p h1 seen", "h1 copied",
                                "h1 staged", "dQ(t-1) full seen", "dQ read", "dQ staged", "reduce issued"]):
            put("epi " + nm, ep[e])
print(f"{w}: median tile period (MMA p_full0 -> next) {np.median(per):.0f} clk over {len(per)} CTAs")
for k_, v_ in sorted(agg.items(), key=lambda kv: np.median(kv[1])):
    print(f"  {k_:32s} {np.median(v_):8.0f}   (p10 {np.percentile(v_, 10):7.0f}, p90 {np.percentile(v_, 90):7.0f})")
