#!/usr/bin/env python
"""Pipeline timeline of the forward kernel from a SIGATTN_TRACE build (debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_fwd.py [workload]

Trace slots per CTA (clock64): 512+si S issued (MMA warp), 1024+si PV issue start (P observed),
1536+si PV issued, 3072+si owning pair waits for S, 2048+si S observed, 2560+si P arrived,
3584+3c epilogue of item c: wait start / O observed / stores done.
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
if w == "c3":
    cfg = I.C3
else:
    _, N, d = w.split(":")
    cfg = I.c2(int(N), int(d))
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / math.sqrt(cfg.d), -math.log(cfg.N)
for _ in range(3):
    sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
t = buf.view(148, 4096).cpu().numpy().astype(np.float64)

agg = {"s_wait": [], "sigma": [], "period": [], "s_lead": [], "p_to_pv": []}
epi = {"o_wait": [], "stores": []}
for cta in range(148):
    r = t[cta]
    n = int((r[512:1024] > 0).sum())
    n = min(n, 500)
    if n < 8:
        continue
    for si in range(4, n):
        ws, so, pa = r[3072 + si], r[2048 + si], r[2560 + si]
        sis, pvs = r[512 + si], r[1024 + si]
        if min(ws, so, pa, sis, pvs) <= 0:
            continue
        agg["s_wait"].append(so - ws)          # pair idle waiting for S
        agg["sigma"].append(pa - so)           # sigma of one tile (pair)
        agg["s_lead"].append(so - sis)         # S issue -> observed by pair
        agg["p_to_pv"].append(pvs - pa)        # P arrive -> PV issue start
        if r[2048 + si - 2] > 0:
            agg["period"].append(so - r[2048 + si - 2])
    for c in range(0, 170):
        a0, a1, a2 = r[3584 + 3 * c], r[3584 + 3 * c + 1], r[3584 + 3 * c + 2]
        if a0 > 0 and a1 > 0 and a2 > 0:
            epi["o_wait"].append(a1 - a0)
            epi["stores"].append(a2 - a1)
print(f"workload {w}")
for k_, v_ in list(agg.items()) + list(epi.items()):
    a = np.array(v_)
    if len(a):
        print("%-8s n=%6d  median %7.0f  mean %7.0f  p10 %7.0f  p90 %7.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                           np.percentile(a, 10), np.percentile(a, 90)))
r = t[0]
t0 = r[512]
print(" si   S_issue  pair_wait  S_obs   P_arr   PV_start")
for si in range(0, 24):
    print("%3d " % si + " ".join("%8d" % (x - t0 if x > 0 else -1) for x in
                                 (r[512 + si], r[3072 + si], r[2048 + si], r[2560 + si], r[1024 + si])))
