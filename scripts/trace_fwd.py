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
    parts = w.split(":")   # c2:N:d[:pad]
    cfg = I.c2(int(parts[1]), int(parts[2]))
    if len(parts) > 3:
        n_ = int(round(cfg.N * (1 - float(parts[3]))))
        cfg = I.Config(cfg.name + "_pad", B=cfg.B, H=cfg.H, N=cfg.N, d=cfg.d, lengths=[n_] * cfg.B, seed=0)
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / math.sqrt(cfg.d), -math.log(max(cfg.nk))
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
g0, g1 = t[:, 4094], t[:, 4095]
ok = (g0 > 0) & (g1 > 0)
base = g0[ok].min()
ntile = (t[:, 512:1024] > 0).sum(1)
print("CTA start (us after first): max %.1f | CTA end: min %.1f median %.1f max %.1f | tiles per CTA min %d max %d" % (
    (g0[ok].max() - base) / 1e3, (g1[ok].min() - base) / 1e3, np.median(g1[ok] - base) / 1e3, (g1[ok].max() - base) / 1e3,
    ntile.min(), ntile.max()))
mhz = (t[ok, 4093] - t[ok, 4092]) / (g1[ok] - g0[ok]) * 1e3
print("SM clock (clock64 / globaltimer over each CTA): median %.0f MHz, min %.0f" % (np.median(mhz), mhz.min()))
for k_, v_ in list(agg.items()) + list(epi.items()):
    a = np.array(v_)
    if len(a):
        print("%-8s n=%6d  median %7.0f  mean %7.0f  p10 %7.0f  p90 %7.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                           np.percentile(a, 10), np.percentile(a, 90)))
for cta in range(4):
    r = t[cta]
    n = int((r[512:1024] > 0).sum())
    ne = int(((r[3584:4092:3] > 0)).sum())
    k0 = r[4092]
    print("CTA %d (clk after start): first S issue %d, last S issue %d (#%d), last epilogue done %d (#%d), end %d" % (
        cta, r[512] - k0, r[512 + n - 1] - k0, n, r[3584 + 3 * (ne - 1) + 2] - k0, ne, r[4093] - k0))
r = t[0]
t0 = r[512]
print(" item  epi_wait  O_obs  stores_done")
for c in range(0, 8):
    print("%4d " % c + " ".join("%8d" % (r[3584 + 3 * c + e] - t0 if r[3584 + 3 * c + e] > 0 else -1) for e in range(3)))
print(" si   S_issue  pair_wait  S_obs   P_arr   PV_start")
for si in range(0, 24):
    print("%3d " % si + " ".join("%8d" % (x - t0 if x > 0 else -1) for x in
                                 (r[512 + si], r[3072 + si], r[2048 + si], r[2560 + si], r[1024 + si])))
