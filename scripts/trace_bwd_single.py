#!/usr/bin/env python
"""Joint timeline of the d=64 fused backward (single MMA issuer) for tiles 41..46 of every CTA (SIGATTN_TRACE build).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd_single.py [c3|c2:N]
Slots (bwd.cuh): MMA warp t: p_full0 passed, 512+t S/dP(t+1,h0) issued, 1024+t p_full1 passed, 1536+t dQ(t) issued,
3328+(t-40)*8+e (0 dV/dK(t,h0) issued, 5 K/V waited, 6 Q/dO(t+1) waited, 7 ds_copied waited, 1 dV/dK(t,h1) issued,
2 S/dP(t+1,h1) issued, 3 dQ waits passed); compute 2048+(warp*8+t-40)*8+e (0 S h0 seen, 1 h0 done, 2 h0 arrived,
3 S h1 seen, 4 h1 done, 5 h1 arrived); epilogue 3072+(t-40)*16+e (staging mode: 0..6; dQ drain of tile t-1 (lagged)
or t (direct staging): 7 dQ full seen, 8 dQ read, 9 dQ staged, 10 reduce issued).  All times relative to the MMA
warp passing p_full0 of tile t.
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
if w == "c3":
    cfg = I.C3
else:   # c2:N[:pad]
    parts = w.split(":")
    cfg = I.c2(int(parts[1]), 64)
    if len(parts) > 2:
        n_ = int(round(cfg.N * (1 - float(parts[2]))))
        cfg = I.Config(cfg.name + "_pad", B=cfg.B, H=cfg.H, N=cfg.N, d=64, lengths=[n_] * cfg.B, seed=0)
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / 8, -math.log(max(cfg.nk))
for _ in range(3):
    sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
T = buf.view(148, 4096).cpu().numpy().astype(np.float64)
g0, g1 = T[:, 4094], T[:, 4095]
ok = (g0 > 0) & (g1 > 0)
mhz = (T[ok, 4093] - T[ok, 4092]) / (g1[ok] - g0[ok]) * 1e3
print("CTA end (us after first start): min %.1f median %.1f max %.1f; SM clock %.0f MHz" % (
    (g1[ok].min() - g0[ok].min()) / 1e3, np.median(g1[ok] - g0[ok].min()) / 1e3, (g1[ok].max() - g0[ok].min()) / 1e3,
    np.median(mhz)))
for cta in range(3):
    r = T[cta]
    nt = int((r[0:512] > 0).sum())
    k0 = r[4092]
    print("CTA %d: %d tiles, first p_full0 %d clk after start, last dQ issued %d, end %d" % (
        cta, nt, r[0] - k0, r[1536 + nt - 1] - k0, r[4093] - k0))
for cta in (0, 1, 40, 100):
    r = T[cta]
    print("CTA %3d warp end (k clk after start): " % cta + " ".join("%d:%.0f" % (w_, (r[4064 + w_] - r[4092]) / 1e3)
                                                                for w_ in range(24) if r[4064 + w_] > 0))
per, agg = [], {}
for cta in range(148):
    r = T[cta]
    if r[40] <= 0 or r[48] <= 0:
        continue
    per.append(np.median(np.diff(r[40:48])))
    for t in range(41, 47):
        base = r[t]

        def put(name, val):
            if val > 0:
                agg.setdefault(name, []).append(val - base)
        m = r[3328 + (t - 40) * 8: 3328 + (t - 40) * 8 + 8]
        put("MMA a dV/dK(t,h0) issued", m[0])
        put("MMA b K/V waited", m[5])
        put("MMA c Q/dO(t+1) waited", m[6])
        put("MMA d ds_copied0 waited", m[7])
        put("MMA e S/dP(t+1,h0) issued", r[512 + t])
        put("MMA f p_full1 passed", r[1024 + t])
        put("MMA g dV/dK(t,h1) issued", m[1])
        put("MMA h S/dP(t+1,h1) issued", m[2])
        put("MMA i dQ waits passed", m[3])
        put("MMA j dQ(t) issued", r[1536 + t])
        put("MMA k next p_full0", r[t + 1])
        ev = r[2048:3072].reshape(16, 8, 8)[:, t - 40, :]
        for e, nm in enumerate(["S h0 seen", "h0 done", "h0 arrived", "S h1 seen", "h1 done", "h1 arrived",
                                "h0 sigma done", "h0 dP loaded"]):
            vals = ev[:, e]
            if (vals > 0).all():
                put("cmp first " + nm, vals.min())
                put("cmp last  " + nm, vals.max())
        ep = r[3072 + (t - 40) * 16: 3072 + (t - 40) * 16 + 11]
        for e, nm in enumerate(["p h0 seen", "h0 copied", "ds_free ok", "h0 staged", "p h1 seen", "h1 copied",
                                "h1 staged", "dQ full seen", "dQ read", "dQ staged", "reduce issued"]):
            put("epi " + nm, ep[e])
print(f"{w}: median tile period (MMA p_full0 -> next) {np.median(per):.0f} clk over {len(per)} CTAs")
for k_, v_ in sorted(agg.items(), key=lambda kv: np.median(kv[1])):
    print(f"  {k_:32s} {np.median(v_):8.0f}   (p10 {np.percentile(v_, 10):7.0f}, p90 {np.percentile(v_, 90):7.0f})")
