#!/usr/bin/env python
"""Compute-warp phases of the d=64 backward kernel (SIGATTN_TRACE build, debug tool).

Events per compute warp and tile t in [40, 48): 0 S(h0) observed, 1 h0 sigma/dS done, 2 h0 arrived,
3 S(h1) observed, 4 h1 done, 5 h1 arrived (slot 4*512 + (warp*8 + t-40)*8 + e).
usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_bwd_phases.py
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
t = buf.view(148, 4096).cpu().numpy().astype(np.float64)
acc = {k_: [] for k_ in ("h0 compute", "h0 store+arrive", "wait S h1", "h1 compute", "h1 store+arrive",
                         "wait S h0(next)", "tile period")}
for cta in range(148):
    ev = t[cta, 4 * 512:4 * 512 + 16 * 64].reshape(16, 8, 8)
    if (ev[:, :, :6] <= 0).any():
        continue
    for wp in range(16):
        e = ev[wp]
        acc["h0 compute"] += list(e[:, 1] - e[:, 0])
        acc["h0 store+arrive"] += list(e[:, 2] - e[:, 1])
        acc["wait S h1"] += list(e[:, 3] - e[:, 2])
        acc["h1 compute"] += list(e[:, 4] - e[:, 3])
        acc["h1 store+arrive"] += list(e[:, 5] - e[:, 4])
        acc["wait S h0(next)"] += list(e[1:, 0] - e[:-1, 5])
        acc["tile period"] += list(np.diff(e[:, 0]))
print(f"workload {w}")
for k_, v_ in acc.items():
    a = np.array(v_)
    if len(a):
        print("%-18s n=%6d median %6.0f mean %6.0f p10 %6.0f p90 %6.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                          np.percentile(a, 10), np.percentile(a, 90)))

# MMA warp vs compute warp 0 vs epilogue warpgroup, tiles 40..47
mm = {k_: [] for k_ in ("P0 arrive -> MMA sees P0", "MMA sees P0 -> S(t+1,h0) issued", "S(t+1,h0) issued -> observed",
                        "P1 arrive -> MMA sees P1", "MMA sees P1 -> dQ(t) issued", "epi: P0 seen -> dS h0 copied",
                        "P0 arrive -> epi sees P0")}
for cta in range(148):
    r = t[cta]
    ev = r[4 * 512:4 * 512 + 16 * 64].reshape(16, 8, 8)
    if (ev[:, :, :6] <= 0).any():
        continue
    e = ev.max(axis=0)   # latest warp per event (the barrier completes with the last arrival)
    for j in range(8):
        tt = 40 + j
        mp0, mq0, mp1, mdq = r[tt], r[512 + tt], r[1024 + tt], r[1536 + tt]
        ep0, ecp = r[3072 + j * 16 + 0], r[3072 + j * 16 + 1]
        if min(mp0, mq0, mp1, mdq) <= 0:
            continue
        mm["P0 arrive -> MMA sees P0"].append(mp0 - e[j, 2])
        mm["MMA sees P0 -> S(t+1,h0) issued"].append(mq0 - mp0)
        if j < 7:
            mm["S(t+1,h0) issued -> observed"].append(ev[:, j + 1, 0].max() - mq0)
        mm["P1 arrive -> MMA sees P1"].append(mp1 - e[j, 5])
        mm["MMA sees P1 -> dQ(t) issued"].append(mdq - mp1)
        if ep0 > 0 and ecp > 0:
            mm["epi: P0 seen -> dS h0 copied"].append(ecp - ep0)
            mm["P0 arrive -> epi sees P0"].append(ep0 - e[j, 2])
for k_, v_ in mm.items():
    a = np.array(v_)
    if len(a):
        print("%-34s n=%5d median %6.0f mean %6.0f p10 %6.0f p90 %6.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                          np.percentile(a, 10), np.percentile(a, 90)))

# MMA warp detail (slots 3328 + j*8 + e): 4 starts waiting P0(t), 0 mma2(t,h0) issued, 1 mma2(t,h1) issued,
# 2 S(t+1,h1) issued, 3 dQ(t) waits satisfied
md = {k_: [] for k_ in ("wait P0 start -> sees P0", "sees P0 -> mma2 h0 issued", "mma2 h0 -> S(t+1,h0) issued",
                        "S(t+1,h0) issued -> sees P1", "sees P1 -> mma2 h1 issued", "mma2 h1 -> S(t+1,h1) issued",
                        "S(t+1,h1) issued -> dQ waits done", "dQ waits done -> dQ issued",
                        "dQ issued -> wait P0(t+1) start")}
for cta in range(148):
    r = t[cta]
    for j in range(7):
        tt = 40 + j
        d = r[3328 + j * 8: 3328 + j * 8 + 8]
        mp0, mq0, mp1, mdq = r[tt], r[512 + tt], r[1024 + tt], r[1536 + tt]
        nxt = r[3328 + (j + 1) * 8 + 4]
        if min(d[0], d[1], d[2], d[3], d[4], mp0, mq0, mp1, mdq, nxt) <= 0:
            continue
        md["wait P0 start -> sees P0"].append(mp0 - d[4])
        md["sees P0 -> mma2 h0 issued"].append(d[0] - mp0)
        md["mma2 h0 -> S(t+1,h0) issued"].append(mq0 - d[0])
        md["S(t+1,h0) issued -> sees P1"].append(mp1 - mq0)
        md["sees P1 -> mma2 h1 issued"].append(d[1] - mp1)
        md["mma2 h1 -> S(t+1,h1) issued"].append(d[2] - d[1])
        md["S(t+1,h1) issued -> dQ waits done"].append(d[3] - d[2])
        md["dQ waits done -> dQ issued"].append(mdq - d[3])
        md["dQ issued -> wait P0(t+1) start"].append(nxt - mdq)
for k_, v_ in md.items():
    a = np.array(v_)
    if len(a):
        print("%-34s n=%5d median %6.0f mean %6.0f p10 %6.0f p90 %6.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                          np.percentile(a, 10), np.percentile(a, 90)))

me = {k_: [] for k_ in ("mma2 h0 issued -> kv ok", "qdo_full wait", "ds_copied0 wait", "-> S(t+1,h0) issued")}
for cta in range(148):
    r = t[cta]
    for j in range(7):
        d = r[3328 + j * 8: 3328 + j * 8 + 8]
        mq0 = r[512 + 40 + j]
        if min(d[0], d[5], d[6], d[7], mq0) <= 0:
            continue
        me["mma2 h0 issued -> kv ok"].append(d[5] - d[0])
        me["qdo_full wait"].append(d[6] - d[5])
        me["ds_copied0 wait"].append(d[7] - d[6])
        me["-> S(t+1,h0) issued"].append(mq0 - d[7])
for k_, v_ in me.items():
    a = np.array(v_)
    if len(a):
        print("%-34s n=%5d median %6.0f mean %6.0f p10 %6.0f p90 %6.0f clk" % (k_, len(a), np.median(a), a.mean(),
                                                                          np.percentile(a, 10), np.percentile(a, 90)))
