#!/usr/bin/env python
"""Per-item timeline of the d=128 two-tile forward (fwd2.cuh) from a SIGATTN_TRACE build (debug tool).

usage (GPU box): SIGATTN_LIB=paper_2604_27124_b200/libsigattn_trace.so python scripts/trace_fwd2.py [N [pad]]
Slots per CTA (clock64): MMA warp, item c: c Q wait start, 512+c Q ready, 1024+c first S issued, 1536+c last PV
issued; sigma warp 0 (tile A), item c: 3584+3c epilogue wait start, +1 O observed, +2 stores done; 4064+w warp w
end; 4092/4093 kernel start/end clock, 4094/4095 globaltimer.
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import _lib, inputs as I  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pad = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
cfg = I.c2(N, 128)
n = int(round(N * (1 - pad)))
cfg = I.Config(cfg.name, B=cfg.B, H=cfg.H, N=N, d=128, lengths=[n] * cfg.B, seed=0)
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / math.sqrt(128), -math.log(n)
for _ in range(3):
    sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sigattn_set_trace_buffer(buf.data_ptr())
sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
torch.cuda.synchronize()
lib.sigattn_set_trace_buffer(None)
T = buf.view(148, 4096).cpu().numpy().astype(np.float64)
g0, g1 = T[:, 4094], T[:, 4095]
ok = (g0 > 0) & (g1 > 0)
mhz = (T[ok, 4093] - T[ok, 4092]) / (g1[ok] - g0[ok]) * 1e3
print(f"N={N} pad={pad} B={cfg.B} H={cfg.H}: CTA end (us): min %.1f median %.1f max %.1f; SM clock %.0f MHz" % (
    (g1[ok].min() - g0[ok].min()) / 1e3, np.median(g1[ok] - g0[ok].min()) / 1e3, (g1[ok].max() - g0[ok].min()) / 1e3,
    np.median(mhz)))
for cta in (0, 1, 100, 147):
    r = T[cta]
    k0 = r[4092]
    ni = int((r[512:1024] > 0).sum())
    print(f"CTA {cta}: {ni} items; end {r[4093] - k0:.0f} clk; warp ends (k clk): " +
          " ".join("%d:%.0f" % (w_, (r[4064 + w_] - k0) / 1e3) for w_ in range(20) if r[4064 + w_] > 0))
    print("  item  Qwait  Qready  S0issued  lastPV  epi_wait  O_obs  stored   (clk after kernel start)")
    for c in range(ni):
        vals = [r[c], r[512 + c], r[1024 + c], r[1536 + c], r[3584 + 3 * c], r[3584 + 3 * c + 1], r[3584 + 3 * c + 2]]
        print("  %4d " % c + " ".join("%8d" % (x - k0 if x > 0 else -1) for x in vals))
