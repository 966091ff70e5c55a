#!/usr/bin/env python
"""Small invocations of every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck).

usage (GPU box): compute-sanitizer --tool memcheck python scripts/sanitize_run.py
Runs: C1 (B=2 H=2 N=256 d=64, lengths 256/97) and a ragged d=128 case (N=320, lengths 320/129/0),
forward (fwd.cuh d=64, fwd2.cuh d=128), fused backward (bwd.cuh, bwd128.cuh), deterministic backward
(dq.cuh + the key-tile pass), and the fused context-parallel calls (fwd_cp, bwd_cp push, finalize).
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import attention as A, inputs as I  # noqa: E402

cases = [I.C1, I.Config("ragged_d128", B=3, H=2, N=320, d=128, lengths=[320, 129, 0], seed=3)]
if "--many" in sys.argv:   # more work items than the 148 persistent CTAs (multi-item pipelines)
    lens = [1024, 0, 1, 127, 129, 640, 1000, 385] * 2
    cases += [I.Config("many_d64", B=16, H=4, N=1024, d=64, lengths=lens, seed=4),
              I.Config("many_d128", B=16, H=4, N=1024, d=128, lengths=lens, seed=4)]
for cfg in cases:
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1.0 / math.sqrt(cfg.d), -math.log(cfg.N)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
    dq2, dk2, dv2 = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, deterministic=True)
    torch.cuda.synchronize()
    print(cfg.name, "fwd/bwd/det ok", float(o.float().abs().max()), float(dq.float().abs().max()), flush=True)
# fused context parallelism, two virtual ranks on this device
cfg = I.Config("cp_small", B=2, H=2, N=256, d=64, lengths=[256, 97], seed=5)
q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
n = 128
acc = [torch.zeros((2, 2, n, 64), device="cuda") for _ in range(2)]
dacc = [torch.zeros((2, 2, n, 64), device="cuda") for _ in range(2)]
tab = torch.tensor([t.data_ptr() for t in acc], dtype=torch.int64, device="cuda")
dtab = torch.tensor([t.data_ptr() for t in dacc], dtype=torch.int64, device="cuda")
for r in range(2):
    kb, vb = (t[:, :, r * n:(r + 1) * n].contiguous() for t in (k, v))
    nk_r = torch.tensor([max(0, min(n, L - r * n)) for L in cfg.lengths], dtype=torch.int32, device="cuda")
    A.sigattn_fwd_cp(q, kb, vb, nq, nk_r, 1 / 8, -math.log(256), tab, 2, r)
    A.sigattn_bwd_cp(q, kb, vb, do, nq, nk_r, 1 / 8, -math.log(256), dtab, 2, r)
outs = [A.sigattn_cp_finalize(acc[r], nq, 256, 2, r) for r in range(2)]
torch.cuda.synchronize()
print("cp fused ok", float(outs[0].float().abs().max()), flush=True)
