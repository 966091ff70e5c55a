#!/usr/bin/env python
"""C3 fwd+bwd step timed as a loop of public-API calls without per-kernel profiling events (debug
tool for launch-overlap A/B).  usage: SIGATTN_LIB=... python scripts/time_step_loop.py [steps]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402
from paper_2604_27124_b200 import inputs as I  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = I.C3
q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
alpha, b = 1 / math.sqrt(cfg.d), -math.log(cfg.N)
fws = torch.empty(sa.fwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dtype=torch.uint8, device="cuda")
ws = torch.empty(sa.bwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dtype=torch.uint8, device="cuda")
o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))


def step():
    sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=o, workspace=fws)
    sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, dq=dq, dk=dk, dv=dv, workspace=ws)


for _ in range(5):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{os.path.basename(os.environ.get('SIGATTN_LIB', 'libsigattn.so'))}: C3 step {e0.elapsed_time(e1) / steps:.4f} ms")
