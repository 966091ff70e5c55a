#!/usr/bin/env python
"""Per-CTA start/end (globaltimer) of the fwd and bwd kernels on C3: load balance (debug tool)."""
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
lib = _lib.load()
for name in ("fwd", "bwd"):
    f = (lambda: sa.sigattn_fwd(q, k, v, nq, nk, 1 / 8, -math.log(8192))) if name == "fwd" else \
        (lambda: sa.sigattn_bwd(q, k, v, do, nq, nk, 1 / 8, -math.log(8192)))
    for _ in range(3):
        f()
    buf = torch.zeros(148 * 4096, dtype=torch.int64, device="cuda")
    lib.sigattn_set_trace_buffer(buf.data_ptr())
    f()
    torch.cuda.synchronize()
    lib.sigattn_set_trace_buffer(None)
    t = buf.view(148, 4096).cpu().numpy()
    st, en = t[:, 4094].astype(np.float64), t[:, 4095].astype(np.float64)
    t0 = st.min()
    dur = en - st
    print(f"{name}: start spread {st.max() - t0:.0f} ns; CTA busy ns min {dur.min():.0f} median {np.median(dur):.0f} "
          f"max {dur.max():.0f}; kernel span {en.max() - t0:.0f} ns; mean/max busy = {dur.mean() / dur.max():.3f}")
