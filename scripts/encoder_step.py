#!/usr/bin/env python
"""Training-step time of Table 4's 12-layer 160M encoder body with sigmoid attention (this package,
[B, N, H, d] in place) vs the same body with PyTorch SDPA softmax attention -- the end-to-end
context of P:171-178 (debug / context tool, not the bench metric).

usage (GPU box): python scripts/encoder_step.py [B] [N]
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27124_b200.encoder import SigmoidEncoder  # noqa: E402
from paper_2604_27124_b200 import inputs as I  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
torch.manual_seed(0)
lens = torch.tensor((I.C3_LENGTHS * 4)[:B], dtype=torch.int32, device="cuda")
model = SigmoidEncoder(dropout=0.0).cuda().to(torch.bfloat16)
x = torch.randn(B, N, 768, device="cuda", dtype=torch.bfloat16)


def softmax_attention(self, h, seqlens):
    Bh, Nh, _ = h.shape
    q, k, v = (m(h).view(Bh, Nh, self.heads, self.d).transpose(1, 2) for m in (self.q_proj, self.k_proj, self.v_proj))
    mask = (torch.arange(Nh, device=h.device)[None, :] < seqlens[:, None].long())[:, None, None, :]
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=mask)
    return self.o_proj(o.transpose(1, 2).reshape(Bh, Nh, self.hidden))


def step():
    y = model(x, lens)
    y.float().square().mean().backward()


def timeit(n=5):
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


t_sig = timeit()
from paper_2604_27124_b200 import encoder as E  # noqa: E402
orig = E.SigmoidEncoderLayer.attention
E.SigmoidEncoderLayer.attention = softmax_attention
t_soft = timeit()
E.SigmoidEncoderLayer.attention = orig
print(f"12-layer 160M encoder body, B={B} N={N} jagged (C3 lengths), bf16, fwd+bwd (no optimizer):")
print(f"  sigmoid attention (this package): {t_sig:8.2f} ms/step")
print(f"  softmax SDPA (PyTorch, masked):    {t_soft:8.2f} ms/step   ratio {t_soft / t_sig:.2f}x")
