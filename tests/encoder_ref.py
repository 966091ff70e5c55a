"""Test-only plain-PyTorch fp32 composition of the encoder layer (paper_2604_27124_b200/encoder.py).

Lives under tests/ on purpose: it is a second implementation of the method (sigmoid attention
written out with torch ops) and must never be importable from the product package.  The layer's
attention itself is checked against the fp64 oracle (tests/test_parity_gpu.py); this reference only
covers the surrounding LayerNorm / projections / MLP and the gradients flowing through them.
"""
import math
from typing import Optional

import torch
def reference_attention_fp32(layer, x: torch.Tensor, seqlens: Optional[torch.Tensor]):
    """Plain-PyTorch fp32 composition of the same layer (test reference): sigma(QK^T/sqrt(d) - log N)
    with padded keys masked to zero weight and padded query rows zero."""
    B, N, _ = x.shape
    H, d = layer.heads, layer.d

    def lin(m, t):
        return torch.nn.functional.linear(t, m.weight.float(), m.bias.float())

    def ln(m, t):
        return torch.nn.functional.layer_norm(t, (layer.hidden,), m.weight.float(), m.bias.float(), m.eps)

    h = ln(layer.ln1, x)
    q, k, v = (lin(m, h).view(B, N, H, d).transpose(1, 2) for m in (layer.q_proj, layer.k_proj, layer.v_proj))
    p = torch.sigmoid(q @ k.transpose(-1, -2) / math.sqrt(d) - math.log(N))
    if seqlens is not None:
        ar = torch.arange(N, device=x.device)
        valid = (ar[None, :] < seqlens[:, None].long())
        p = p * valid[:, None, None, :] * valid[:, None, :, None]
    o = (p @ v).transpose(1, 2).reshape(B, N, layer.hidden)
    x = x + lin(layer.o_proj, o)
    return x + lin(layer.fc2, torch.nn.functional.gelu(lin(layer.fc1, ln(layer.ln2, x))))
