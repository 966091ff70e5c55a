"""Pre-LN bidirectional encoder layer with the sigmoid-attention op.

The 160M-parameter model of PAPER.md Table 4: 12 layers, hidden 768, 12 heads of
d = 64, FFN 3072 with GELU, pre-norm LayerNorm (eps 1e-5), dropout 0.02, init std 0.02, bf16.
Attention is ``sigmoid_attention`` in the paper's [B, N, H, d] layout: the q/k/v
projections write [B, N, H*d] = [B, N, H, d] directly, so the op reads them in place (no
transposes), with b = -log N and the padded keys of each sequence at zero weight.

Only the attention runs in this package's kernels; the projections, LayerNorm and MLP are plain
PyTorch (cuBLAS) -- this module is the integration of the hot path into a model, not part of it.
"""
from __future__ import annotations

from typing import Optional

import torch
from torch import nn

from .attention import sigmoid_attention


class SigmoidEncoderLayer(nn.Module):
    def __init__(self, hidden: int = 768, heads: int = 12, ffn: int = 3072, dropout: float = 0.02,
                 eps: float = 1e-5, init_std: float = 0.02):
        super().__init__()
        if hidden % heads != 0 or hidden // heads not in (64, 128):
            raise ValueError("head dimension must be 64 or 128")
        self.hidden, self.heads, self.d = hidden, heads, hidden // heads
        self.ln1 = nn.LayerNorm(hidden, eps=eps)
        self.q_proj = nn.Linear(hidden, hidden)
        self.k_proj = nn.Linear(hidden, hidden)
        self.v_proj = nn.Linear(hidden, hidden)
        self.o_proj = nn.Linear(hidden, hidden)
        self.ln2 = nn.LayerNorm(hidden, eps=eps)
        self.fc1 = nn.Linear(hidden, ffn)
        self.fc2 = nn.Linear(ffn, hidden)
        self.drop = nn.Dropout(dropout)
        for m in (self.q_proj, self.k_proj, self.v_proj, self.o_proj, self.fc1, self.fc2):
            nn.init.normal_(m.weight, std=init_std)
            nn.init.zeros_(m.bias)

    def attention(self, x: torch.Tensor, seqlens: Optional[torch.Tensor]) -> torch.Tensor:
        B, N, _ = x.shape
        shape = (B, N, self.heads, self.d)
        q = self.q_proj(x).view(shape)
        k = self.k_proj(x).view(shape)
        v = self.v_proj(x).view(shape)
        o = sigmoid_attention(q, k, v, seqlens_q=seqlens, seqlens_k=seqlens, layout="bshd")
        return self.o_proj(o.reshape(B, N, self.hidden))

    def forward(self, x: torch.Tensor, seqlens: Optional[torch.Tensor] = None) -> torch.Tensor:
        x = x + self.drop(self.attention(self.ln1(x), seqlens))
        return x + self.drop(self.fc2(self.drop(torch.nn.functional.gelu(self.fc1(self.ln2(x))))))


class SigmoidEncoder(nn.Module):
    """Table 4's 12-layer encoder body (embeddings and heads are task-specific and not included)."""

    def __init__(self, layers: int = 12, hidden: int = 768, heads: int = 12, ffn: int = 3072,
                 dropout: float = 0.02):
        super().__init__()
        self.layers = nn.ModuleList(SigmoidEncoderLayer(hidden, heads, ffn, dropout) for _ in range(layers))
        self.ln_f = nn.LayerNorm(hidden, eps=1e-5)

    def forward(self, x: torch.Tensor, seqlens: Optional[torch.Tensor] = None) -> torch.Tensor:
        for layer in self.layers:
            x = layer(x, seqlens)
        return self.ln_f(x)

