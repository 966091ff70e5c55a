"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's callers.

This module holds NO arithmetic of the method (no scores, no sigmoid, no bias formula): only
shapes, length distributions and seeded random tensors.  It is the single piece both sides of a
parity check may share.

Recipe:
  * every tensor is [B, H, N, d] contiguous;
  * valid entries are i.i.d. N(0, 1) fp32 drawn from ``torch.Generator('cpu').manual_seed(seed)``
    in the order Q, K, V, dO, then rounded (RN) to the compute dtype;
  * pad entries (rows >= n of their sequence) are 0, or -- for the pad-independence tests --
    i.i.d. finite values from a second generator (``pad="random"``) or a constant (``pad=1e6``);
  * jagged lengths follow the CellxGene-like log-normal of PAPER.md Fig. 1: the C3
    batch is ``round(exp(N(7.5, 0.75)))`` clamped to [200, 8192] from numpy PCG64(1), pinned
    below as a literal.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np
import torch

# C3 lengths: round(exp(N(7.5, 0.75))) clamped to [200, 8192], numpy PCG64 seed 1, 32 draws.
C3_LENGTHS = [2343, 3348, 2317, 680, 3565, 2527, 1209, 2796, 2377, 2254, 1847, 2724, 1041, 1600,
              1259, 2833, 1863, 1452, 1006, 1491, 1819, 1470, 4772, 3847, 237, 438, 1586, 1317,
              2122, 2128, 8192, 785]


def lognormal_lengths(n: int, mu: float = 7.5, sigma: float = 0.75, lo: int = 200,
                      hi: int = 8192, seed: int = 1) -> list:
    """Jagged lengths: round(exp(N(mu, sigma))) clamped to [lo, hi] (Fig. 1 analogue)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.exp(rng.normal(mu, sigma, n))
    return [int(v) for v in np.clip(np.round(x), lo, hi).astype(np.int64)]


@dataclass
class Config:
    """One workload: [B, H, N, d] with per-sequence valid lengths."""
    name: str
    B: int
    H: int
    N: int
    d: int
    lengths: Optional[list] = None      # None => unpadded (all N valid)
    dtype: str = "bf16"
    seed: int = 0
    fwd_only: bool = False
    Nk: Optional[int] = None            # key length if different from N (CP shards)
    lengths_k: Optional[list] = None

    @property
    def nq(self) -> list:
        return list(self.lengths) if self.lengths is not None else [self.N] * self.B

    @property
    def nk(self) -> list:
        if self.lengths_k is not None:
            return list(self.lengths_k)
        if self.Nk is not None and self.lengths is None:
            return [self.Nk] * self.B
        return self.nq

    @property
    def N_k(self) -> int:
        return self.Nk if self.Nk is not None else self.N


def torch_dtype(name: str) -> torch.dtype:
    return {"bf16": torch.bfloat16, "fp16": torch.float16, "f32": torch.float32}[name]


# BASELINE.json configs.  C2/C4/C5 are families; these are their named members.
C1 = Config("c1_parity_B2_H2_N256_d64", B=2, H=2, N=256, d=64, lengths=[256, 97], seed=0)
C1_FP16 = Config("c1_parity_fp16", B=2, H=2, N=256, d=64, lengths=[256, 97], dtype="fp16", seed=0)
C3 = Config("c3_jagged_B32_N8192_H12_d64", B=32, H=12, N=8192, d=64, lengths=C3_LENGTHS, seed=1)


def c2(N: int, d: int) -> Config:
    """Forward-only sweep member: token budget 16384, H=16, unpadded."""
    return Config(f"c2_fwd_N{N}_d{d}", B=max(1, 16384 // N), H=16, N=N, d=d, seed=0, fwd_only=True)


def c4_layer(layer: int) -> Config:
    """One attention layer of the 160M encoder (Table 4): B=16, H=12, N=8192, d=64."""
    return Config(f"c4_layer{layer}", B=16, H=12, N=8192, d=64, seed=100 + layer)


def c5(H: int = 16, d: int = 128) -> Config:
    """Single 16K sequence for key-split context parallelism."""
    return Config(f"c5_cp_N16384_H{H}_d{d}", B=1, H=H, N=16384, d=d, seed=0)


def _fill_pad(t: torch.Tensor, lengths: Sequence[int], pad: Union[str, float, None],
              gen: torch.Generator) -> None:
    """t is [B, H, N, d] fp32; overwrite rows >= lengths[b] with the pad fill."""
    B, H, N, d = t.shape
    for b in range(B):
        n = int(lengths[b])
        if n >= N:
            continue
        if pad is None or pad == 0 or pad == "zero":
            t[b, :, n:, :] = 0.0
        elif pad == "random":
            t[b, :, n:, :] = torch.randn((H, N - n, d), generator=gen) * 3.0
        else:
            t[b, :, n:, :] = float(pad)


def make_inputs(cfg: Config, device: Union[str, torch.device] = "cpu", pad=None,
                with_dout: bool = True, pad_seed: int = 12345):
    """Seeded (q, k, v, dout) in the compute dtype on ``device`` plus int32 lengths.

    Draw order Q, K, V, dO from one CPU generator so the same seed gives the same values on
    every machine; values are rounded to the compute dtype on the CPU, then moved.
    """
    g = torch.Generator("cpu").manual_seed(cfg.seed)
    gp = torch.Generator("cpu").manual_seed(pad_seed)
    Nk = cfg.N_k
    q = torch.randn((cfg.B, cfg.H, cfg.N, cfg.d), generator=g)
    k = torch.randn((cfg.B, cfg.H, Nk, cfg.d), generator=g)
    v = torch.randn((cfg.B, cfg.H, Nk, cfg.d), generator=g)
    dout = torch.randn((cfg.B, cfg.H, cfg.N, cfg.d), generator=g) if with_dout else None
    _fill_pad(q, cfg.nq, pad, gp)
    _fill_pad(k, cfg.nk, pad, gp)
    _fill_pad(v, cfg.nk, pad, gp)
    if dout is not None:
        _fill_pad(dout, cfg.nq, pad, gp)
    dt = torch_dtype(cfg.dtype)
    out = [t.to(dt).to(device) if t is not None else None for t in (q, k, v, dout)]
    nq = torch.tensor(cfg.nq, dtype=torch.int32, device=device)
    nk = torch.tensor(cfg.nk, dtype=torch.int32, device=device)
    return out[0], out[1], out[2], out[3], nq, nk


def make_inputs_gpu_fast(cfg: Config, device, seed_offset: int = 0):
    """Large-config generator (bench): draws on the device with a seeded CUDA generator.

    Used only where the oracle checks sampled rows through the same tensors (copied back), so
    both sides still see identical values.  Pad rows are zero.
    """
    g = torch.Generator(device=device).manual_seed(cfg.seed + seed_offset)
    dt = torch_dtype(cfg.dtype)
    Nk = cfg.N_k
    q = torch.randn((cfg.B, cfg.H, cfg.N, cfg.d), generator=g, device=device, dtype=torch.float32)
    k = torch.randn((cfg.B, cfg.H, Nk, cfg.d), generator=g, device=device, dtype=torch.float32)
    v = torch.randn((cfg.B, cfg.H, Nk, cfg.d), generator=g, device=device, dtype=torch.float32)
    dout = torch.randn((cfg.B, cfg.H, cfg.N, cfg.d), generator=g, device=device, dtype=torch.float32)
    nq_t = torch.tensor(cfg.nq, dtype=torch.int32, device=device)
    nk_t = torch.tensor(cfg.nk, dtype=torch.int32, device=device)
    ar = torch.arange(cfg.N, device=device)
    ark = torch.arange(Nk, device=device)
    mq = (ar[None, :] < nq_t[:, None].long()).to(torch.float32)[:, None, :, None]
    mk = (ark[None, :] < nk_t[:, None].long()).to(torch.float32)[:, None, :, None]
    q = (q * mq).to(dt); dout = (dout * mq).to(dt)
    k = (k * mk).to(dt); v = (v * mk).to(dt)
    return q, k, v, dout, nq_t, nk_t
