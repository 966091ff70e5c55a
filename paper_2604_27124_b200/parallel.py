"""Multi-GPU plumbing for the sigmoid-attention hot path, one process per GPU.

Two ways to spread the work, both built on torch.distributed (NCCL on GPUs; gloo in the CPU tests):

1. Batch x head sharding (config C4).  (b, h) pairs are fully independent -- no softmax
   normalisation, no cross-head coupling (Eq. 2) -- so each rank runs the fused kernels on its
   own pairs and the op needs NO collective.  Jagged batches are balanced with LPT on the valid-token
   cost n_q[b] * n_k[b].  A rank's pairs are viewed as a [P, 1, N, d] batch (one head per entry, the
   sequence's lengths repeated), so the same kernels run unchanged.

2. Key-split context parallelism (config C5), in two variants.  Sigmoid weights are decoupled across keys:
   O = sum_r sigma(Q K_r^T alpha + b) V_r with the SAME global bias b = -log N (never the shard
   length), so partial outputs are simply summed -- no log-sum-exp merge as in softmax ring
   attention.  Rank r holds query block r and key block r:
       forward : all-gather Q;  O_r = fwd(Q, K_r, V_r) in fp32;  reduce-scatter(sum) over query blocks
       backward: all-gather dO; (dQ_r, dK_r, dV_r) = bwd(Q, K_r, V_r, dO) with fp32 dQ_r;
                 dK_r, dV_r are complete (keys are owned); reduce-scatter(sum) dQ_r over query blocks.

   fused (fused=True): no partial tensor and no reduce-scatter.  Every rank maps
   every rank's fp32 accumulator [B, H, N/G, d] (CUDA IPC, PeerAccumulators).  The forward
   kernel's epilogue reduce-adds each partial O row straight into its owner's accumulator
   (sigattn_fwd_cp, system-scope red.global.add over NVLink), overlapped with the attention math of
   the other tiles; the backward sums dQ over the rank's key tiles in L2 and a push kernel
   reduce-adds each row into its owner (sigattn_bwd_cp).  A stream-ordered cross-rank barrier and
   sigattn_cp_finalize (fp32 -> bf16, padded rows 0) complete the op.

The attention calls default to the CUDA library (attention.sigattn_fwd / sigattn_bwd).  The `impl`
hook exists so the CPU tests can drive the same orchestration through gloo with a stand-in; the
product path never substitutes anything for the kernels.
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist


# ------------------------------------------------------------------------------------------------
# batch x head sharding
def lpt_assign(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of items to `world` bins (ties: lower index first).

    Returns, per rank, the item indices in assignment order.  Greedy LPT is within 4/3 of the
    optimal makespan; for the C3/C4 batches it is within a few percent of perfect balance.
    """
    if world <= 0:
        raise ValueError("world must be positive")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return out


def shard_pairs(B: int, H: int, nq: Sequence[int], nk: Sequence[int], world: int) -> List[List[tuple]]:
    """(b, h) pairs per rank, LPT-balanced on the valid-token cost n_q[b] * n_k[b] (App. B.1)."""
    pairs = [(b, h) for b in range(B) for h in range(H)]
    costs = [int(nq[b]) * int(nk[b]) for b, _ in pairs]
    return [[pairs[i] for i in idx] for idx in lpt_assign(costs, world)]


def gather_pairs(t: torch.Tensor, pairs: Sequence[tuple]) -> torch.Tensor:
    """[B, H, N, d] -> [P, 1, N, d] holding the given (b, h) pairs (a copy; contiguous)."""
    B, H = t.shape[:2]
    idx = torch.tensor([b * H + h for b, h in pairs], dtype=torch.long, device=t.device)
    return t.reshape(B * H, 1, *t.shape[2:]).index_select(0, idx).contiguous()


def pair_lengths(lengths: Optional[torch.Tensor], pairs: Sequence[tuple], N: int, device) -> torch.Tensor:
    if lengths is None:
        return torch.full((len(pairs),), N, dtype=torch.int32, device=device)
    lens = lengths.to(device=device, dtype=torch.int32)
    return lens[torch.tensor([b for b, _ in pairs], dtype=torch.long, device=device)].contiguous()


# ------------------------------------------------------------------------------------------------
# key-split context parallelism
@dataclass
class CPShard:
    """Where this rank sits in a key/query split of a length-N sequence into `world` blocks."""
    rank: int
    world: int
    N: int

    @property
    def block(self) -> int:
        if self.N % self.world:
            raise ValueError("context-parallel split needs N divisible by the world size")
        return self.N // self.world

    def local_len(self, n_valid: int) -> int:
        """Valid tokens of a length-n_valid sequence that fall in this rank's block."""
        return max(0, min(self.block, n_valid - self.rank * self.block))


def _is_nccl(group=None) -> bool:
    return dist.get_backend(group) == "nccl"


def _all_gather_into(buf: torch.Tensor, x: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor; with gloo, CUDA tensors are staged through host memory (gloo has no
    CUDA all-gather) -- the multi-process tests on one GPU take that path, NCCL runs take the other."""
    if x.is_cuda and not _is_nccl(group):
        hb = torch.empty(buf.shape, dtype=buf.dtype)
        dist.all_gather_into_tensor(hb, x.cpu(), group=group)
        buf.copy_(hb)
    else:
        dist.all_gather_into_tensor(buf, x, group=group)


def _all_gather_seq(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[B, H, n, d] blocks from every rank -> [B, H, world * n, d] in rank order."""
    if world == 1:
        return x.contiguous()
    B, H, n, d = x.shape
    buf = torch.empty((world * B, H, n, d), dtype=x.dtype, device=x.device)   # rank-major along dim 0
    _all_gather_into(buf, x.contiguous(), group=group)
    return buf.view(world, B, H, n, d).permute(1, 2, 0, 3, 4).reshape(B, H, world * n, d).contiguous()


def _reduce_scatter_seq(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[B, H, world * n, d] partial sums on every rank -> this rank's [B, H, n, d] block of the sum."""
    if world == 1:
        return x
    B, H, N, d = x.shape
    n = N // world
    src = x.reshape(B, H, world, n, d).permute(2, 0, 1, 3, 4).reshape(world * B, H, n, d).contiguous()
    out = torch.empty((B, H, n, d), dtype=x.dtype, device=x.device)
    dist.reduce_scatter_tensor(out, src, op=dist.ReduceOp.SUM, group=group)
    return out


def _default_fwd(q, k, v, nq, nk, scale, bias):
    from .attention import sigattn_fwd
    return sigattn_fwd(q, k, v, nq, nk, scale, bias, out_f32=True)


def _default_bwd(q, k, v, do, nq, nk, scale, bias):
    from .attention import sigattn_bwd
    return sigattn_bwd(q, k, v, do, nq, nk, scale, bias, dq_f32=True)


def cp_forward(q_blk: torch.Tensor, k_blk: torch.Tensor, v_blk: torch.Tensor, shard: CPShard,
               lengths: Optional[Sequence[int]] = None, scale: Optional[float] = None,
               bias: Optional[float] = None, group=None, impl_fwd: Optional[Callable] = None):
    """Key-split CP forward.  q_blk/k_blk/v_blk: this rank's [B, H, N/G, d] blocks.

    Returns (o_blk in q's dtype, q_full) -- q_full is kept for the backward.
    bias defaults to -log N of the GLOBAL length (reading R1), never the block length.
    """
    impl_fwd = impl_fwd or _default_fwd
    B, H, n, d = q_blk.shape
    N = shard.N
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    bias = -math.log(N) if bias is None else float(bias)
    q_full = _all_gather_seq(q_blk, shard.world, group)
    lengths = [N] * B if lengths is None else list(lengths)
    nq = torch.tensor(lengths, dtype=torch.int32, device=q_blk.device)
    nk = torch.tensor([shard.local_len(x) for x in lengths], dtype=torch.int32, device=q_blk.device)
    o_part = impl_fwd(q_full, k_blk, v_blk, nq, nk, scale, bias)          # fp32 [B, H, N, d]
    o_blk = _reduce_scatter_seq(o_part, shard.world, group)
    return o_blk.to(q_blk.dtype), q_full


def cp_backward(q_full: torch.Tensor, k_blk: torch.Tensor, v_blk: torch.Tensor, do_blk: torch.Tensor,
                shard: CPShard, lengths: Optional[Sequence[int]] = None, scale: Optional[float] = None,
                bias: Optional[float] = None, group=None, impl_bwd: Optional[Callable] = None):
    """Key-split CP backward -> (dq_blk, dk_blk, dv_blk), all this rank's blocks."""
    impl_bwd = impl_bwd or _default_bwd
    B, H, N, d = q_full.shape
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    bias = -math.log(shard.N) if bias is None else float(bias)
    do_full = _all_gather_seq(do_blk, shard.world, group)
    lengths = [shard.N] * B if lengths is None else list(lengths)
    nq = torch.tensor(lengths, dtype=torch.int32, device=q_full.device)
    nk = torch.tensor([shard.local_len(x) for x in lengths], dtype=torch.int32, device=q_full.device)
    dq_part, dk_blk, dv_blk = impl_bwd(q_full, k_blk, v_blk, do_full, nq, nk, scale, bias)   # dq fp32
    if dq_part.dtype not in (torch.float32, torch.float64):
        dq_part = dq_part.float()          # partials are summed in fp32
    dq_blk = _reduce_scatter_seq(dq_part, shard.world, group)
    return dq_blk.to(q_full.dtype), dk_blk, dv_blk


class CPSigmoidAttentionFn(torch.autograd.Function):
    """Autograd wrapper of the key-split CP op (saves the gathered Q, never O or P)."""

    @staticmethod
    def forward(ctx, q_blk, k_blk, v_blk, shard, lengths, scale, bias, group):
        o_blk, q_full = cp_forward(q_blk, k_blk, v_blk, shard, lengths, scale, bias, group)
        ctx.save_for_backward(q_full, k_blk, v_blk)
        ctx.args = (shard, lengths, scale, bias, group)
        return o_blk

    @staticmethod
    def backward(ctx, do_blk):
        q_full, k_blk, v_blk = ctx.saved_tensors
        shard, lengths, scale, bias, group = ctx.args
        dq, dk, dv = cp_backward(q_full, k_blk, v_blk, do_blk.contiguous(), shard, lengths, scale, bias, group)
        return dq, dk, dv, None, None, None, None, None


def cp_sigmoid_attention(q_blk, k_blk, v_blk, shard: CPShard, lengths=None, scale=None, bias=None, group=None):
    return CPSigmoidAttentionFn.apply(q_blk, k_blk, v_blk, shard, lengths, scale, bias, group)


# ------------------------------------------------------------------------------------------------
# fused key-split CP: the reduction runs inside the kernels
def cross_rank_sync(group=None, device=None) -> None:
    """Every rank's earlier stream work is complete before any rank's later stream work starts.
    NCCL: a one-element all-reduce is a stream-ordered barrier (a rank's all-reduce finishes only once
    every rank has reached it, i.e. after their preceding kernels).  gloo: host synchronisation."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if _is_nccl(group):
            t = torch.zeros(1, dtype=torch.float32, device=device)
            dist.all_reduce(t, group=group)
        else:
            torch.cuda.synchronize(device)
            dist.barrier(group=group)


class PeerAccumulators:
    """This rank's fp32 accumulator [B, H, N / G, d] for the rows it owns, plus a device table of
    every rank's accumulator mapped on this device (CUDA IPC handles exchanged through
    torch.distributed; peer access over NVLink).  world == 1: the table holds this rank's own buffer.
    Collective: every rank of the group constructs it in the same order."""

    def __init__(self, B: int, H: int, rows: int, d: int, device, group=None):
        from .attention import ipc_export, ipc_import
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.acc = torch.zeros((B, H, rows, d), dtype=torch.float32, device=device)
        self._imported: List[int] = []
        if self.world == 1:
            ptrs = [self.acc.data_ptr()]
        else:
            handles: List[Optional[bytes]] = [None] * self.world
            dist.all_gather_object(handles, ipc_export(self.acc), group=group)
            ptrs = []
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self.acc.data_ptr())
                else:
                    p = ipc_import(h)
                    self._imported.append(p)
                    ptrs.append(p)
        self.table = torch.tensor(ptrs, dtype=torch.int64, device=device)

    def close(self) -> None:
        from .attention import ipc_close
        for p in self._imported:
            ipc_close(p)
        self._imported = []


def cp_forward_fused(q_blk: torch.Tensor, k_blk: torch.Tensor, v_blk: torch.Tensor, shard: CPShard,
                     peers: PeerAccumulators, lengths: Optional[Sequence[int]] = None,
                     scale: Optional[float] = None, bias: Optional[float] = None, group=None):
    """Key-split CP forward with the partial-O reduction fused into the kernel epilogue.
    Returns (o_blk [B, H, N/G, d] in q's dtype, q_full)."""
    from .attention import sigattn_cp_finalize, sigattn_fwd_cp
    B, H, n, d = q_blk.shape
    N = shard.N
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    bias = -math.log(N) if bias is None else float(bias)
    q_full = _all_gather_seq(q_blk, shard.world, group)
    lengths = [N] * B if lengths is None else list(lengths)
    nq = torch.tensor(lengths, dtype=torch.int32, device=q_blk.device)
    nk = torch.tensor([shard.local_len(x) for x in lengths], dtype=torch.int32, device=q_blk.device)
    peers.acc.zero_()
    cross_rank_sync(group, q_blk.device)           # every owner's accumulator is zero
    sigattn_fwd_cp(q_full, k_blk, v_blk, nq, nk, scale, bias, peers.table, shard.world, shard.rank)
    cross_rank_sync(group, q_blk.device)           # every rank's reduce-adds have landed
    o_blk = sigattn_cp_finalize(peers.acc, nq, N, shard.world, shard.rank, dtype=q_blk.dtype)
    return o_blk, q_full


def cp_backward_fused(q_full: torch.Tensor, k_blk: torch.Tensor, v_blk: torch.Tensor, do_blk: torch.Tensor,
                      shard: CPShard, peers: PeerAccumulators, lengths: Optional[Sequence[int]] = None,
                      scale: Optional[float] = None, bias: Optional[float] = None, group=None):
    """Key-split CP backward with the dQ reduction fused into the kernel epilogue -> (dq_blk, dk_blk, dv_blk)."""
    from .attention import sigattn_bwd_cp, sigattn_cp_finalize
    B, H, N, d = q_full.shape
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    bias = -math.log(shard.N) if bias is None else float(bias)
    do_full = _all_gather_seq(do_blk, shard.world, group)
    lengths = [shard.N] * B if lengths is None else list(lengths)
    nq = torch.tensor(lengths, dtype=torch.int32, device=q_full.device)
    nk = torch.tensor([shard.local_len(x) for x in lengths], dtype=torch.int32, device=q_full.device)
    peers.acc.zero_()
    cross_rank_sync(group, q_full.device)
    dk_blk, dv_blk = sigattn_bwd_cp(q_full, k_blk, v_blk, do_full, nq, nk, scale, bias, peers.table, shard.world,
                                    shard.rank)
    cross_rank_sync(group, q_full.device)
    dq_blk = sigattn_cp_finalize(peers.acc, nq, shard.N, shard.world, shard.rank, dtype=q_full.dtype)
    return dq_blk, dk_blk, dv_blk
