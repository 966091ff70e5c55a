"""Python boundary of the sigmoid-attention hot path (same names as include/sigattn.h).

Argument marshalling only: tensors are checked, device pointers and the current CUDA stream are
handed to libsigattn.so, and every step of the method (work list, zero fill, the fwd / bwd
kernels, dQ finalisation) runs in the library's kernels.  There is no CPU / PyTorch fallback.

    O = sigma(alpha Q K^T + b) V     (Eq. 2; padding semantics Alg. 1)
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional, Union

import torch

from . import _lib

BiasArg = Union[None, float, str, torch.Tensor]


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SIGATTN_BF16
    if t.dtype == torch.float16:
        return _lib.SIGATTN_FP16
    raise TypeError(f"sigattn: dtype {t.dtype} unsupported (bf16 / fp16)")


_LAYOUTS = ("bhsd", "bshd")


def _check_qkv(q, k, v, layout: str = "bhsd"):
    """Returns B, H, Nq, Nk, d.  layout 'bhsd': tensors are [B, H, N, d]; 'bshd': [B, N, H, d], the
    paper's [Z, L, H, D] -- read in place through strided TMA views."""
    if layout not in _LAYOUTS:
        raise ValueError(f"sigattn: layout must be one of {_LAYOUTS}")
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not t.is_cuda:
            raise ValueError(f"sigattn: {name} must be a CUDA tensor (no CPU fallback)")
        if t.dim() != 4:
            raise ValueError(f"sigattn: {name} must be 4-D ({layout})")
        if not t.is_contiguous():
            raise ValueError(f"sigattn: {name} must be contiguous ({layout})")
    if layout == "bhsd":
        B, H, Nq, d = q.shape
        Nk = k.shape[2]
        ok = k.shape[:2] == (B, H) and k.shape[3] == d
    else:
        B, Nq, H, d = q.shape
        Nk = k.shape[1]
        ok = k.shape[0] == B and k.shape[2:] == (H, d)
    if not ok or v.shape != k.shape:
        raise ValueError(f"sigattn: shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)} ({layout})")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("sigattn: q, k, v must share a dtype")
    return B, H, Nq, Nk, d


def _shape(layout, B, H, N, d):
    return (B, H, N, d) if layout == "bhsd" else (B, N, H, d)


def _layout_flag(layout):
    return _lib.SIGATTN_F_LAYOUT_BSHD if layout == "bshd" else 0


def _lens(t: Optional[torch.Tensor], B: int, device) -> Optional[torch.Tensor]:
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        t = torch.tensor(list(t), dtype=torch.int32)
    t = t.to(device=device, dtype=torch.int32).contiguous()
    if t.numel() != B:
        raise ValueError("sigattn: seqlens must have B entries")
    return t


def resolve_bias(bias: BiasArg, Nk: int, seqlens_k: Optional[torch.Tensor], B: int, device):
    """b = -log n.  None -> scalar -log(Nk) (padded length, reading R1);
    'per_seq' -> device tensor -log(n_k[b]) (Alg. 1's b in R^Z); float; or a [B] tensor."""
    if bias is None:
        return -math.log(Nk), None
    if isinstance(bias, str):
        if bias != "per_seq":
            raise ValueError("sigattn: bias must be None, a float, 'per_seq' or a [B] tensor")
        n = seqlens_k.to(torch.float32) if seqlens_k is not None else torch.full((B,), float(Nk), device=device)
        return 0.0, (-torch.log(torch.clamp(n, min=1.0))).contiguous()
    if isinstance(bias, torch.Tensor):
        t = bias.to(device=device, dtype=torch.float32).reshape(-1).contiguous()
        if t.numel() == 1:
            return float(t.item()), None
        if t.numel() != B:
            raise ValueError("sigattn: bias tensor must have 1 or B entries")
        return 0.0, t
    return float(bias), None


def _ptr(t: Optional[torch.Tensor]):
    return t.data_ptr() if t is not None else None


def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _workspace(ws: Optional[torch.Tensor], need: int, device) -> torch.Tensor:
    """Caller-owned device workspace of at least `need` bytes (allocated here when not given)."""
    if ws is None or ws.numel() * ws.element_size() < need:
        if ws is not None:
            raise ValueError(f"sigattn: workspace too small ({ws.numel() * ws.element_size()} < {need} bytes)")
        return torch.empty(max(need, 1), dtype=torch.uint8, device=device)
    if not ws.is_cuda or ws.device != torch.device(device) or not ws.is_contiguous():
        raise ValueError("sigattn: workspace must be a contiguous CUDA tensor on the inputs' device")
    return ws


def _check_out(name: str, t: torch.Tensor, shape, dtype, device):
    if (tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or not t.is_cuda
            or t.device != device):
        raise ValueError(f"sigattn: {name} must be a contiguous {dtype} CUDA tensor of shape {tuple(shape)} on "
                         f"{device} (got {tuple(t.shape)} {t.dtype} on {t.device})")


def fwd_workspace_bytes(B, H, Nq, Nk, d, dtype=torch.bfloat16) -> int:
    p = _lib.make_params(B, H, Nq, Nk, d, _lib.SIGATTN_BF16 if dtype == torch.bfloat16 else _lib.SIGATTN_FP16,
                         None, None, 1.0, 0.0, None, 0)
    return int(_lib.load().sigattn_fwd_workspace_bytes(ctypes.byref(p)))


def sigattn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seqlens_q=None, seqlens_k=None,
                scale: Optional[float] = None, bias: BiasArg = None, out: Optional[torch.Tensor] = None,
                out_f32: bool = False, zero_pad_out: bool = True, layout: str = "bhsd",
                sanitize_pad: bool = False, workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Forward (Alg. 1).  Returns O [B, H, Nq, d] ([B, Nq, H, d] for layout='bshd') in q.dtype
    (fp32 if out_f32: a CP partial).  workspace: optional uint8 CUDA tensor of at least
    fwd_workspace_bytes(...) bytes (the device work list), reused across calls on one stream."""
    lib = _lib.load()
    B, H, Nq, Nk, d = _check_qkv(q, k, v, layout)
    sq = _lens(seqlens_q, B, q.device)
    sk = _lens(seqlens_k, B, q.device) if seqlens_k is not None else sq if Nk == Nq else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    b_scalar, b_tensor = resolve_bias(bias, Nk, sk, B, q.device)
    odt = torch.float32 if out_f32 else q.dtype
    oshape = _shape(layout, B, H, Nq, d)
    if out is None:
        out = torch.empty(oshape, dtype=odt, device=q.device)
    else:
        _check_out("out", out, oshape, odt, q.device)
    flags = ((_lib.SIGATTN_F_OUT_F32_PARTIAL if out_f32 else 0) | (0 if zero_pad_out else _lib.SIGATTN_F_NO_ZERO_PAD_OUT)
             | _layout_flag(layout) | (_lib.SIGATTN_F_SANITIZE_PAD if sanitize_pad else 0))
    p = _lib.make_params(B, H, Nq, Nk, d, _dtype_code(q), _ptr(sq), _ptr(sk), scale, b_scalar, _ptr(b_tensor), flags)
    need = int(lib.sigattn_fwd_workspace_bytes(ctypes.byref(p)))
    workspace = _workspace(workspace, need, q.device)
    _lib.check(lib.sigattn_fwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                               workspace.data_ptr(), need, _stream_handle(q.device)))
    return out


def bwd_workspace_bytes(B, H, Nq, Nk, d, dtype=torch.bfloat16) -> int:
    p = _lib.make_params(B, H, Nq, Nk, d, _lib.SIGATTN_BF16 if dtype == torch.bfloat16 else _lib.SIGATTN_FP16,
                         None, None, 1.0, 0.0, None, 0)
    return int(_lib.load().sigattn_bwd_workspace_bytes(ctypes.byref(p)))


def sigattn_bwd(q, k, v, dout, seqlens_q=None, seqlens_k=None, scale=None, bias: BiasArg = None,
                dq=None, dk=None, dv=None, workspace: Optional[torch.Tensor] = None, dq_f32: bool = False,
                deterministic: bool = False, dbias: Optional[torch.Tensor] = None, layout: str = "bhsd",
                sanitize_pad: bool = False):
    """Backward (Alg. 2 + Alg. 3, fused).  Returns (dQ, dK, dV); dQ is fp32 if dq_f32 (CP partial).

    deterministic=True runs the paper's two passes instead (dK/dV key-tile-owned, dQ
    query-tile-owned): no atomics, bitwise reproducible, ~40% more tensor work.
    dbias: optional fp32 [B] CUDA tensor that receives dL/db_z = sum over heads and valid (i, j) of
    dS_ij -- the gradient of a learnable per-sequence bias.
    """
    lib = _lib.load()
    B, H, Nq, Nk, d = _check_qkv(q, k, v, layout)
    if dq_f32 and layout != "bhsd":
        raise ValueError("sigattn: dq_f32 (CP partial) needs layout='bhsd'")
    if dout.shape != q.shape or dout.dtype != q.dtype or not dout.is_contiguous():
        raise ValueError("sigattn: dout must match q")
    sq = _lens(seqlens_q, B, q.device)
    sk = _lens(seqlens_k, B, q.device) if seqlens_k is not None else sq if Nk == Nq else None
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    b_scalar, b_tensor = resolve_bias(bias, Nk, sk, B, q.device)
    dq_dtype = torch.float32 if dq_f32 else q.dtype
    dq_shape = _shape(layout, B, H, Nq, d)
    if dq is None:
        dq = torch.empty(dq_shape, dtype=dq_dtype, device=q.device)
    else:
        _check_out("dq", dq, dq_shape, dq_dtype, q.device)
    if dk is None:
        dk = torch.empty_like(k)
    else:
        _check_out("dk", dk, k.shape, k.dtype, q.device)
    if dv is None:
        dv = torch.empty_like(v)
    else:
        _check_out("dv", dv, v.shape, v.dtype, q.device)
    flags = ((_lib.SIGATTN_F_DQ_F32_PARTIAL if dq_f32 else 0) | (_lib.SIGATTN_F_BWD_DETERMINISTIC if deterministic else 0)
             | _layout_flag(layout) | (_lib.SIGATTN_F_SANITIZE_PAD if sanitize_pad else 0))
    if dbias is not None and (dbias.dtype != torch.float32 or dbias.numel() != B or not dbias.is_contiguous()
                              or not dbias.is_cuda or dbias.device != q.device):
        raise ValueError("sigattn: dbias must be a contiguous fp32 CUDA tensor with B entries")
    p = _lib.make_params(B, H, Nq, Nk, d, _dtype_code(q), _ptr(sq), _ptr(sk), scale, b_scalar, _ptr(b_tensor), flags,
                         _ptr(dbias))
    need = int(lib.sigattn_bwd_workspace_bytes(ctypes.byref(p)))
    workspace = _workspace(workspace, need, q.device)
    _lib.check(lib.sigattn_bwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(),
                               dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), workspace.data_ptr(), need,
                               _stream_handle(q.device)))
    return dq, dk, dv


def _mask_lens_and_flag(key_padding_mask: torch.Tensor):
    """(seqlens [B] int32 on device, whether the mask is non-prefix) -- both from the library kernel."""
    lib = _lib.load()
    m = key_padding_mask.to(torch.uint8).contiguous()
    B, N = m.shape
    seqlens = torch.empty(B, dtype=torch.int32, device=m.device)
    flag = torch.empty(1, dtype=torch.int32, device=m.device)
    _lib.check(lib.sigattn_mask_to_seqlens(m.data_ptr(), B, N, seqlens.data_ptr(), flag.data_ptr(),
                                           _stream_handle(m.device)))
    return seqlens, int(flag.item()) != 0


def sigattn_mask_to_seqlens(key_padding_mask: torch.Tensor, check_prefix: bool = True) -> torch.Tensor:
    """PyTorch key_padding_mask [B, N] (True = pad) -> int32 valid lengths, on device."""
    lib = _lib.load()
    m = key_padding_mask.to(torch.uint8).contiguous()
    B, N = m.shape
    seqlens = torch.empty(B, dtype=torch.int32, device=m.device)
    flag = torch.empty(1, dtype=torch.int32, device=m.device)
    _lib.check(lib.sigattn_mask_to_seqlens(m.data_ptr(), B, N, seqlens.data_ptr(), flag.data_ptr(),
                                           _stream_handle(m.device)))
    if check_prefix and int(flag.item()) != 0:
        raise ValueError("sigattn: key_padding_mask is not a prefix mask (valid tokens after padding)")
    return seqlens


def sigattn_mask_to_index(key_padding_mask: torch.Tensor):
    """General key_padding_mask [B, N] (True = pad) -> (index [B, N] int32, seqlens [B] int32), on
    device: index lists each sequence's valid positions in order, then its padded ones."""
    lib = _lib.load()
    m = key_padding_mask.to(torch.uint8).contiguous()
    B, N = m.shape
    index = torch.empty((B, N), dtype=torch.int32, device=m.device)
    seqlens = torch.empty(B, dtype=torch.int32, device=m.device)
    _lib.check(lib.sigattn_mask_to_index(m.data_ptr(), B, N, index.data_ptr(), seqlens.data_ptr(),
                                         _stream_handle(m.device)))
    return index, seqlens


def copy_valid_rows(src: torch.Tensor, dst: torch.Tensor, lens, layout: str = "bhsd") -> int:
    """Padding-aware transfer: copy only rows [0, lens[b]) of every (b, h) slab of src into dst (host
    <-> device or device <-> device, asynchronous on the current stream of the CUDA side); rows past
    lens[b] of dst are left as they are.  lens: host sequence of B ints (a CPU tensor or list).
    Returns the bytes copied.  See include/sigattn.h sigattn_copy_valid_rows."""
    lib = _lib.load()
    if src.shape != dst.shape or src.dtype != dst.dtype or not src.is_contiguous() or not dst.is_contiguous():
        raise ValueError("sigattn: copy_valid_rows needs contiguous tensors of one shape and dtype")
    if src.is_cuda == dst.is_cuda and not src.is_cuda:
        raise ValueError("sigattn: copy_valid_rows copies to or from a CUDA tensor")
    if src.dim() != 4:
        raise ValueError("sigattn: copy_valid_rows needs a [B, H, N, d] (or [B, N, H, d]) tensor")
    B = src.shape[0]
    H, N = (src.shape[2], src.shape[1]) if layout == "bshd" else (src.shape[1], src.shape[2])
    lens_h = torch.as_tensor(lens, dtype=torch.int32).cpu().contiguous()
    if lens_h.numel() != B:
        raise ValueError("sigattn: lens must have B entries")
    kind = 1 if dst.is_cuda and not src.is_cuda else 2 if src.is_cuda and not dst.is_cuda else 3
    dev = dst.device if dst.is_cuda else src.device
    nbytes = ctypes.c_int64(0)
    _lib.check(lib.sigattn_copy_valid_rows(src.data_ptr(), dst.data_ptr(), B, H, N,
                                           src.shape[-1] * src.element_size(), lens_h.data_ptr(),
                                           1 if layout == "bshd" else 0, kind, _stream_handle(dev),
                                           ctypes.byref(nbytes)))
    return int(nbytes.value)


def sigattn_permute_rows(x: torch.Tensor, index: torch.Tensor, scatter: bool) -> torch.Tensor:
    """[B, H, N, d] row gather (out[:, :, r] = x[:, :, index[r]]) or scatter (out[:, :, index[r]] = x[:, :, r])."""
    lib = _lib.load()
    if not x.is_contiguous() or x.dim() != 4:
        raise ValueError("sigattn: permute_rows needs a contiguous [B, H, N, d] tensor")
    B, H, N, d = x.shape
    out = torch.empty_like(x)
    _lib.check(lib.sigattn_permute_rows(x.data_ptr(), out.data_ptr(), index.data_ptr(), B, H, N, d,
                                        1 if scatter else 0, _stream_handle(x.device)))
    return out


class _PermuteRows(torch.autograd.Function):
    """Row permutation along N; its gradient is the inverse permutation (library kernels both ways)."""

    @staticmethod
    def forward(ctx, x, index, scatter):
        ctx.save_for_backward(index)
        ctx.scatter = scatter
        return sigattn_permute_rows(x, index, scatter)

    @staticmethod
    def backward(ctx, g):
        (index,) = ctx.saved_tensors
        return sigattn_permute_rows(g.contiguous(), index, not ctx.scatter), None, None


def valid_flops(B: int, H: int, d: int, nq, nk, forward: bool) -> int:
    """App. B.1 FLOP credit on valid tokens: sum_b {4|10} H d n_q[b] n_k[b]."""
    import numpy as np
    a = np.ascontiguousarray(np.asarray(nq, dtype=np.int32))
    c = np.ascontiguousarray(np.asarray(nk, dtype=np.int32))
    r = _lib.load().sigattn_valid_flops(int(B), int(H), int(d), a.ctypes.data, c.ctypes.data, 1 if forward else 0)
    if r < 0:
        raise ValueError("sigattn_valid_flops: bad arguments")
    return int(r)


def worklist_host(kind: int, B: int, H: int, Nq: int, Nk: int, nq, nk):
    """Host mirror of the device work list: list of (b, h, tile, cost) in visiting order."""
    import numpy as np
    lib = _lib.load()
    a = np.ascontiguousarray(np.asarray(nq, dtype=np.int32))
    c = np.ascontiguousarray(np.asarray(nk, dtype=np.int32))
    n = lib.sigattn_worklist_host(kind, B, H, Nq, Nk, a.ctypes.data, c.ctypes.data, None, 0)
    if n < 0:
        raise ValueError("sigattn_worklist_host: bad arguments")
    out = np.zeros((max(n, 1), 4), dtype=np.int32)
    lib.sigattn_worklist_host(kind, B, H, Nq, Nk, a.ctypes.data, c.ctypes.data, out.ctypes.data, n)
    return [tuple(int(x) for x in r) for r in out[:n]]


class SigmoidAttentionFn(torch.autograd.Function):
    """Autograd op: saves q, k, v and the lengths -- never O or P (P is recomputed)."""

    @staticmethod
    def forward(ctx, q, k, v, seqlens_q, seqlens_k, scale, bias, deterministic=False, layout="bhsd"):
        o = sigattn_fwd(q, k, v, seqlens_q, seqlens_k, scale, bias, layout=layout)
        ctx.layout = layout
        ctx.save_for_backward(q, k, v, seqlens_q, seqlens_k, bias if isinstance(bias, torch.Tensor) else None)
        ctx.scale = scale
        ctx.bias = None if isinstance(bias, torch.Tensor) else bias
        ctx.deterministic = deterministic
        # a bias tensor that requires grad is a learnable bias ("fixed or learnable"): one value
        # per sequence ([B]) or one shared scalar (1 element; its gradient is the sum over sequences)
        ctx.bias_grad = (isinstance(bias, torch.Tensor) and bias.requires_grad
                         and bias.numel() in (1, q.shape[0]))
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, sq, sk, bt = ctx.saved_tensors
        bias = bt if bt is not None else ctx.bias
        db = torch.empty(q.shape[0], dtype=torch.float32, device=q.device) if ctx.bias_grad else None
        dq, dk, dv = sigattn_bwd(q, k, v, do.contiguous(), sq, sk, ctx.scale, bias,
                                 deterministic=ctx.deterministic, dbias=db, layout=ctx.layout)
        dbias = None
        if db is not None:
            dbias = (db.sum() if bt.numel() == 1 else db).to(bt.dtype).reshape(bt.shape)
        return dq, dk, dv, None, None, None, dbias, None, None


def sigmoid_attention(q, k, v, seqlens_q=None, seqlens_k=None, key_padding_mask=None,
                      scale: Optional[float] = None, bias: BiasArg = None, deterministic: bool = False,
                      layout: str = "bhsd"):
    """O = sigma(scale * Q K^T + bias) V with padded keys at zero weight; differentiable.

    deterministic=True selects the paper's two-pass backward (bitwise reproducible dQ).

    q [B,H,Nq,d], k/v [B,H,Nk,d] (bf16/fp16, CUDA, contiguous) -- or, with layout='bshd', the
    paper's [B,N,H,d].  Lengths as int32 [B] tensors, or a PyTorch key_padding_mask [B, Nk]
    (True = pad; prefix masks only).
    """
    ndim = 2 if layout == "bhsd" else 1
    if key_padding_mask is not None:
        if seqlens_k is not None:
            raise ValueError("give seqlens or key_padding_mask, not both")
        lens, nonprefix = _mask_lens_and_flag(key_padding_mask)
        if nonprefix:
            # general mask: compact every sequence (stable), attend with prefix lengths, scatter back
            # -- exact, the op is equivariant under a joint permutation of queries and keys (Eq. 2)
            if layout != "bhsd" or q.shape[2] != k.shape[2] or seqlens_q is not None:
                raise ValueError("sigattn: a non-prefix key_padding_mask needs self-attention in 'bhsd' layout")
            index, lens = sigattn_mask_to_index(key_padding_mask)
            qc, kc, vc = (_PermuteRows.apply(t.contiguous(), index, False) for t in (q, k, v))
            oc = SigmoidAttentionFn.apply(qc, kc, vc, lens, lens, scale, bias, deterministic, layout)
            return _PermuteRows.apply(oc, index, True)
        seqlens_k = lens
        if seqlens_q is None and q.shape[ndim] == k.shape[ndim]:
            seqlens_q = seqlens_k
    B = q.shape[0]
    sq = _lens(seqlens_q, B, q.device)
    sk = _lens(seqlens_k, B, q.device)
    if sk is None and sq is not None and q.shape[ndim] == k.shape[ndim]:
        sk = sq
    return SigmoidAttentionFn.apply(q, k, v, sq, sk, scale, bias, deterministic, layout)


# ------------------------------------------------------------------------------------------------
# key-split context parallelism with the reduction fused into the kernels (include/sigattn.h,
# sigattn_fwd_cp / sigattn_bwd_cp / sigattn_cp_finalize; A4).  peer_table: int64 CUDA tensor
# [world] of device pointers to every rank's fp32 accumulator [B, H, Nq / world, d] (see
# parallel.PeerAccumulators); the orchestration (zeroing, cross-rank ordering) is the caller's.
def _cp_params(world: int, rank: int, peer_table: torch.Tensor, device):
    if peer_table.dtype != torch.int64 or peer_table.numel() != world or not peer_table.is_cuda \
            or peer_table.device != device:
        raise ValueError("sigattn: peer_table must be an int64 CUDA tensor of `world` device pointers on the "
                         "inputs' device")
    return _lib.SigattnCpParams(int(world), int(rank), peer_table.data_ptr())


def sigattn_fwd_cp(q, k, v, seqlens_q, seqlens_k, scale, bias: float, peer_table: torch.Tensor, world: int,
                   rank: int, workspace: Optional[torch.Tensor] = None):
    """Partial forward over this rank's key block, reduce-added into the owners' accumulators.
    q: all queries [B, H, Nq, d]; k, v: this rank's block [B, H, Nk, d]; bias: the GLOBAL scalar b."""
    lib = _lib.load()
    B, H, Nq, Nk, d = _check_qkv(q, k, v, "bhsd")
    sq = _lens(seqlens_q, B, q.device)
    sk = _lens(seqlens_k, B, q.device)
    p = _lib.make_params(B, H, Nq, Nk, d, _dtype_code(q), _ptr(sq), _ptr(sk), float(scale), float(bias), None, 0)
    cp = _cp_params(world, rank, peer_table, q.device)
    need = int(lib.sigattn_fwd_workspace_bytes(ctypes.byref(p)))
    workspace = _workspace(workspace, need, q.device)
    _lib.check(lib.sigattn_fwd_cp(ctypes.byref(p), ctypes.byref(cp), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                  workspace.data_ptr(), need, _stream_handle(q.device)))


def sigattn_bwd_cp(q, k, v, dout, seqlens_q, seqlens_k, scale, bias: float, peer_table: torch.Tensor, world: int,
                   rank: int, dk=None, dv=None, workspace: Optional[torch.Tensor] = None):
    """Backward over this rank's key block: returns (dK, dV) of the block (complete); alpha dS K, summed
    over this rank's key tiles, is reduce-added into the owners' fp32 dQ accumulators by the library's
    push kernel.  dout: all queries [B, H, Nq, d]."""
    lib = _lib.load()
    B, H, Nq, Nk, d = _check_qkv(q, k, v, "bhsd")
    if dout.shape != q.shape or dout.dtype != q.dtype or not dout.is_contiguous():
        raise ValueError("sigattn: dout must match q")
    sq = _lens(seqlens_q, B, q.device)
    sk = _lens(seqlens_k, B, q.device)
    if dk is None:
        dk = torch.empty_like(k)
    else:
        _check_out("dk", dk, k.shape, k.dtype, q.device)
    if dv is None:
        dv = torch.empty_like(v)
    else:
        _check_out("dv", dv, v.shape, v.dtype, q.device)
    p = _lib.make_params(B, H, Nq, Nk, d, _dtype_code(q), _ptr(sq), _ptr(sk), float(scale), float(bias), None, 0)
    cp = _cp_params(world, rank, peer_table, q.device)
    need = int(lib.sigattn_bwd_cp_workspace_bytes(ctypes.byref(p)))
    workspace = _workspace(workspace, need, q.device)
    _lib.check(lib.sigattn_bwd_cp(ctypes.byref(p), ctypes.byref(cp), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                  dout.data_ptr(), dk.data_ptr(), dv.data_ptr(), workspace.data_ptr(), need,
                                  _stream_handle(q.device)))
    return dk, dv


def sigattn_cp_finalize(acc: torch.Tensor, seqlens_q, Nq: int, world: int, rank: int, dtype=torch.bfloat16,
                        out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """This rank's complete fp32 accumulator [B, H, Nq / world, d] -> [B, H, Nq / world, d] in dtype,
    rows past the global valid length exact 0."""
    lib = _lib.load()
    if acc.dtype != torch.float32 or acc.dim() != 4 or not acc.is_contiguous() or not acc.is_cuda:
        raise ValueError("sigattn: acc must be a contiguous fp32 CUDA tensor [B, H, Nq / world, d]")
    B, H, rows, d = acc.shape
    if rows * world != Nq:
        raise ValueError("sigattn: acc rows must be Nq / world")
    sq = _lens(seqlens_q, B, acc.device)
    if out is None:
        out = torch.empty(acc.shape, dtype=dtype, device=acc.device)
    else:
        _check_out("out", out, acc.shape, dtype, acc.device)
    code = _lib.SIGATTN_BF16 if dtype == torch.bfloat16 else _lib.SIGATTN_FP16
    p = _lib.make_params(B, H, Nq, Nq, d, code, _ptr(sq), None, 1.0, 0.0, None, 0)
    _lib.check(lib.sigattn_cp_finalize(ctypes.byref(p), int(world), int(rank), acc.data_ptr(), out.data_ptr(),
                                       _stream_handle(acc.device)))
    return out


def ipc_export(t: torch.Tensor) -> bytes:
    """CUDA IPC handle (plus offset) of a device tensor's memory, for another process's ipc_import."""
    lib = _lib.load()
    n = int(lib.sigattn_ipc_handle_bytes())
    buf = ctypes.create_string_buffer(n)
    _lib.check(lib.sigattn_ipc_export(t.data_ptr(), buf))
    return buf.raw


def ipc_import(handle: bytes) -> int:
    """Maps another process's exported buffer on the current device; returns the device pointer."""
    lib = _lib.load()
    ptr = ctypes.c_void_p()
    _lib.check(lib.sigattn_ipc_import(ctypes.c_char_p(handle), ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.load().sigattn_ipc_close(ctypes.c_void_p(ptr)))
