"""GPU parity of the fused key-split context parallelism (A4).

sigattn_fwd_cp / sigattn_bwd_cp reduce-add every partial O / dQ row from the kernel epilogue
straight into its owner's fp32 accumulator through a device table of peer pointers.  Two checks:

* virtual ranks (one process, one GPU): G accumulators on the device and G calls, one per key
  block, each writing into all G accumulators -- the owner / row arithmetic and the reduction are
  exercised for G = 1, 2, 4 exactly as on G GPUs; the finalised blocks are compared with the fp64
  oracle of the unsplit problem.
* two processes sharing the GPU: the accumulators are exchanged through CUDA IPC
  (sigattn_ipc_export / import, PeerAccumulators) and the ranks run parallel.cp_forward_fused /
  cp_backward_fused over gloo -- the multi-process path of an NVLink run, on one device.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2604_27124_b200 import inputs as I

pytestmark = pytest.mark.gpu
TOL = 1e-2


def f64(t):
    return t.detach().to(torch.float64).cpu().numpy()


def relerr(got, ref):
    den = np.abs(ref).max()
    return float(np.abs(got).max()) if den == 0 else float(np.abs(got - ref).max() / den)


def _cfg(d, lengths, N):
    return I.Config(f"cp_fused_d{d}", B=len(lengths), H=2, N=N, d=d, lengths=lengths, seed=11)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("world,lengths", [(1, [512, 301]), (2, [512, 301]), (4, [512, 130, 0, 385])])
def test_cp_fused_virtual_ranks(d, world, lengths):
    import paper_2604_27124_b200 as sa
    from paper_2604_27124_b200 import attention as A
    N = 512
    cfg = _cfg(d, lengths, N)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1.0 / math.sqrt(d), -math.log(N)
    n = N // world
    B, H = cfg.B, cfg.H
    o_acc = [torch.full((B, H, n, d), float("nan"), device="cuda").zero_() for _ in range(world)]
    dq_acc = [torch.zeros((B, H, n, d), device="cuda") for _ in range(world)]
    o_tab = torch.tensor([t.data_ptr() for t in o_acc], dtype=torch.int64, device="cuda")
    dq_tab = torch.tensor([t.data_ptr() for t in dq_acc], dtype=torch.int64, device="cuda")
    dk_parts, dv_parts = [], []
    for r in range(world):
        sl = slice(r * n, (r + 1) * n)
        kb, vb = k[:, :, sl].contiguous(), v[:, :, sl].contiguous()
        nk_r = torch.tensor([max(0, min(n, L - r * n)) for L in lengths], dtype=torch.int32, device="cuda")
        A.sigattn_fwd_cp(q, kb, vb, nq, nk_r, alpha, b, o_tab, world, r)
        dk_r, dv_r = A.sigattn_bwd_cp(q, kb, vb, do, nq, nk_r, alpha, b, dq_tab, world, r,
                                      dk=torch.full_like(kb, float("nan")), dv=torch.full_like(vb, float("nan")))
        dk_parts.append(dk_r)
        dv_parts.append(dv_r)
    torch.cuda.synchronize()
    o = torch.cat([A.sigattn_cp_finalize(o_acc[r], nq, N, world, r) for r in range(world)], dim=2)
    dq = torch.cat([A.sigattn_cp_finalize(dq_acc[r], nq, N, world, r) for r in range(world)], dim=2)
    dk, dv = torch.cat(dk_parts, dim=2), torch.cat(dv_parts, dim=2)
    bias = np.full(B, b)
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias)
    errs = {}
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        errs[name] = relerr(f64(got), ref)
        assert errs[name] <= TOL, (name, errs[name])
    for bb, L in enumerate(lengths):   # padded rows exact 0
        for t in (o, dq, dk, dv):
            assert torch.all(t[bb, :, L:] == 0)
    print(f"cp fused d={d} G={world}", errs)
    del sa


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, d, lengths, N, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)   # both ranks share the one GPU; their buffers meet through CUDA IPC
        from paper_2604_27124_b200 import parallel as par
        cfg = _cfg(d, lengths, N)
        q, k, v, do, _, _ = I.make_inputs(cfg, "cuda")
        shard = par.CPShard(rank, world, N)
        sl = slice(rank * shard.block, (rank + 1) * shard.block)
        blk = lambda t: t[:, :, sl].contiguous()  # noqa: E731
        peers_o = par.PeerAccumulators(cfg.B, cfg.H, shard.block, d, "cuda")
        peers_dq = par.PeerAccumulators(cfg.B, cfg.H, shard.block, d, "cuda")
        o_blk, q_full = par.cp_forward_fused(blk(q), blk(k), blk(v), shard, peers_o, lengths)
        dq_blk, dk_blk, dv_blk = par.cp_backward_fused(q_full, blk(k), blk(v), blk(do), shard, peers_dq, lengths)
        torch.cuda.synchronize()
        torch.save({n_: t.cpu() for n_, t in (("o", o_blk), ("dq", dq_blk), ("dk", dk_blk), ("dv", dv_blk))},
                   os.path.join(out_dir, f"r{rank}.pt"))
        dist.barrier()
        peers_o.close()
        peers_dq.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d", [64, 128])
def test_cp_fused_two_processes_ipc(tmp_path, d):
    N, lengths, world = 512, [512, 301], 2
    mp.spawn(_ipc_worker, args=(world, _free_port(), d, lengths, N, str(tmp_path)), nprocs=world, join=True)
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    cfg = _cfg(d, lengths, N)
    q, k, v, do, _, _ = I.make_inputs(cfg, "cpu")
    alpha, bias = 1.0 / math.sqrt(d), np.full(cfg.B, -math.log(N))
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias)
    for name, ref in (("o", ro), ("dq", rdq), ("dk", rdk), ("dv", rdv)):
        got = torch.cat([p[name] for p in parts], dim=2)
        e = relerr(f64(got), ref)
        assert e <= TOL, (name, e)
