"""Multi-process (gloo, CPU) tests of the multi-GPU plumbing in paper_2604_27124_b200.parallel.

The key-split context-parallel orchestration (all-gather Q / dO, fp32 partials, reduce-scatter over
query blocks, global bias, per-shard key lengths) is driven through torch.distributed exactly as on
GPUs; only the per-rank attention call is a CPU stand-in (the fp64 oracle), so the collectives'
layouts and the additivity of sigmoid attention over key blocks are checked end to end.
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
from paper_2604_27124_b200 import parallel as par


def test_lpt_assign_balance_and_cover():
    costs = [n * n for n in I.C3_LENGTHS for _ in range(12)]
    for world in (1, 2, 4, 8):
        bins = par.lpt_assign(costs, world)
        flat = sorted(i for b in bins for i in b)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in b) for b in bins]
        lower = max(sum(costs) / world, max(costs))
        assert max(loads) <= 1.05 * lower, (world, max(loads) / lower)
    assert par.lpt_assign([5, 1, 1, 1], 2) == [[0], [1, 2, 3]]


def test_shard_pairs_and_gather():
    B, H, N, d = 3, 2, 8, 4
    t = torch.arange(B * H * N * d, dtype=torch.float32).reshape(B, H, N, d)
    shards = par.shard_pairs(B, H, [8, 2, 5], [8, 2, 5], 2)
    assert sorted(p for s in shards for p in s) == [(b, h) for b in range(B) for h in range(H)]
    g = par.gather_pairs(t, shards[0])
    for i, (b, h) in enumerate(shards[0]):
        assert torch.equal(g[i, 0], t[b, h])
    lens = par.pair_lengths(torch.tensor([8, 2, 5]), shards[1], N, "cpu")
    assert lens.tolist() == [[8, 2, 5][b] for b, _ in shards[1]]


def test_cp_shard_lengths():
    s = par.CPShard(rank=2, world=4, N=64)
    assert s.block == 16
    assert [par.CPShard(r, 4, 64).local_len(40) for r in range(4)] == [16, 16, 8, 0]
    with pytest.raises(ValueError):
        par.CPShard(0, 3, 64).block


# ---------------------------------------------------------------- gloo world > 1
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_fwd(q, k, v, nq, nk, scale, bias):
    o = oracle.fwd(q.numpy(), k.numpy(), v.numpy(), nq.tolist(), nk.tolist(), scale, np.full(q.shape[0], bias))
    return torch.from_numpy(o)


def _oracle_bwd(q, k, v, do, nq, nk, scale, bias):
    dq, dk, dv = oracle.bwd(q.numpy(), k.numpy(), v.numpy(), do.numpy(), nq.tolist(), nk.tolist(), scale,
                            np.full(q.shape[0], bias))
    return torch.from_numpy(dq), torch.from_numpy(dk), torch.from_numpy(dv)


def _cp_worker(rank, world, port, lengths, N, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, d = len(lengths), 2, 8
        g = torch.Generator().manual_seed(7)
        q, k, v, do = (torch.randn((B, H, N, d), generator=g, dtype=torch.float64) for _ in range(4))
        for b, n in enumerate(lengths):
            for t in (q, k, v, do):
                t[b, :, n:] = 0
        shard = par.CPShard(rank, world, N)
        sl = slice(rank * shard.block, (rank + 1) * shard.block)
        blk = lambda t: t[:, :, sl].contiguous()  # noqa: E731
        o_blk, q_full = par.cp_forward(blk(q), blk(k), blk(v), shard, lengths, impl_fwd=_oracle_fwd)
        dq_blk, dk_blk, dv_blk = par.cp_backward(q_full, blk(k), blk(v), blk(do), shard, lengths,
                                                 impl_bwd=_oracle_bwd)
        torch.save({"o": o_blk, "dq": dq_blk, "dk": dk_blk, "dv": dv_blk, "q_full": q_full},
                   os.path.join(result_dir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,lengths", [(2, [32, 32]), (2, [32, 19]), (4, [32, 7])])
def test_cp_key_split_matches_unsplit_oracle(tmp_path, world, lengths):
    N = 32
    mp.spawn(_cp_worker, args=(world, _free_port(), lengths, N, str(tmp_path)), nprocs=world, join=True)
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    B, H, d = len(lengths), 2, 8
    g = torch.Generator().manual_seed(7)
    q, k, v, do = (torch.randn((B, H, N, d), generator=g, dtype=torch.float64) for _ in range(4))
    for b, n in enumerate(lengths):
        for t in (q, k, v, do):
            t[b, :, n:] = 0
    alpha, bias = 1 / math.sqrt(d), np.full(B, -math.log(N))
    ro = oracle.fwd(q.numpy(), k.numpy(), v.numpy(), lengths, lengths, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(q.numpy(), k.numpy(), v.numpy(), do.numpy(), lengths, lengths, alpha, bias)
    cat = lambda key: torch.cat([p[key] for p in parts], dim=2).numpy()  # noqa: E731
    assert np.abs(parts[0]["q_full"].numpy() - q.numpy()).max() == 0          # all-gather layout
    for name, got, ref in (("o", cat("o"), ro), ("dq", cat("dq"), rdq), ("dk", cat("dk"), rdk), ("dv", cat("dv"), rdv)):
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), name
