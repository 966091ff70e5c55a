"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same inputs.

Bar (BASELINE.json north star): max|gpu - ref| / max|ref| <= 1e-2 for bf16 (O, dQ, dK, dV) and
<= 2e-3 for the fp16 forward; padded rows exactly 0; finite pad content never changes O, dK, dV.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2604_27124_b200 import inputs as I

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
FP16_FWD_TOL = 2e-3


def _sa():
    import paper_2604_27124_b200 as sa
    return sa


def f64(t):
    return t.detach().to(torch.float64).cpu().numpy()


def relerr(got, ref):
    den = np.abs(ref).max()
    if den == 0:
        return float(np.abs(got).max())
    return float(np.abs(got - ref).max() / den)


def run_case(cfg, bias=None, check_bwd=True, pad=None, tol=BF16_TOL, nan_prefill=False, deterministic=False):
    """nan_prefill: outputs are preallocated full of NaN, so every element (padded rows included)
    must be written by the kernels (the pad fill runs inside the attention kernels)."""
    sa = _sa()
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda", pad=pad)
    alpha = 1.0 / math.sqrt(cfg.d)
    b = -math.log(cfg.N_k) if bias is None else bias
    nan = (lambda t: torch.full_like(t, float("nan"))) if nan_prefill else (lambda t: None)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=nan(q))
    torch.cuda.synchronize()
    bias_np = np.full(cfg.B, b) if np.isscalar(b) else b.double().cpu().numpy()
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias_np)
    e = relerr(f64(o), ro)
    assert e <= tol, f"O rel err {e}"
    for bb in range(cfg.B):
        assert torch.all(o[bb, :, cfg.nq[bb]:] == 0), "padded query rows must be exactly 0"
    res = {"o": e}
    if check_bwd:
        dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, dq=nan(q), dk=nan(k), dv=nan(v),
                                    deterministic=deterministic)
        torch.cuda.synchronize()
        rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias_np)
        for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            err = relerr(f64(got), ref)
            res[name] = err
            assert err <= BF16_TOL, f"{name} rel err {err}"
        for bb in range(cfg.B):
            assert torch.all(dq[bb, :, cfg.nq[bb]:] == 0)
            assert torch.all(dk[bb, :, cfg.nk[bb]:] == 0) and torch.all(dv[bb, :, cfg.nk[bb]:] == 0)
    return res


def test_c1_bf16_fwd_bwd():
    """BASELINE config 1: B=2 H=2 N=256 d=64, lengths {256, 97}, b = -log N, fwd+bwd vs oracle."""
    r = run_case(I.C1)
    print("C1 bf16", r)


def test_c1_fp16_fwd():
    r = run_case(I.C1_FP16, check_bwd=False, tol=FP16_FWD_TOL)
    print("C1 fp16", r)


def test_c1_fp16_bwd():
    run_case(I.C1_FP16, check_bwd=True, tol=FP16_FWD_TOL)


@pytest.mark.parametrize("cfg", [
    I.Config("ragged_N200", B=4, H=3, N=200, d=64, lengths=[200, 1, 129, 127], seed=3),
    I.Config("ragged_N384", B=3, H=2, N=384, d=64, lengths=[384, 255, 257], seed=4),
    I.Config("zero_len", B=3, H=2, N=256, d=64, lengths=[0, 256, 5], seed=5),
    I.Config("unpadded_N512", B=1, H=4, N=512, d=64, seed=6),
    I.Config("many_short", B=40, H=2, N=128, d=64, lengths=[1 + (7 * i) % 128 for i in range(40)], seed=7),
])
def test_ragged_and_edge_cases(cfg):
    run_case(cfg)


@pytest.mark.parametrize("cfg", [
    I.Config("nan_ragged", B=5, H=2, N=300, d=64, lengths=[300, 1, 129, 0, 256], seed=20),
    I.Config("nan_cross", B=3, H=2, N=320, d=64, lengths=[320, 0, 7], Nk=200, lengths_k=[200, 150, 0], seed=21),
    I.Config("nan_d128", B=4, H=2, N=300, d=128, lengths=[300, 65, 0, 128], seed=22),
    I.Config("nan_d128_cross", B=3, H=2, N=200, d=128, lengths=[200, 63, 9], Nk=330, lengths_k=[0, 330, 129], seed=23),
])
def test_every_output_element_written(cfg):
    """Outputs prefilled with NaN: valid rows match the oracle and every padded row is exactly 0."""
    run_case(cfg, nan_prefill=True)


def test_cross_lengths_nq_ne_nk():
    cfg = I.Config("cross", B=3, H=2, N=320, d=64, lengths=[320, 100, 7], Nk=200, lengths_k=[200, 150, 1], seed=8)
    run_case(cfg)


def test_per_sequence_bias():
    cfg = I.Config("perseq", B=3, H=2, N=256, d=64, lengths=[256, 60, 200], seed=9)
    b = -torch.log(torch.tensor(cfg.nk, dtype=torch.float32)).cuda()
    run_case(cfg, bias=b)


@pytest.mark.parametrize("cfg", [
    I.Config("d128", B=2, H=2, N=256, d=128, lengths=[256, 97], seed=10),
    I.Config("d128_ragged", B=3, H=2, N=300, d=128, lengths=[300, 129, 1], seed=11),
])
def test_d128_fwd_bwd(cfg):
    run_case(cfg)


def test_d128_fp16():
    cfg = I.Config("d128f16", B=2, H=2, N=256, d=128, lengths=[256, 97], dtype="fp16", seed=12)
    run_case(cfg, tol=FP16_FWD_TOL)


@pytest.mark.parametrize("cfg", [
    I.Config("d128_many", B=9, H=3, N=200, d=128, lengths=[200, 1, 63, 64, 65, 127, 128, 129, 0], seed=18),
    I.Config("d128_cross", B=2, H=2, N=320, d=128, lengths=[320, 100], Nk=192, lengths_k=[192, 70], seed=19),
])
def test_d128_ragged_edges(cfg):
    run_case(cfg)


def test_pad_independence_bitwise():
    """Finite pad content (0 vs 1e3 vs random) leaves O, dK, dV bitwise equal; dQ within tol."""
    sa = _sa()
    cfg = I.Config("padind", B=3, H=2, N=256, d=64, lengths=[256, 97, 130], seed=13)
    outs = []
    for pad in (None, 1e3, "random"):
        q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda", pad=pad)
        o = sa.sigattn_fwd(q, k, v, nq, nk)
        dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk)
        outs.append((o, dq, dk, dv))
    for o, dq, dk, dv in outs[1:]:
        assert torch.equal(o, outs[0][0])
        assert torch.equal(dk, outs[0][2]) and torch.equal(dv, outs[0][3])
        assert relerr(f64(dq), f64(outs[0][1])) < 1e-2


def test_forward_deterministic():
    sa = _sa()
    q, k, v, do, nq, nk = I.make_inputs(I.C1, "cuda")
    o1 = sa.sigattn_fwd(q, k, v, nq, nk)
    o2 = sa.sigattn_fwd(q, k, v, nq, nk)
    assert torch.equal(o1, o2)


def test_cp_partial_sum_fp32():
    """Key-split partials (fp32 out) summed == unsplit O (A4) within bf16 tolerance."""
    sa = _sa()
    cfg = I.Config("cp", B=1, H=2, N=512, d=64, seed=14)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    b = -math.log(512)
    full = sa.sigattn_fwd(q, k, v, None, None, None, b, out_f32=True)
    parts = [sa.sigattn_fwd(q, k[:, :, lo:lo + 128].contiguous(), v[:, :, lo:lo + 128].contiguous(), None, None,
                            None, b, out_f32=True) for lo in range(0, 512, 128)]
    s = sum(parts)
    ro = oracle.fwd(f64(q), f64(k), f64(v), [512], [512], 1 / 8, [b])
    assert relerr(f64(s), ro) <= BF16_TOL
    assert relerr(f64(full), ro) <= BF16_TOL


def test_autograd_and_mask_path():
    sa = _sa()
    cfg = I.Config("ag", B=2, H=2, N=256, d=64, lengths=[256, 77], seed=15)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    mask = torch.arange(256, device="cuda")[None, :] >= nk[:, None]
    assert torch.equal(sa.sigattn_mask_to_seqlens(mask), nk)
    bad = mask.clone(); bad[0, 3] = True
    with pytest.raises(ValueError):
        sa.sigattn_mask_to_seqlens(bad)
    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
    o = sa.sigmoid_attention(qq, kk, vv, key_padding_mask=mask)
    o.backward(do)
    alpha = 1 / 8
    bias = np.full(2, -math.log(256))
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias)
    assert relerr(f64(o), ro) <= BF16_TOL
    for got, ref in ((qq.grad, rdq), (kk.grad, rdk), (vv.grad, rdv)):
        assert relerr(f64(got), ref) <= BF16_TOL


def _sampled_rows(n, N, rng, k=96):
    """Boundary rows of every tile around n plus random rows."""
    rows = {0, max(n - 1, 0), min(n, N - 1), N - 1}
    for t in range(0, N, 128):
        rows.update({t, min(t + 127, N - 1)})
    rows.update(rng.integers(0, N, size=k).tolist())
    return sorted(rows)


def test_c3_full_size_sampled():
    """C3 (B=32 N=8192 H=12 d=64 jagged) at full size, in the bench's launch configuration:
    sampled rows of several (b, h) against the row-sampled oracle."""
    sa = _sa()
    cfg = I.C3
    q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
    alpha, b = 1 / 8, -math.log(8192)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    bias = np.full(cfg.B, b)
    for (bb, hh) in [(30, 0), (30, 11), (24, 5), (0, 3), (22, 7)]:
        qs, ks, vs, dos = (f64(t[bb:bb + 1, hh:hh + 1]) for t in (q, k, v, do))
        nqb, nkb = [cfg.nq[bb]], [cfg.nk[bb]]
        rows = _sampled_rows(cfg.nq[bb], cfg.N, rng)
        ro = oracle.fwd_rows(qs, ks, vs, 0, 0, rows, nqb, nkb, alpha, [b])
        rdq = oracle.dq_rows(qs, ks, vs, dos, 0, 0, rows, nqb, nkb, alpha, [b])
        rdk, rdv = oracle.dkdv_rows(qs, ks, vs, dos, 0, 0, rows, nqb, nkb, alpha, [b])
        for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            g = f64(got[bb, hh])[rows]
            err = relerr(g, ref)
            assert err <= BF16_TOL, f"{name} (b={bb}, h={hh}) rel err {err}"


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bias,scale", [(0.0, None), (3.0, None), (-1.0, 0.5), (-30.0, None), (-3.2, 0.02),
                                        (-4.6, 0.01), (-5.5, None), (-8.5, 0.5), (-12.0, 1.0)])
def test_sigmoid_slow_and_saturated_paths(bias, scale, d):
    """Logits above -2 (bias 0 / +3 / large scale) exercise the exact-range sigma path; logits in
    (-4, -2] the quadratic tier (bias -3.2, scale 0.02); <= -4 the linear tier (bias -4.6); bias -5.5
    with unit-variance logits fails the tier-4 vote in some chunks only (speculation on/off per warp);
    bias -30 saturates to P ~ 0.  Biases <= -8.3 make the forward and the d = 128 backward speculate
    the <= -4 tier (kSpec4MaxBias); with large scales (-8.5 / 0.5, -12 / 1.0) that speculation fails
    in many chunks (reload from TMEM, exact tiers).  Both kernels, d = 64 and 128, must stay within the
    bf16 bound."""
    sa = _sa()
    cfg = I.Config("slowpath", B=2, H=2, N=256, d=d, lengths=[256, 150], seed=21)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha = 1.0 / math.sqrt(cfg.d) if scale is None else scale
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, bias)
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, bias)
    bias_np = np.full(cfg.B, bias)
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias_np)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias_np)
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        err = relerr(f64(got), ref)
        assert err <= BF16_TOL, f"{name} rel err {err} (bias={bias}, scale={scale})"


@pytest.mark.parametrize("d", [64, 128])
def test_cp_backward_partials_sum(d):
    """Key-split backward: per-block fp32 dQ partials (DQ_F32_PARTIAL) sum to dQ; dK/dV blocks are
    the unsplit dK/dV rows (keys are owned) -- the CP exchange of SURVEY 8e, simulated on one GPU."""
    sa = _sa()
    cfg = I.Config("cpb", B=2, H=2, N=512, d=d, lengths=[512, 300], seed=16)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    b = -math.log(512)
    G, blk = 4, 128
    dq_sum = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
    dks, dvs = [], []
    for r in range(G):
        ks, vs = (t[:, :, r * blk:(r + 1) * blk].contiguous() for t in (k, v))
        nk_r = torch.clamp(nk - r * blk, 0, blk).to(torch.int32)
        dq_r, dk_r, dv_r = sa.sigattn_bwd(q, ks, vs, do, nq, nk_r, None, b, dq_f32=True)
        assert dq_r.dtype == torch.float32
        dq_sum += dq_r
        dks.append(dk_r)
        dvs.append(dv_r)
    bias = np.full(2, b)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, 1 / math.sqrt(d), bias)
    assert relerr(f64(dq_sum), rdq) <= BF16_TOL
    assert relerr(f64(torch.cat(dks, 2)), rdk) <= BF16_TOL
    assert relerr(f64(torch.cat(dvs, 2)), rdv) <= BF16_TOL


def test_cp_autograd_world1_nccl():
    """cp_sigmoid_attention through torch.distributed (NCCL, world 1) + autograd."""
    import os
    import torch.distributed as dist
    from paper_2604_27124_b200 import parallel as par
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29641")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
        created = True
    try:
        cfg = I.Config("cpw1", B=1, H=2, N=256, d=64, seed=17)
        q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
        qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
        o = par.cp_sigmoid_attention(qq, kk, vv, par.CPShard(0, 1, 256))
        o.backward(do)
        b = np.full(1, -math.log(256))
        ro = oracle.fwd(f64(q), f64(k), f64(v), [256], [256], 1 / 8, b)
        rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), [256], [256], 1 / 8, b)
        assert relerr(f64(o), ro) <= BF16_TOL
        for got, ref in ((qq.grad, rdq), (kk.grad, rdk), (vv.grad, rdv)):
            assert relerr(f64(got), ref) <= BF16_TOL
    finally:
        if created:
            dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------
# deterministic backward: the paper's Alg. 2 (query-tile-owned dQ) + Alg. 3 (key-tile-owned dK/dV)
@pytest.mark.parametrize("cfg", [
    I.C1,
    I.C1_FP16,
    I.Config("det_ragged", B=5, H=2, N=300, d=64, lengths=[300, 1, 129, 0, 256], seed=30),
    I.Config("det_cross", B=3, H=2, N=320, d=64, lengths=[320, 0, 7], Nk=200, lengths_k=[200, 150, 0], seed=31),
    I.Config("det_d128", B=4, H=2, N=300, d=128, lengths=[300, 65, 0, 128], seed=32),
    I.Config("det_d128_cross", B=3, H=2, N=200, d=128, lengths=[200, 63, 9], Nk=330, lengths_k=[0, 330, 129], seed=33),
])
def test_deterministic_backward_parity(cfg):
    run_case(cfg, nan_prefill=True, deterministic=True, tol=FP16_FWD_TOL if cfg.dtype == "fp16" else BF16_TOL)


@pytest.mark.parametrize("d", [64, 128])
def test_deterministic_backward_bitwise(d):
    """Same inputs twice -> bitwise identical dQ, dK, dV; dK/dV also equal the fused kernel's."""
    sa = _sa()
    cfg = I.Config("det_bits", B=4, H=3, N=640, d=d, lengths=[640, 333, 129, 500], seed=34)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    r1 = sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=True)
    r2 = sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=True)
    rf = sa.sigattn_bwd(q, k, v, do, nq, nk)
    torch.cuda.synchronize()
    for a, b_ in zip(r1, r2):
        assert torch.equal(a, b_)
    assert torch.equal(r1[1], rf[1]) and torch.equal(r1[2], rf[2])   # dK, dV: same arithmetic
    assert relerr(f64(r1[0]), f64(rf[0])) < 1e-2


def test_deterministic_autograd():
    sa = _sa()
    cfg = I.Config("det_ag", B=2, H=2, N=256, d=64, lengths=[256, 100], seed=35)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    grads = []
    for det in (False, True):
        qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
        o = sa.sigmoid_attention(qq, kk, vv, seqlens_q=nq, seqlens_k=nk, deterministic=det)
        o.backward(do)
        grads.append((qq.grad, kk.grad, vv.grad))
    assert torch.equal(grads[0][1], grads[1][1]) and torch.equal(grads[0][2], grads[1][2])
    assert relerr(f64(grads[1][0]), f64(grads[0][0])) < 1e-2


# ---------------------------------------------------------------------------------------------
# learnable per-sequence bias: dL/db_z = sum over heads and valid (i, j) of dS
@pytest.mark.parametrize("cfg,det", [
    (I.C1, False),
    (I.Config("db_ragged", B=5, H=3, N=300, d=64, lengths=[300, 1, 129, 0, 256], seed=40), False),
    (I.Config("db_ragged_det", B=5, H=3, N=300, d=64, lengths=[300, 1, 129, 0, 256], seed=40), True),
    (I.Config("db_d128", B=3, H=2, N=260, d=128, lengths=[260, 65, 200], seed=41), False),
    (I.Config("db_d128_det", B=3, H=2, N=260, d=128, lengths=[260, 65, 200], seed=41), True),
])
def test_bias_gradient(cfg, det):
    sa = _sa()
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    bias = torch.tensor([-math.log(max(n, 1)) + 0.1 * i for i, n in enumerate(cfg.nk)], dtype=torch.float32,
                        device="cuda")
    db = torch.full((cfg.B,), float("nan"), dtype=torch.float32, device="cuda")   # must be overwritten
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, bias=bias, dbias=db, deterministic=det)
    torch.cuda.synchronize()
    ref = oracle.dbias(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, 1.0 / math.sqrt(cfg.d),
                       bias.double().cpu().numpy())
    got = db.double().cpu().numpy()
    # dS is summed in fp32 from the same sigma the kernel uses; the oracle is fp64 on the rounded inputs
    assert np.abs(got - ref).max() <= 1e-2 * max(np.abs(ref).max(), 1e-6), (got, ref)
    # the requested gradient does not change dQ, dK, dV
    dq2, dk2, dv2 = sa.sigattn_bwd(q, k, v, do, nq, nk, bias=bias, deterministic=det)
    assert torch.equal(dk, dk2) and torch.equal(dv, dv2)


def test_bias_gradient_autograd():
    sa = _sa()
    cfg = I.Config("db_ag", B=3, H=2, N=256, d=64, lengths=[256, 100, 17], seed=42)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    bias = torch.tensor([-5.0, -4.0, -3.0], device="cuda", requires_grad=True)
    o = sa.sigmoid_attention(q, k, v, seqlens_q=nq, seqlens_k=nk, bias=bias)
    o.backward(do)
    ref = oracle.dbias(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, 1 / 8, [-5.0, -4.0, -3.0])
    assert np.abs(bias.grad.double().cpu().numpy() - ref).max() <= 1e-2 * np.abs(ref).max()


def _check_sampled(cfg, pairs, q, k, v, do, o, grads, alpha, b, rng, nrand=96):
    """Sampled rows of the given (b, h) pairs against the row-sampled oracle (exact per row)."""
    bias = [b]
    for (bb, hh) in pairs:
        qs, ks, vs = (f64(t[bb:bb + 1, hh:hh + 1]) for t in (q, k, v))
        nqb, nkb = [cfg.nq[bb]], [cfg.nk[bb]]
        rows = _sampled_rows(cfg.nq[bb], cfg.N, rng, k=nrand)
        checks = [("o", o, oracle.fwd_rows(qs, ks, vs, 0, 0, rows, nqb, nkb, alpha, bias))]
        if grads is not None:
            dos = f64(do[bb:bb + 1, hh:hh + 1])
            dq, dk, dv = grads
            rdk, rdv = oracle.dkdv_rows(qs, ks, vs, dos, 0, 0, rows, nqb, nkb, alpha, bias)
            checks += [("dq", dq, oracle.dq_rows(qs, ks, vs, dos, 0, 0, rows, nqb, nkb, alpha, bias)),
                       ("dk", dk, rdk), ("dv", dv, rdv)]
        for name, got, ref in checks:
            err = relerr(f64(got[bb, hh])[rows], ref)
            assert err <= BF16_TOL, f"{cfg.name} {name} (b={bb}, h={hh}) rel err {err}"


@pytest.mark.parametrize("N,d", [(16384, 128), (16384, 64), (1024, 128), (1024, 64)])
def test_c2_full_size_sampled(N, d):
    """C2 forward sweep members at full size (B = 16384/N, H = 16, unpadded), in the bench's launch
    configuration (`bench.py --workload c2:N:d`): sampled rows of two (b, h) pairs."""
    sa = _sa()
    cfg = I.c2(N, d)
    q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
    alpha, b = 1 / math.sqrt(d), -math.log(N)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    _check_sampled(cfg, [(0, 0), (cfg.B - 1, 15)], q, k, v, do, o, None, alpha, b, rng)


def test_c4_layer_full_size_sampled():
    """C4: one 160M-encoder attention layer (B=16, H=12, N=8192, d=64, unpadded) fwd + bwd at full
    size (`bench.py --workload c4`): sampled rows of three (b, h) pairs."""
    sa = _sa()
    cfg = I.c4_layer(0)
    q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
    alpha, b = 1 / 8, -math.log(8192)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    grads = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    _check_sampled(cfg, [(0, 0), (7, 5), (15, 11)], q, k, v, do, o, grads, alpha, b, rng, nrand=48)


def test_c5_full_size_sampled():
    """C5: the single 16K sequence (H=16, d=128) fwd + bwd at full size, unsplit (`bench.py --workload
    c5`), and the same sequence as a G=8 key split (fp32 partials summed), as the CP ranks compute it."""
    sa = _sa()
    cfg = I.c5(16, 128)
    q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, "cuda")
    alpha, b = 1 / math.sqrt(128), -math.log(16384)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    grads = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    _check_sampled(cfg, [(0, 0), (0, 9)], q, k, v, do, o, grads, alpha, b, rng, nrand=32)
    # key split over G = 8 shards with the GLOBAL bias: partial fp32 outputs sum to O
    G, blk = 8, 16384 // 8
    acc = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
    for r in range(G):
        ks, vs = k[:, :, r * blk:(r + 1) * blk].contiguous(), v[:, :, r * blk:(r + 1) * blk].contiguous()
        acc += sa.sigattn_fwd(q, ks, vs, nq, torch.full_like(nk, blk), alpha, b, out_f32=True)
    torch.cuda.synchronize()
    rows = _sampled_rows(16384, 16384, rng, k=32)
    for hh in (0, 9):
        ref = oracle.fwd_rows(f64(q[:, hh:hh + 1]), f64(k[:, hh:hh + 1]), f64(v[:, hh:hh + 1]), 0, 0, rows,
                              [16384], [16384], alpha, [b])
        err = relerr(f64(acc[0, hh])[rows], ref)
        assert err <= BF16_TOL, f"c5 key-split sum (h={hh}) rel err {err}"


def _to_bshd(t):
    return t.transpose(1, 2).contiguous()


@pytest.mark.parametrize("d,dtype,det", [(64, "bf16", False), (64, "fp16", True), (128, "bf16", False),
                                         (128, "bf16", True)])
def test_layout_bshd_matches_bhsd(d, dtype, det):
    """The paper's [Z, L, H, D] layout through strided TMA views: same arithmetic as the
    [B, H, N, d] path, so O, dK, dV (and dQ in deterministic mode) are bitwise equal; padded rows 0."""
    sa = _sa()
    cfg = I.Config("bshd", B=3, H=3, N=320, d=d, lengths=[320, 129, 7], dtype=dtype, seed=31)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1 / math.sqrt(d), -math.log(320)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b)
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, deterministic=det)
    qs, ks, vs, dos = (_to_bshd(t) for t in (q, k, v, do))
    nan = lambda t: torch.full_like(t, float("nan"))  # noqa: E731
    o2 = sa.sigattn_fwd(qs, ks, vs, nq, nk, alpha, b, out=nan(qs), layout="bshd")
    dq2, dk2, dv2 = sa.sigattn_bwd(qs, ks, vs, dos, nq, nk, alpha, b, dq=nan(qs), dk=nan(ks), dv=nan(vs),
                                   deterministic=det, layout="bshd")
    o32 = sa.sigattn_fwd(qs, ks, vs, nq, nk, alpha, b, out_f32=True, layout="bshd")
    torch.cuda.synchronize()
    assert o2.shape == (3, 320, 3, d)
    for name, a_, b_ in (("o", o, o2), ("dk", dk, dk2), ("dv", dv, dv2)):
        assert torch.equal(a_, b_.transpose(1, 2)), f"{name}: bshd != bhsd"
    if det:
        assert torch.equal(dq, dq2.transpose(1, 2))
    rdq = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, np.full(3, b))[0]
    assert relerr(f64(dq2.transpose(1, 2)), rdq) <= BF16_TOL
    assert relerr(f64(o32.transpose(1, 2)), f64(o)) <= 4e-3
    for bb, n in enumerate(cfg.nq):
        assert torch.all(o2[bb, n:] == 0) and torch.all(dq2[bb, n:] == 0)
        assert torch.all(dk2[bb, n:] == 0) and torch.all(dv2[bb, n:] == 0)


def test_layout_bshd_autograd():
    """sigmoid_attention(..., layout='bshd') with a key_padding_mask: gradients through the library."""
    sa = _sa()
    cfg = I.Config("bshd_ag", B=2, H=2, N=256, d=64, lengths=[256, 100], seed=32)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    mask = torch.arange(256, device="cuda")[None, :] >= nk[:, None]
    qq, kk, vv = (_to_bshd(t).requires_grad_(True) for t in (q, k, v))
    o = sa.sigmoid_attention(qq, kk, vv, key_padding_mask=mask, layout="bshd")
    o.backward(_to_bshd(do))
    bias = np.full(2, -math.log(256))
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, 1 / 8, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, 1 / 8, bias)
    assert relerr(f64(o.transpose(1, 2)), ro) <= BF16_TOL
    for got, ref in ((qq.grad, rdq), (kk.grad, rdk), (vv.grad, rdv)):
        assert relerr(f64(got.transpose(1, 2)), ref) <= BF16_TOL


def test_encoder_layer_integration():
    """§8f f4: the op inside Table 4's pre-LN encoder layer (hidden 768, 12 heads, d = 64), bf16,
    jagged lengths, [B, N, H, d] projections read in place.
    (1) The layer's own attention call -- the q/k/v projection outputs it produced, the output it
        fed to o_proj, the incoming gradient dO and the dQ/dK/dV it returned, captured with hooks --
        against the fp64 oracle (fwd and bwd), every element.
    (2) Forward and input/weight gradients of the whole layer against the same layer composed in
        plain PyTorch fp32 (tests/encoder_ref.py, test-only), for the surrounding plumbing."""
    from paper_2604_27124_b200.encoder import SigmoidEncoderLayer
    from encoder_ref import reference_attention_fp32
    torch.manual_seed(5)
    layer = SigmoidEncoderLayer(dropout=0.0).cuda().to(torch.bfloat16)
    B, N = 3, 384
    lens = torch.tensor([384, 200, 57], dtype=torch.int32, device="cuda")
    x = torch.randn(B, N, 768, device="cuda").to(torch.bfloat16).requires_grad_(True)
    cap = {}

    def keep(name):
        def fwd_hook(mod, inp, out):
            cap[name] = out.detach()
            out.register_hook(lambda g: cap.__setitem__("d" + name, g.detach()))
        return fwd_hook

    def keep_o(mod, inp):
        cap["o"] = inp[0].detach()
        inp[0].register_hook(lambda g: cap.__setitem__("do", g.detach()))

    hooks = [layer.q_proj.register_forward_hook(keep("q")), layer.k_proj.register_forward_hook(keep("k")),
             layer.v_proj.register_forward_hook(keep("v")), layer.o_proj.register_forward_pre_hook(keep_o)]
    y = layer(x, lens)
    gy = torch.randn_like(y)
    y.backward(gy)
    for h_ in hooks:
        h_.remove()
    bhsd = lambda t: f64(t.reshape(B, N, 12, 64).transpose(1, 2))  # noqa: E731
    nl = lens.tolist()
    bias = np.full(B, -math.log(N))
    ro = oracle.fwd(bhsd(cap["q"]), bhsd(cap["k"]), bhsd(cap["v"]), nl, nl, 1 / 8, bias)
    assert relerr(bhsd(cap["o"]), ro) <= BF16_TOL
    rdq, rdk, rdv = oracle.bwd(bhsd(cap["q"]), bhsd(cap["k"]), bhsd(cap["v"]), bhsd(cap["do"]), nl, nl, 1 / 8, bias)
    for name, ref in (("dq", rdq), ("dk", rdk), ("dv", rdv)):
        assert relerr(bhsd(cap[name]), ref) <= BF16_TOL, name
    layer_f = SigmoidEncoderLayer(dropout=0.0).cuda()   # fp32 copy of the same (bf16) weights
    layer_f.load_state_dict({k_: v_.float() for k_, v_ in layer.state_dict().items()})
    xr = x.detach().float().requires_grad_(True)
    yr = reference_attention_fp32(layer_f, xr, lens)
    yr.backward(gy.float())
    assert relerr(f64(y - x), f64(yr - xr)) <= 3e-2
    assert relerr(f64(x.grad), f64(xr.grad)) <= 3e-2
    # weight gradient of the query projection flows through sigattn_bwd's dQ
    wq = layer.q_proj.weight
    assert relerr(f64(wq.grad), f64(layer_f.q_proj.weight.grad)) <= 5e-2


@pytest.mark.parametrize("d", [64, 128])
def test_skip_accounting_device_counters(d):
    """Padded-tile skipping measured on the device (SURVEY 8(c) skip accounting): the
    kernels execute exactly sum_b ceil(n_q/Bq) ceil(n_k/128) tile pairs per head -- none for n = 0,
    none past a sequence's last valid tile -- in the forward, the backward and the deterministic dQ
    pass (Bq = 128, except the d = 128 backward's 64-query tiles)."""
    from paper_2604_27124_b200 import _lib
    sa = _sa()
    cfg = I.Config("skip", B=4, H=3, N=640, d=d, lengths=[640, 300, 1, 0], seed=41)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.sigattn_set_debug_counters(cnt.data_ptr())
    try:
        sa.sigattn_fwd(q, k, v, nq, nk)
        sa.sigattn_bwd(q, k, v, do, nq, nk)
        sa.sigattn_bwd(q, k, v, do, nq, nk, deterministic=True)
        torch.cuda.synchronize()
    finally:
        lib.sigattn_set_debug_counters(None)
    c = lambda n, t: -(-n // t)  # noqa: E731
    fwd = cfg.H * sum(c(n, 128) * c(n, 128) for n in cfg.nq)
    bq = 128 if d == 64 else 64
    bwd = cfg.H * sum(c(n, 128) * c(n, bq) for n in cfg.nq)
    got = cnt.tolist()
    assert got[0] == fwd, (got, fwd)
    # fused backward + the deterministic run's key-tile pass both count into [1]
    assert got[1] == 2 * bwd, (got, bwd)
    assert got[2] == fwd, (got, fwd)
    dense = cfg.H * cfg.B * c(640, 128) ** 2
    assert got[0] < dense


@pytest.mark.parametrize("d", [64, 128])
def test_sanitize_pad_nan_inputs(d):
    """SIGATTN_F_SANITIZE_PAD: NaN in the padded rows of Q, K, V, dO (DESIGN R3: a tensor core
    computes 0 * NaN = NaN) -- with the flag the outputs are finite, match the oracle on the valid
    inputs and keep exact-zero padded rows; only rows [n, ceil128(n)) of the inputs are rewritten."""
    sa = _sa()
    cfg = I.Config("nanpad", B=3, H=2, N=384, d=d, lengths=[384, 200, 57], seed=43)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    ref = [f64(t) for t in (q, k, v, do)]           # oracle inputs: zero pad
    for t in (q, k, v, do):
        for bb, n in enumerate(cfg.nq):
            t[bb, :, n:] = float("nan")
    alpha, b = 1 / math.sqrt(d), -math.log(384)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, sanitize_pad=True)
    dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, sanitize_pad=True)
    torch.cuda.synchronize()
    bias = np.full(cfg.B, b)
    ro = oracle.fwd(ref[0], ref[1], ref[2], cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(*ref, cfg.nq, cfg.nk, alpha, bias)
    for name, got, r in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        assert torch.isfinite(got).all(), name
        assert relerr(f64(got), r) <= BF16_TOL, name
    for bb, n in enumerate(cfg.nq):
        assert torch.all(o[bb, :, n:] == 0) and torch.all(dk[bb, :, n:] == 0)
        t1 = min(-(-n // 128) * 128, 384)
        assert torch.all(v[bb, :, n:t1] == 0) and torch.isnan(v[bb, :, t1:]).all()


@pytest.mark.parametrize("d", [64, 128])
def test_nonprefix_key_padding_mask(d):
    """§8f f3: a general (non-prefix) key_padding_mask -- valid tokens anywhere -- through the
    library's stable compaction (mask_to_index + row gather), the prefix-length kernels and the
    inverse scatter; forward and gradients against the oracle evaluated on the compacted sequences
    (exact: sigma attention is equivariant under a joint permutation of queries and keys), and padded
    positions exactly 0 in O and every gradient."""
    sa = _sa()
    B, H, N = 2, 2, 320
    g = torch.Generator().manual_seed(44)
    mask = torch.rand((B, N), generator=g) < torch.tensor([[0.3], [0.6]])   # True = pad, scattered
    mask = mask.cuda()
    q, k, v, do = (torch.randn((B, H, N, d), generator=g).to(torch.bfloat16).cuda() for _ in range(4))
    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
    o = sa.sigmoid_attention(qq, kk, vv, key_padding_mask=mask)
    o.backward(do)
    torch.cuda.synchronize()
    alpha, b = 1 / math.sqrt(d), -math.log(N)
    for bb in range(B):
        keep = (~mask[bb]).nonzero().flatten()
        n = int(keep.numel())
        sel = lambda t: f64(t[bb:bb + 1][:, :, keep])  # noqa: E731
        ro = oracle.fwd(sel(q), sel(k), sel(v), [n], [n], alpha, [b])
        rdq, rdk, rdv = oracle.bwd(sel(q), sel(k), sel(v), sel(do), [n], [n], alpha, [b])
        for name, got, ref in (("o", o, ro), ("dq", qq.grad, rdq), ("dk", kk.grad, rdk), ("dv", vv.grad, rdv)):
            assert relerr(sel(got.detach()), ref) <= BF16_TOL, (name, bb)
            assert torch.all(got.detach()[bb][:, mask[bb]] == 0), (name, bb)
    idx, lens = sa.sigattn_mask_to_index(mask)
    assert lens.tolist() == (~mask).sum(1).tolist()
    for bb in range(B):   # stable: valid positions in order, then padded positions in order
        ref_idx = torch.cat([(~mask[bb]).nonzero().flatten(), mask[bb].nonzero().flatten()]).to(torch.int32)
        assert torch.equal(idx[bb], ref_idx)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("deterministic", [False, True])
def test_no_zero_pad_out_valid_rows(d, deterministic):
    """SIGATTN_F_NO_ZERO_PAD_OUT leaves padded rows unspecified, but every VALID row is written --
    including the exact zeros of a sequence whose key set is empty (n_k = 0 < n_q) or whose query set
    is empty (dK = dV = 0 on its valid keys).  Outputs are prefilled with NaN."""
    sa = _sa()
    cfg = I.Config("nozero", B=4, H=2, N=320, d=d, lengths=[320, 77, 5, 0], Nk=256, lengths_k=[256, 0, 129, 200],
                   seed=60 + d)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1.0 / math.sqrt(d), -math.log(256)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=torch.full_like(q, float("nan")), zero_pad_out=False)
    p = sa.attention
    dq, dk, dv = (torch.full_like(t, float("nan")) for t in (q, k, v))
    flags = p._lib.SIGATTN_F_NO_ZERO_PAD_OUT | (p._lib.SIGATTN_F_BWD_DETERMINISTIC if deterministic else 0)
    lib = p._lib.load()
    prm = p._lib.make_params(cfg.B, cfg.H, cfg.N, cfg.N_k, d, 0, nq.data_ptr(), nk.data_ptr(), alpha, b, None, flags)
    need = int(lib.sigattn_bwd_workspace_bytes(__import__("ctypes").byref(prm)))
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    p._lib.check(lib.sigattn_bwd(__import__("ctypes").byref(prm), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                 do.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), need,
                                 torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    bias = np.full(cfg.B, b)
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias)
    for name, got, ref, lens in (("o", o, ro, cfg.nq), ("dq", dq, rdq, cfg.nq), ("dk", dk, rdk, cfg.nk),
                                 ("dv", dv, rdv, cfg.nk)):
        g = f64(got)
        for bb in range(cfg.B):
            valid = g[bb, :, :lens[bb]]
            assert np.isfinite(valid).all(), f"{name}: valid rows of sequence {bb} not written"
            assert np.abs(valid - ref[bb, :, :lens[bb]]).max(initial=0) <= BF16_TOL * np.abs(ref).max()
    assert torch.all(o[1, :, :77] == 0), "n_k = 0: valid O rows are exact zeros"
    assert torch.all(dk[3, :, :200] == 0) and torch.all(dv[3, :, :200] == 0), "n_q = 0: dK = dV = 0"


def test_scalar_learnable_bias_gradient_b_gt_1():
    """A 1-element learnable bias shared by all sequences (B > 1) gets d loss / d b = sum over
    sequences of the per-sequence gradient (it used to get None)."""
    sa = _sa()
    cfg = I.Config("db_scalar", B=3, H=2, N=256, d=64, lengths=[256, 100, 17], seed=43)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    bias = torch.tensor([-4.5], device="cuda", requires_grad=True)
    o = sa.sigmoid_attention(q, k, v, seqlens_q=nq, seqlens_k=nk, bias=bias)
    o.backward(do)
    assert bias.grad is not None and bias.grad.shape == (1,)
    ref = oracle.dbias(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, 1 / 8, [-4.5] * 3).sum()
    assert abs(float(bias.grad.item()) - ref) <= 1e-2 * abs(ref)


def test_output_buffer_validation():
    """Caller-supplied outputs / workspaces of the wrong shape, dtype or size are rejected before any
    launch (a bf16 dq with dq_f32 used to be memset as fp32)."""
    sa = _sa()
    cfg = I.Config("val", B=2, H=2, N=256, d=64, seed=44)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    with pytest.raises(ValueError, match="dq"):
        sa.sigattn_bwd(q, k, v, do, dq=torch.empty_like(q), dq_f32=True)
    with pytest.raises(ValueError, match="dk"):
        sa.sigattn_bwd(q, k, v, do, dk=torch.empty(2, 2, 128, 64, dtype=q.dtype, device="cuda"))
    with pytest.raises(ValueError, match="dv"):
        sa.sigattn_bwd(q, k, v, do, dv=torch.empty_like(v).transpose(2, 3).contiguous().transpose(2, 3))
    with pytest.raises(ValueError, match="out"):
        sa.sigattn_fwd(q, k, v, out=torch.empty_like(q, dtype=torch.float32))
    with pytest.raises(ValueError, match="workspace too small"):
        sa.sigattn_fwd(q, k, v, workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError, match="workspace too small"):
        sa.sigattn_bwd(q, k, v, do, workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("layout", ["bhsd", "bshd"])
def test_pad_fill_many_slabs(d, layout):
    """The idle-warp pad fills (a 32-slab step per lane group, 512-byte blocks dealt over all workers)
    at B*H = 144 slabs -- five steps, the last one partial -- with empty, one-row, tile-edge and full
    sequences and n_q != n_k: outputs prefilled with NaN, every padded row exactly 0 (P:593, P:638,
    P:692), valid rows equal to the oracle; the [B, N, H, d] layout bitwise equal to [B, H, N, d]."""
    sa = _sa()
    lq = [0, 1, 127, 128, 129, 255, 384, 300] * 3
    lk = [384, 5, 0, 128, 200, 129, 384, 1] * 3
    cfg = I.Config("fill", B=24, H=6, N=384, d=d, lengths=lq, Nk=384, lengths_k=lk, seed=70 + d)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1.0 / math.sqrt(d), -math.log(384)
    nan = lambda t: torch.full_like(t, float("nan"))  # noqa: E731
    if layout == "bhsd":
        o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=nan(q))
        dq, dk, dv = sa.sigattn_bwd(q, k, v, do, nq, nk, alpha, b, dq=nan(q), dk=nan(k), dv=nan(v))
    else:
        qs, ks, vs, dos = (_to_bshd(t) for t in (q, k, v, do))
        o = sa.sigattn_fwd(qs, ks, vs, nq, nk, alpha, b, out=nan(qs), layout="bshd").transpose(1, 2)
        dq, dk, dv = (t.transpose(1, 2) for t in sa.sigattn_bwd(qs, ks, vs, dos, nq, nk, alpha, b, dq=nan(qs),
                                                                  dk=nan(ks), dv=nan(vs), layout="bshd"))
    torch.cuda.synchronize()
    bias = np.full(cfg.B, b)
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, bias)
    rdq, rdk, rdv = oracle.bwd(f64(q), f64(k), f64(v), f64(do), cfg.nq, cfg.nk, alpha, bias)
    for name, got, ref, lens in (("o", o, ro, lq), ("dq", dq, rdq, lq), ("dk", dk, rdk, lk), ("dv", dv, rdv, lk)):
        g = f64(got)
        assert np.isfinite(g).all(), f"{name}: an element was never written"
        e = relerr(g, ref)
        assert e <= BF16_TOL, f"{name} rel err {e}"
        for bb, n in enumerate(lens):
            assert (g[bb, :, n:] == 0).all(), f"{name}: padded rows of sequence {bb} not exactly 0"


@pytest.mark.parametrize("layout", ["bhsd", "bshd"])
def test_copy_valid_rows_roundtrip(layout):
    """Padding-aware transfers (sigattn_copy_valid_rows): host -> device -> device -> host moves exactly
    the valid rows (byte count = sum of n_b * H rows) and leaves every padded row of the destination
    untouched; an attention step fed through them matches the padded-copy step bitwise."""
    sa = _sa()
    B, H, N, d = 5, 3, 300, 64
    lens = [300, 0, 1, 129, 256]
    shape = (B, N, H, d) if layout == "bshd" else (B, H, N, d)
    g = torch.Generator().manual_seed(5)
    src = torch.randn(shape, generator=g).to(torch.bfloat16).pin_memory()
    dev = torch.full(shape, 7.0, dtype=torch.bfloat16, device="cuda")
    nb = sa.copy_valid_rows(src, dev, lens, layout=layout)
    assert nb == sum(lens) * H * d * 2
    dev2 = torch.full_like(dev, 9.0)
    sa.copy_valid_rows(dev, dev2, lens, layout=layout)
    back = torch.full(shape, 5.0, dtype=torch.bfloat16).pin_memory()
    sa.copy_valid_rows(dev2, back, lens, layout=layout)
    torch.cuda.synchronize()
    for b, n in enumerate(lens):
        if layout == "bshd":
            v_ref, v_dev, v_back = src[b, :n], dev[b, :n].cpu(), back[b, :n]
            p_dev, p_back = dev[b, n:].cpu(), back[b, n:]
        else:
            v_ref, v_dev, v_back = src[b, :, :n], dev[b, :, :n].cpu(), back[b, :, :n]
            p_dev, p_back = dev[b, :, n:].cpu(), back[b, :, n:]
        assert torch.equal(v_dev, v_ref) and torch.equal(v_back, v_ref)
        assert torch.all(p_dev == 7.0) and torch.all(p_back == 5.0), "padded rows must not be touched"
    # an attention step through the valid-row path equals the padded-copy path
    cfg = I.Config("e2e", B=4, H=2, N=320, d=64, lengths=[320, 129, 7, 0], seed=80)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, bias = 1 / 8, -math.log(320)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    dq_, dk_, dv_ = (torch.zeros_like(t) for t in (q, k, v))
    for h_, d_ in ((hq, dq_), (hk, dk_), (hv, dv_)):
        sa.copy_valid_rows(h_, d_, cfg.nq)
    o_valid = sa.sigattn_fwd(dq_, dk_, dv_, nq, nk, alpha, bias)
    o_full = sa.sigattn_fwd(q, k, v, nq, nk, alpha, bias)
    ho = torch.zeros(o_full.shape, dtype=o_full.dtype).pin_memory()
    sa.copy_valid_rows(o_valid, ho, cfg.nq)
    torch.cuda.synchronize()
    assert torch.equal(o_valid, o_full), "outputs must not depend on padded input rows (R3)"
    assert torch.equal(ho, o_full.cpu())


def test_pad_fill_many_slabs_no_zero_pad_out():
    """SIGATTN_F_NO_ZERO_PAD_OUT through the rewritten fill (pad_rows = 0: only the valid rows of
    sequences with an empty key set are written, as exact zeros) at 144 slabs: padded rows keep the
    caller's NaN, every valid row matches the oracle."""
    sa = _sa()
    lq = [0, 1, 127, 128, 129, 255, 384, 300] * 3
    lk = [384, 0, 0, 128, 200, 0, 384, 1] * 3
    cfg = I.Config("fill_nz", B=24, H=6, N=384, d=64, lengths=lq, Nk=384, lengths_k=lk, seed=77)
    q, k, v, do, nq, nk = I.make_inputs(cfg, "cuda")
    alpha, b = 1.0 / 8, -math.log(384)
    o = sa.sigattn_fwd(q, k, v, nq, nk, alpha, b, out=torch.full_like(q, float("nan")), zero_pad_out=False)
    torch.cuda.synchronize()
    ro = oracle.fwd(f64(q), f64(k), f64(v), cfg.nq, cfg.nk, alpha, np.full(cfg.B, b))
    g = f64(o)
    for bb, (n, m) in enumerate(zip(lq, lk)):
        valid = g[bb, :, :n]
        assert np.isfinite(valid).all(), f"valid rows of sequence {bb} not written"
        assert np.abs(valid - ro[bb, :, :n]).max(initial=0) <= BF16_TOL * np.abs(ro).max()
        if m == 0:
            assert (valid == 0).all(), "n_k = 0: valid O rows are exact zeros"
        # rows past the last valid 128-row tile are never written with the flag
        r1 = min((n + 127) // 128 * 128, 384) if n > 0 and m > 0 else n
        assert np.isnan(g[bb, :, r1:]).all(), f"padded rows of sequence {bb} must be left untouched"
