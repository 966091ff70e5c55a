"""Pins for the fp64 oracle (oracle/), independent of the oracle's own code.

Each test checks the oracle against something the paper or mathematics fixes (a hand-worked
example, a closed form, an invariant, an independent library composition, finite differences),
chosen so that a plausible slip in the oracle -- a dropped alpha, a wrong sign, a transposed
operand, a missing mask, dS without the (1-P) factor -- fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_case(B=2, H=2, Nq=9, Nk=None, d=4, nq=None, nk=None, seed=0, pad=0.0):
    rng = np.random.default_rng(seed)
    Nk = Nq if Nk is None else Nk
    q = rng.standard_normal((B, H, Nq, d))
    k = rng.standard_normal((B, H, Nk, d))
    v = rng.standard_normal((B, H, Nk, d))
    do = rng.standard_normal((B, H, Nq, d))
    nq = np.array([Nq] * B if nq is None else nq, np.int32)
    nk = np.array(list(nq) if nk is None else nk, np.int32)
    for b in range(B):
        q[b, :, nq[b]:] = pad
        do[b, :, nq[b]:] = pad
        k[b, :, nk[b]:] = pad
        v[b, :, nk[b]:] = pad
    return q, k, v, do, nq, nk


def torch_reference(q, k, v, do, nq, nk, alpha, bias):
    """Independent composition with torch fp64 library ops + autograd (not the oracle's code)."""
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    qt = torch.tensor(q, requires_grad=True)
    kt = torch.tensor(k, requires_grad=True)
    vt = torch.tensor(v, requires_grad=True)
    mq = torch.arange(Nq)[None, :] < torch.tensor(nq)[:, None]          # [B, Nq]
    mk = torch.arange(Nk)[None, :] < torch.tensor(nk)[:, None]          # [B, Nk]
    valid = (mq[:, :, None] & mk[:, None, :])[:, None]                  # [B,1,Nq,Nk]
    s = alpha * torch.matmul(qt, kt.transpose(-1, -2)) + torch.tensor(bias, dtype=torch.float64)[:, None, None, None]
    p = torch.where(valid, torch.sigmoid(s), torch.zeros((), dtype=torch.float64))
    o = torch.matmul(p, vt)
    o = torch.where(mq[:, None, :, None], o, torch.zeros((), dtype=torch.float64))
    (o * torch.tensor(do)).sum().backward()
    return o.detach().numpy(), qt.grad.numpy(), kt.grad.numpy(), vt.grad.numpy()


def relmax(a, b):
    den = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() / den


# --------------------------------------------------------------------------------------------
def test_golden_worked_example():
    """Hand-derived values (tests/golden/worked_two_token.json, Eq. 2 P:117 + Alg. 1-3)."""
    g = json.load(open(os.path.join(GOLDEN, "worked_two_token.json")))
    inp = g["inputs"]
    sh = (1, 1, 3, 1)
    q = np.array(inp["q"]).reshape(sh); k = np.array(inp["k"]).reshape(sh)
    v = np.array(inp["v"]).reshape(sh); do = np.array(inp["dout"]).reshape(sh)
    n = [inp["n"]]
    o = oracle.fwd(q, k, v, n, n, alpha=inp["alpha"], bias=[inp["bias"]])
    dq, dk, dv = oracle.bwd(q, k, v, do, n, n, alpha=inp["alpha"], bias=[inp["bias"]])
    tol = g["tolerance_abs"]
    for name, got in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        np.testing.assert_allclose(got.reshape(-1), g["expected"][name], atol=tol, rtol=0)
    # the expected dk entries are -3/4 ln 3 and -1/2 ln 3 (derivation in the fixture)
    assert abs(g["expected"]["dk"][0] + 0.75 * math.log(3)) < 1e-15


@pytest.mark.parametrize("case", [
    dict(B=2, H=2, Nq=9, d=4, nq=[9, 5]),
    dict(B=3, H=1, Nq=7, Nk=11, d=3, nq=[7, 2, 4], nk=[11, 6, 1]),
    dict(B=1, H=3, Nq=16, d=8),
    dict(B=2, H=2, Nq=6, d=5, nq=[0, 6]),
])
def test_against_independent_torch_autograd(case):
    """Library reduction: torch fp64 sigmoid/matmul/autograd composition of Eq. 2 (<= 1e-12)."""
    q, k, v, do, nq, nk = rand_case(seed=3, **case)
    alpha = 0.37
    bias = np.array([-0.5 - 0.3 * b for b in range(q.shape[0])])
    o = oracle.fwd(q, k, v, nq, nk, alpha, bias)
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, alpha, bias)
    ro, rdq, rdk, rdv = torch_reference(q, k, v, do, nq, nk, alpha, bias)
    for got, ref in ((o, ro), (dq, rdq), (dk, rdk), (dv, rdv)):
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_central_finite_differences():
    """dQ, dK, dV match central FD of L = sum(dO * O): h=1e-5, rel <= 1e-6."""
    q, k, v, do, nq, nk = rand_case(B=1, H=1, Nq=4, d=2, nq=[3], seed=7)
    alpha, bias = 0.8, np.array([-0.4])
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, alpha, bias)

    def loss(q_, k_, v_):
        return float((oracle.fwd(q_, k_, v_, nq, nk, alpha, bias) * do).sum())

    h = 1e-5
    for name, x, g in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        fd = np.zeros_like(x)
        for idx in np.ndindex(x.shape):
            xp = x.copy(); xp[idx] += h
            xm = x.copy(); xm[idx] -= h
            args_p = dict(q_=q, k_=k, v_=v); args_m = dict(q_=q, k_=k, v_=v)
            args_p[name + "_"] = xp; args_m[name + "_"] = xm
            fd[idx] = (loss(**args_p) - loss(**args_m)) / (2 * h)
        assert relmax(g, fd) <= 1e-6, name


def test_q_zero_closed_form():
    """Q = 0: O_i = sigma(b) sum_{j<n_k} v_j; dV_j = sigma(b) sum_{i<n_q} dO_i;
    dQ_i = alpha sigma'(b) sum_j <dO_i, v_j> k_j; dK = 0 (BASELINE north star, Eq. 2)."""
    q, k, v, do, nq, nk = rand_case(B=2, H=2, Nq=10, d=6, nq=[10, 4], seed=11)
    q[:] = 0.0
    alpha, bias = 0.25, np.array([-math.log(10), 0.7])
    o = oracle.fwd(q, k, v, nq, nk, alpha, bias)
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, alpha, bias)
    for b in range(2):
        s = 1.0 / (1.0 + math.exp(-bias[b]))
        for h in range(2):
            n = nq[b]
            exp_o = s * v[b, h, :n].sum(0)
            np.testing.assert_allclose(o[b, h, :n], np.broadcast_to(exp_o, (n, 6)), rtol=1e-13, atol=1e-13)
            assert np.all(o[b, h, n:] == 0)
            exp_dv = s * do[b, h, :n].sum(0)
            np.testing.assert_allclose(dv[b, h, :n], np.broadcast_to(exp_dv, (n, 6)), rtol=1e-13, atol=1e-13)
            dP = do[b, h, :n] @ v[b, h, :n].T
            exp_dq = alpha * s * (1 - s) * dP @ k[b, h, :n]
            np.testing.assert_allclose(dq[b, h, :n], exp_dq, rtol=1e-12, atol=1e-13)
    assert np.all(dk == 0)


def test_single_key_closed_form():
    """n = 1 single token: O = sigma(alpha q.k + b) v."""
    rng = np.random.default_rng(5)
    q = rng.standard_normal((1, 1, 1, 8)); k = rng.standard_normal((1, 1, 1, 8)); v = rng.standard_normal((1, 1, 1, 8))
    alpha, b = 1 / math.sqrt(8), 0.0   # b = -log(1) = 0
    o = oracle.fwd(q, k, v, [1], [1], alpha, [b])
    x = alpha * float((q * k).sum()) + b
    np.testing.assert_allclose(o.reshape(-1), (1 / (1 + math.exp(-x))) * v.reshape(-1), rtol=1e-14)


def test_saturation():
    """bias +30: P ~ 1 so O ~ sum_valid v, dV ~ sum_valid dO, dQ ~ dK ~ 0; bias -30: O ~ 0."""
    q, k, v, do, nq, nk = rand_case(B=1, H=1, Nq=8, d=4, nq=[6], seed=2)
    o = oracle.fwd(q, k, v, nq, nk, 0.1, [30.0])
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, 0.1, [30.0])
    np.testing.assert_allclose(o[0, 0, :6], np.broadcast_to(v[0, 0, :6].sum(0), (6, 4)), atol=1e-10)
    np.testing.assert_allclose(dv[0, 0, :6], np.broadcast_to(do[0, 0, :6].sum(0), (6, 4)), atol=1e-10)
    assert np.abs(dq).max() < 1e-10 and np.abs(dk).max() < 1e-10
    o = oracle.fwd(q, k, v, nq, nk, 0.1, [-30.0])
    assert np.abs(o).max() < 1e-10


@pytest.mark.parametrize("fill", [1e6, "random", -3.5])
def test_pad_independence_bitwise(fill):
    """Overwriting pad entries of Q, K, V, dO leaves O, dQ, dK, dV bitwise unchanged."""
    q, k, v, do, nq, nk = rand_case(B=2, H=2, Nq=12, d=4, nq=[12, 7], nk=[9, 3], seed=4)
    ref = [oracle.fwd(q, k, v, nq, nk, 0.3, [-1.0, -2.0])] + list(oracle.bwd(q, k, v, do, nq, nk, 0.3, [-1.0, -2.0]))
    rng = np.random.default_rng(99)
    q2, k2, v2, do2 = q.copy(), k.copy(), v.copy(), do.copy()
    for b in range(2):
        for arr, n in ((q2, nq[b]), (do2, nq[b]), (k2, nk[b]), (v2, nk[b])):
            sl = arr[b, :, n:]
            arr[b, :, n:] = rng.standard_normal(sl.shape) * 50 if fill == "random" else fill
    got = [oracle.fwd(q2, k2, v2, nq, nk, 0.3, [-1.0, -2.0])] + list(oracle.bwd(q2, k2, v2, do2, nq, nk, 0.3, [-1.0, -2.0]))
    for a, b_ in zip(got, ref):
        assert np.array_equal(a, b_)


def test_padded_rows_exact_zero():
    """O, dQ rows i >= n_q and dK, dV rows j >= n_k are exactly 0."""
    q, k, v, do, nq, nk = rand_case(B=2, H=1, Nq=10, d=3, nq=[10, 4], nk=[5, 10], seed=8, pad=2.0)
    o = oracle.fwd(q, k, v, nq, nk, 0.5, [0.1, 0.2])
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, 0.5, [0.1, 0.2])
    for b in range(2):
        assert np.all(o[b, :, nq[b]:] == 0) and np.all(dq[b, :, nq[b]:] == 0)
        assert np.all(dk[b, :, nk[b]:] == 0) and np.all(dv[b, :, nk[b]:] == 0)
        assert np.abs(o[b, :, :nq[b]]).min() > 0  # valid rows are not masked


def test_permutation_equivariance():
    """Jointly permuting valid (k_j, v_j) leaves O unchanged; permuting valid queries permutes O."""
    q, k, v, do, nq, nk = rand_case(B=1, H=2, Nq=11, d=4, nq=[8], seed=6)
    o = oracle.fwd(q, k, v, nq, nk, 0.5, [-1.0])
    perm = np.random.default_rng(1).permutation(8)
    k2, v2 = k.copy(), v.copy()
    k2[:, :, :8] = k[:, :, perm]; v2[:, :, :8] = v[:, :, perm]
    o2 = oracle.fwd(q, k2, v2, nq, nk, 0.5, [-1.0])
    assert np.abs(o2 - o).max() <= 1e-12
    q3 = q.copy(); q3[:, :, :8] = q[:, :, perm]
    o3 = oracle.fwd(q3, k, v, nq, nk, 0.5, [-1.0])
    assert np.abs(o3[:, :, :8] - o[:, :, perm]).max() <= 1e-14


def test_key_split_additivity():
    """A4: O(Q,K,V) = sum_r O(Q,K_r,V_r) with the same global bias -- the CP pin."""
    q, k, v, do, nq, nk = rand_case(B=1, H=2, Nq=12, d=4, seed=9)
    bias = [-math.log(12)]
    o = oracle.fwd(q, k, v, nq, nk, 0.5, bias)
    parts = [(0, 5), (5, 8), (8, 12)]
    acc = np.zeros_like(o)
    dq_acc = np.zeros_like(o)
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, 0.5, bias)
    for lo, hi in parts:
        ks, vs = k[:, :, lo:hi], v[:, :, lo:hi]
        acc += oracle.fwd(q, ks, vs, [12], [hi - lo], 0.5, bias)
        dqr, dkr, dvr = oracle.bwd(q, ks, vs, do, [12], [hi - lo], 0.5, bias)
        dq_acc += dqr
        assert np.abs(dkr - dk[:, :, lo:hi]).max() <= 1e-12   # key-owned grads are local
        assert np.abs(dvr - dv[:, :, lo:hi]).max() <= 1e-12
    assert np.abs(acc - o).max() <= 1e-12
    assert np.abs(dq_acc - dq).max() <= 1e-12


def test_sigma_prime_bound_and_diagonal_jacobian():
    """|dS| <= 1/4 |dP| elementwise; equality when x = 0 (q = 0, b = 0)."""
    q, k, v, do, nq, nk = rand_case(B=1, H=1, Nq=10, d=4, nq=[7], seed=12)
    P, dP, dS = oracle.p_ds(q * 3, k * 3, v, do, 0, 0, nq, nk, 1.0, [0.3])
    assert np.all(np.abs(dS) <= 0.25 * np.abs(dP) + 1e-15)
    assert np.all((P[:7, :7] > 0) & (P[:7, :7] < 1))
    P0, dP0, dS0 = oracle.p_ds(np.zeros_like(q), k, v, do, 0, 0, nq, nk, 1.0, [0.0])
    np.testing.assert_allclose(P0[:7, :7], 0.5, rtol=0, atol=0)
    np.testing.assert_allclose(dS0, 0.25 * dP0, rtol=0, atol=0)
    # diagonal Jacobian: perturbing x_ij changes only P_ij (decoupled weights)
    k2 = k.copy(); k2[0, 0, 2] += 0.1
    P2, _, _ = oracle.p_ds(q * 3, k2 * 3, v, do, 0, 0, nq, nk, 1.0, [0.3])
    changed = np.abs(P2 - P) > 0
    assert changed[:, 2].sum() == 7 and changed.sum() == 7


def test_zero_dout_and_linearity():
    """dO = 0 -> all-zero gradients; O is linear in V; dV does not depend on V."""
    q, k, v, do, nq, nk = rand_case(B=2, H=1, Nq=8, d=3, nq=[8, 5], seed=13)
    z = oracle.bwd(q, k, v, np.zeros_like(do), nq, nk, 0.5, [-1, -1])
    assert all(np.all(t == 0) for t in z)
    o1 = oracle.fwd(q, k, v, nq, nk, 0.5, [-1, -1])
    o2 = oracle.fwd(q, k, 2.0 * v, nq, nk, 0.5, [-1, -1])
    assert np.abs(o2 - 2 * o1).max() <= 1e-14
    dv1 = oracle.bwd(q, k, v, do, nq, nk, 0.5, [-1, -1])[2]
    dv2 = oracle.bwd(q, k, -3 * v, do, nq, nk, 0.5, [-1, -1])[2]
    assert np.array_equal(dv1, dv2)


def test_row_sampled_equals_full():
    """The row-sampled entry points reproduce the full evaluation exactly."""
    q, k, v, do, nq, nk = rand_case(B=2, H=2, Nq=13, Nk=9, d=5, nq=[13, 6], nk=[9, 4], seed=14)
    o = oracle.fwd(q, k, v, nq, nk, 0.4, [-0.2, -0.9])
    dq, dk, dv = oracle.bwd(q, k, v, do, nq, nk, 0.4, [-0.2, -0.9])
    rows_q = [0, 3, 5, 12]
    rows_k = [0, 4, 8]
    for b in range(2):
        for h in range(2):
            assert np.array_equal(oracle.fwd_rows(q, k, v, b, h, rows_q, nq, nk, 0.4, [-0.2, -0.9]), o[b, h, rows_q])
            assert np.array_equal(oracle.dq_rows(q, k, v, do, b, h, rows_q, nq, nk, 0.4, [-0.2, -0.9]), dq[b, h, rows_q])
            dkr, dvr = oracle.dkdv_rows(q, k, v, do, b, h, rows_k, nq, nk, 0.4, [-0.2, -0.9])
            assert np.array_equal(dkr, dk[b, h, rows_k]) and np.array_equal(dvr, dv[b, h, rows_k])


def test_alpha_enters_dq_dk_once():
    """Scale check (Alg. 2, Alg. 3): with alpha -> 2 alpha and Q -> Q/2 the
    scores (hence P, dS) are unchanged, so dQ doubles... times the chain factor: dQ(Q/2, 2a)
    = 2 * dQ(Q, a) / 1 and dK(Q/2, 2a) = dK(Q, a)."""
    q, k, v, do, nq, nk = rand_case(B=1, H=1, Nq=6, d=4, seed=15)
    dq1, dk1, dv1 = oracle.bwd(q, k, v, do, nq, nk, 0.3, [-1.0])
    dq2, dk2, dv2 = oracle.bwd(q / 2, k, v, do, nq, nk, 0.6, [-1.0])
    np.testing.assert_allclose(dq2, 2 * dq1, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(dk2, dk1, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(dv2, dv1, rtol=1e-12, atol=1e-15)


# --------------------------------------------------------------------------------------------
# learnable per-sequence bias ("fixed or learnable"): d L / d b_z
@pytest.mark.parametrize("case", [dict(), dict(Nq=7, Nk=11, nq=[5, 0], nk=[11, 4])])
def test_dbias_against_torch_autograd(case):
    """oracle.dbias == torch fp64 autograd of Eq. 2 w.r.t. a per-sequence bias tensor (<= 1e-12)."""
    q, k, v, do, nq, nk = rand_case(seed=11, **case)
    alpha = 0.45
    bias = np.array([-0.7 + 0.4 * b for b in range(q.shape[0])])
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    bt = torch.tensor(bias, requires_grad=True)
    mq = torch.arange(Nq)[None, :] < torch.tensor(nq)[:, None]
    mk = torch.arange(Nk)[None, :] < torch.tensor(nk)[:, None]
    valid = (mq[:, :, None] & mk[:, None, :])[:, None]
    s = alpha * torch.matmul(torch.tensor(q), torch.tensor(k).transpose(-1, -2)) + bt[:, None, None, None]
    p = torch.where(valid, torch.sigmoid(s), torch.zeros((), dtype=torch.float64))
    o = torch.where(mq[:, None, :, None], torch.matmul(p, torch.tensor(v)), torch.zeros((), dtype=torch.float64))
    (o * torch.tensor(do)).sum().backward()
    got = oracle.dbias(q, k, v, do, nq, nk, alpha, bias)
    ref = bt.grad.numpy()
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_dbias_finite_differences_and_invariants():
    """Central FD of L(b) (h=1e-5, rel <= 1e-7); db is 0 for a sequence with no valid key;
    db is linear in dO and equals the sum over heads of the per-head dS sums (oracle.p_ds)."""
    q, k, v, do, nq, nk = rand_case(B=3, H=2, Nq=5, d=3, nq=[5, 3, 2], nk=[5, 0, 4], seed=12)
    alpha, bias = 0.6, np.array([-0.2, -1.0, 0.3])
    db = oracle.dbias(q, k, v, do, nq, nk, alpha, bias)
    h = 1e-5
    for b in range(3):
        bp, bm = bias.copy(), bias.copy()
        bp[b] += h
        bm[b] -= h
        fd = ((oracle.fwd(q, k, v, nq, nk, alpha, bp) - oracle.fwd(q, k, v, nq, nk, alpha, bm)) * do).sum() / (2 * h)
        assert abs(db[b] - fd) <= 1e-7 * max(1.0, abs(fd))
    assert db[1] == 0.0
    assert np.allclose(oracle.dbias(q, k, v, 2.5 * do, nq, nk, alpha, bias), 2.5 * db, rtol=1e-12, atol=0)
    for b in range(3):
        tot = sum(oracle.p_ds(q, k, v, do, b, hh, nq, nk, alpha, bias)[2].sum() for hh in range(2))
        assert abs(tot - db[b]) <= 1e-12 * max(1.0, abs(tot))
