"""fp64 CPU oracle for padding-aware sigmoid attention (Eq. 2, Alg. 1-3).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2604_27124_b200`` and ``libsigattn.so``) never imports it and shares no code with it.

The arithmetic lives in ``sigattn_oracle.c`` (plain C, fp64, OpenMP over output rows); this
module only builds/loads that library and marshals numpy arrays.  Every function follows the
definition cited in the C file's header.  Inputs are fp64 arrays [B, H, N, d]; callers pass the
same bf16/fp16-rounded values the GPU sees, upcast to fp64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sigattn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i = ctypes.c_int
        dd = ctypes.c_double
        lib.sigattn_oracle_fwd.argtypes = [i, i, i, i, i, _D, _D, _D, _I, _I, dd, _D, _D]
        lib.sigattn_oracle_bwd.argtypes = [i, i, i, i, i, _D, _D, _D, _D, _I, _I, dd, _D, _D, _D, _D]
        lib.sigattn_oracle_fwd_rows.argtypes = [i, i, i, i, _D, _D, _D, _I, _I, dd, _D, i, i, _I, i, _D]
        lib.sigattn_oracle_dq_rows.argtypes = [i, i, i, i, _D, _D, _D, _D, _I, _I, dd, _D, i, i, _I, i, _D]
        lib.sigattn_oracle_dkdv_rows.argtypes = [i, i, i, i, _D, _D, _D, _D, _I, _I, dd, _D, i, i, _I, i, _D, _D]
        lib.sigattn_oracle_p_ds.argtypes = [i, i, i, i, _D, _D, _D, _D, _I, _I, dd, _D, i, i, _D, _D, _D]
        lib.sigattn_oracle_dbias.argtypes = [i, i, i, i, i, _D, _D, _D, _D, _I, _I, dd, _D, _D]
        lib.sigattn_oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D if a.dtype == np.float64 else _I)


def _prep(q, k, v, nq, nk, bias):
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    assert k.shape == (B, H, Nk, d) and v.shape == (B, H, Nk, d)
    nq = _i32(np.full(B, Nq) if nq is None else nq)
    nk = _i32(nq if nk is None else nk)
    bias = _f64(np.full(B, -np.log(Nk)) if bias is None else np.broadcast_to(np.asarray(bias, np.float64), (B,)))
    return q, k, v, nq, nk, bias, (B, H, Nq, Nk, d)


def threads() -> int:
    return int(_load().sigattn_oracle_threads())


def fwd(q, k, v, nq=None, nk=None, alpha=None, bias=None) -> np.ndarray:
    """O = sigma(alpha Q K^T + b) V with padded rows/keys at zero weight; fp64 [B,H,Nq,d]."""
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    o = np.zeros((B, H, Nq, d), np.float64)
    _load().sigattn_oracle_fwd(B, H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(nq), _p(nk), alpha, _p(bias), _p(o))
    return o


def bwd(q, k, v, dout, nq=None, nk=None, alpha=None, bias=None):
    """(dQ, dK, dV) of sum(dout * O) -- Alg. 2/3 quantities from the definition; fp64."""
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    dout = _f64(dout)
    assert dout.shape == (B, H, Nq, d)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    dq = np.zeros((B, H, Nq, d), np.float64)
    dk = np.zeros((B, H, Nk, d), np.float64)
    dv = np.zeros((B, H, Nk, d), np.float64)
    _load().sigattn_oracle_bwd(B, H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(dout), _p(nq), _p(nk), alpha,
                               _p(bias), _p(dq), _p(dk), _p(dv))
    return dq, dk, dv


def dbias(q, k, v, dout, nq=None, nk=None, alpha=None, bias=None) -> np.ndarray:
    """d sum(dout * O) / d b_z for the per-sequence bias: sum over heads and valid (i, j) of dS; [B]."""
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    dout = _f64(dout)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    db = np.zeros((B,), np.float64)
    _load().sigattn_oracle_dbias(B, H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(dout), _p(nq), _p(nk), alpha,
                                 _p(bias), _p(db))
    return db


def fwd_rows(q, k, v, b, h, rows, nq=None, nk=None, alpha=None, bias=None) -> np.ndarray:
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    rows = _i32(rows)
    out = np.zeros((len(rows), d), np.float64)
    _load().sigattn_oracle_fwd_rows(H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(nq), _p(nk), alpha, _p(bias),
                                    int(b), int(h), _p(rows), len(rows), _p(out))
    return out


def dq_rows(q, k, v, dout, b, h, rows, nq=None, nk=None, alpha=None, bias=None) -> np.ndarray:
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    dout = _f64(dout)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    rows = _i32(rows)
    out = np.zeros((len(rows), d), np.float64)
    _load().sigattn_oracle_dq_rows(H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(dout), _p(nq), _p(nk), alpha,
                                   _p(bias), int(b), int(h), _p(rows), len(rows), _p(out))
    return out


def dkdv_rows(q, k, v, dout, b, h, rows, nq=None, nk=None, alpha=None, bias=None):
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    dout = _f64(dout)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    rows = _i32(rows)
    dk = np.zeros((len(rows), d), np.float64)
    dv = np.zeros((len(rows), d), np.float64)
    _load().sigattn_oracle_dkdv_rows(H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(dout), _p(nq), _p(nk), alpha,
                                     _p(bias), int(b), int(h), _p(rows), len(rows), _p(dk), _p(dv))
    return dk, dv


def p_ds(q, k, v, dout, b, h, nq=None, nk=None, alpha=None, bias=None):
    """(P, dP, dS) [Nq, Nk] of one (b, h): the Alg. 2 intermediates (padded entries 0)."""
    q, k, v, nq, nk, bias, (B, H, Nq, Nk, d) = _prep(q, k, v, nq, nk, bias)
    dout = _f64(dout)
    alpha = 1.0 / np.sqrt(d) if alpha is None else float(alpha)
    P = np.zeros((Nq, Nk)); dP = np.zeros((Nq, Nk)); dS = np.zeros((Nq, Nk))
    _load().sigattn_oracle_p_ds(H, Nq, Nk, d, _p(q), _p(k), _p(v), _p(dout), _p(nq), _p(nk), alpha,
                                _p(bias), int(b), int(h), _p(P), _p(dP), _p(dS))
    return P, dP, dS
