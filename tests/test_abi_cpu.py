"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every symbol the
header declares, validates arguments before launching anything, and its host logic (FLOP credit,
work-list / padded-tile skipping) matches closed forms from the paper and SPEC."""
import ctypes
import json
import os
import re

import numpy as np
import pytest
import torch

from paper_2604_27124_b200 import _lib, inputs as I
import paper_2604_27124_b200 as sa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sigattn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sigattn_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert "sigattn_fwd" in syms and "sigattn_bwd" in syms
    for s in syms:
        assert hasattr(lib, s), f"libsigattn.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTED)
    assert b"sm_100a" in lib.sigattn_version()


def test_binary_is_sm100a_tcgen05():
    """The shipped cubin is sm_100a code with tcgen05 MMAs, TMEM loads and TMA (no HMMA)."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    for mnem in ("UTCHMMA", "LDTM", "STTM", "UTMALDG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_flops_pins():
    """App. B.1 and SPEC S:329-331 examples."""
    g = json.load(open(os.path.join(GOLDEN, "flops.json")))
    for ex in g["examples"]:
        got = sa.valid_flops(ex["b"], ex["h"], ex["d"], [ex["n"]] * ex["b"], [ex["n"]] * ex["b"], ex["direction"] == "fwd")
        assert got == ex["flops"], ex
    # quadratic scaling and the 2.5x backward credit
    for n in (1, 7, 300, 8192):
        f1 = sa.valid_flops(1, 3, 64, [n], [n], True)
        assert sa.valid_flops(1, 3, 64, [2 * n], [2 * n], True) == 4 * f1
        assert 2 * sa.valid_flops(1, 3, 64, [n], [n], False) == 5 * f1
    # jagged batches: per-sequence n_q * n_k on valid tokens only
    c3 = sa.valid_flops(32, 12, 64, I.C3_LENGTHS, I.C3_LENGTHS, True)
    assert c3 == 4 * 12 * 64 * sum(n * n for n in I.C3_LENGTHS) == 672246598656
    assert sa.valid_flops(2, 1, 1, [3, 0], [5, 9], True) == 4 * 15
    with pytest.raises(ValueError):
        sa.valid_flops(1, 1, 1, [-1], [2], True)


def test_worklist_skip_counts_closed_form():
    """Padded-tile skipping (Alg. 3): visited query tiles per head =
    sum_z ceil(n_q/128); skipped = sum_z max(0, ceil(L/128) - ceil(n_q/128))."""
    B, H, N = 2, 3, 256
    nq = [256, 97]
    items = sa.worklist_host(0, B, H, N, N, nq, nq)
    assert len(items) == H * (2 + 1)
    skipped_per_head = sum(max(0, -(-N // 128) - (-(-n // 128))) for n in nq)
    assert skipped_per_head == 1
    assert len(items) == H * (B * (N // 128) - skipped_per_head)
    # every (b, h, tile) at most once, only valid tiles, cost = key tiles
    assert len(set((b, h, t) for b, h, t, _ in items)) == len(items)
    for b, h, t, c in items:
        assert t * 128 < nq[b] and c == -(-nq[b] // 128)


def test_worklist_longest_first_and_c3_totals():
    """LPT order (cost non-increasing) and the C3 totals: 6,696 q tiles and sum_b H ceil(n/128)^2
    tile pairs -- 10.6% of the dense 1,572,864."""
    L = I.C3_LENGTHS
    items = sa.worklist_host(0, 32, 12, 8192, 8192, L, L)
    costs = [c for *_, c in items]
    assert all(a >= b for a, b in zip(costs, costs[1:]))
    assert len(items) == 12 * sum(-(-n // 128) for n in L) == 6696
    pairs = sum(costs)
    assert pairs == 12 * sum((-(-n // 128)) ** 2 for n in L) == 166944
    assert 32 * 12 * 64 * 64 == 1572864
    bwd = sa.worklist_host(1, 32, 12, 8192, 8192, L, L)
    assert sum(c for *_, c in bwd) == pairs


def test_worklist_cross_lengths_and_empty():
    # kind 1 (backward): items over key tiles, cost = query tiles; n = 0 sides emit nothing
    items = sa.worklist_host(1, 3, 1, 300, 200, [300, 0, 10], [200, 5, 0])
    assert items == [(0, 0, 0, 3), (0, 0, 1, 3)]
    assert sa.worklist_host(0, 1, 1, 128, 128, [0], [0]) == []


def _params(**kw):
    d = dict(B=1, H=1, Nq=128, Nk=128, d=64, dtype_code=0, seqlens_q_ptr=None, seqlens_k_ptr=None, scale=0.125,
             bias=0.0, bias_ptr=None, flags=0)
    d.update(kw)
    return _lib.make_params(**d)


@pytest.mark.parametrize("kw,status", [
    (dict(d=96), 1), (dict(d=32), 1), (dict(B=0), 1), (dict(Nq=0), 1), (dict(dtype_code=7), 1),
    (dict(B=5000), 2), (dict(scale=float("nan")), 1),
])
def test_fwd_rejects_bad_params_before_launch(kw, status):
    lib = _lib.load()
    p = _params(**kw)
    fake = 1 << 20
    assert lib.sigattn_fwd(ctypes.byref(p), fake, fake, fake, fake, fake, 1 << 20, None) == status
    assert len(lib.sigattn_last_error()) > 0


def test_pointer_checks():
    lib = _lib.load()
    p = _params()
    fneed = lib.sigattn_fwd_workspace_bytes(ctypes.byref(p))
    assert fneed >= 16 + 16 and fneed % 256 == 0
    assert lib.sigattn_fwd(ctypes.byref(p), None, 16, 16, 16, 16, fneed, None) == 1   # null
    assert lib.sigattn_fwd(ctypes.byref(p), 24, 16, 16, 16, 16, fneed, None) == 1     # misaligned
    assert lib.sigattn_fwd(ctypes.byref(p), 16, 16, 16, 16, None, fneed, None) == 1   # no workspace
    assert lib.sigattn_fwd(ctypes.byref(p), 16, 16, 16, 16, 16, fneed - 1, None) == 4  # workspace too small
    need = lib.sigattn_bwd_workspace_bytes(ctypes.byref(p))
    assert need >= 128 * 64 * 4
    assert lib.sigattn_bwd(ctypes.byref(p), 16, 16, 16, 16, 16, 16, 16, 16, need - 1, None) == 4
    bad = _params(d=96)
    assert lib.sigattn_bwd_workspace_bytes(ctypes.byref(bad)) == 0


def test_python_boundary_refuses_cpu_tensors():
    """No CPU fallback: host tensors are rejected loudly."""
    q = torch.zeros(1, 1, 128, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        sa.sigattn_fwd(q, q, q)
    with pytest.raises(ValueError, match="CUDA"):
        sa.sigattn_bwd(q, q, q, q)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()


def test_c_program_links_against_header(tmp_path):
    """A plain C99 program built against include/sigattn.h and linked to libsigattn.so runs the
    host-side entry points (tests/c/abi_test.c) -- the ABI is usable without Python or torch."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib = _lib.load() and _lib.LIB_PATH
    exe = tmp_path / "abi_test"
    libdir = os.path.dirname(lib)
    subprocess.check_call([cc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_test.c"), "-L", libdir, "-l:" + os.path.basename(lib),
                           "-Wl,-rpath," + libdir, "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_test: OK" in r.stdout


def test_copy_valid_rows_rejects_bad_arguments():
    """sigattn_copy_valid_rows validates its arguments before enqueueing any copy (no GPU needed)."""
    lib = _lib.load()
    lens = (ctypes.c_int32 * 2)(3, 1)
    buf = ctypes.create_string_buffer(4096)
    p = ctypes.cast(buf, ctypes.c_void_p).value
    n = ctypes.c_int64(-1)
    cases = [
        dict(src=None), dict(dst=None), dict(lens=None), dict(B=0), dict(H=-1), dict(N=0),
        dict(rb=24),   # row bytes not a multiple of 16
        dict(kind=0), dict(kind=4),
    ]
    for c in cases:
        a = dict(src=p, dst=p + 2048, B=2, H=1, N=4, rb=128, lens=ctypes.cast(lens, ctypes.c_void_p).value, kind=1)
        a.update(c)
        st = lib.sigattn_copy_valid_rows(a["src"], a["dst"], a["B"], a["H"], a["N"], a["rb"], a["lens"], 0,
                                         a["kind"], None, ctypes.byref(n))
        assert st == 1, c   # SIGATTN_EINVAL
    assert n.value == -1, "no bytes reported on a rejected call"
