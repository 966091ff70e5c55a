"""ctypes binding of libsigattn.so (include/sigattn.h): argument marshalling only.

Every step of the method runs inside the library's CUDA kernels.  If the library is missing
this module raises -- there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsigattn.so")

SIGATTN_BF16 = 0
SIGATTN_FP16 = 1
SIGATTN_OK = 0
SIGATTN_F_BWD_DETERMINISTIC = 1 << 0
SIGATTN_F_OUT_F32_PARTIAL = 1 << 1
SIGATTN_F_DQ_F32_PARTIAL = 1 << 2
SIGATTN_F_NO_ZERO_PAD_OUT = 1 << 3
SIGATTN_F_LAYOUT_BSHD = 1 << 4
SIGATTN_F_SANITIZE_PAD = 1 << 5

STATUS_NAMES = {0: "SIGATTN_OK", 1: "SIGATTN_EINVAL", 2: "SIGATTN_EUNSUPPORTED", 3: "SIGATTN_ECUDA",
                4: "SIGATTN_EWORKSPACE"}

EXPORTED = ["sigattn_fwd", "sigattn_fwd_workspace_bytes", "sigattn_bwd", "sigattn_bwd_workspace_bytes", "sigattn_mask_to_seqlens",
            "sigattn_valid_flops", "sigattn_worklist_host", "sigattn_last_error", "sigattn_version",
            "sigattn_launch_count", "sigattn_set_profile_events", "sigattn_set_trace_buffer",
            "sigattn_set_debug_counters", "sigattn_mask_to_index", "sigattn_permute_rows",
            "sigattn_fwd_cp", "sigattn_bwd_cp", "sigattn_bwd_cp_workspace_bytes", "sigattn_cp_finalize",
            "sigattn_ipc_handle_bytes", "sigattn_ipc_export", "sigattn_ipc_import", "sigattn_ipc_close",
            "sigattn_copy_valid_rows"]


class SigattnParams(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int), ("H", ctypes.c_int), ("Nq", ctypes.c_int), ("Nk", ctypes.c_int),
        ("d", ctypes.c_int), ("dtype", ctypes.c_int),
        ("seqlens_q", ctypes.c_void_p), ("seqlens_k", ctypes.c_void_p),
        ("scale", ctypes.c_float), ("bias", ctypes.c_float),
        ("bias_per_seq", ctypes.c_void_p), ("flags", ctypes.c_uint),
        ("dbias", ctypes.c_void_p),
    ]


class SigattnCpParams(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int), ("rank", ctypes.c_int), ("peer_acc", ctypes.c_void_p)]


class SigattnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    """Load libsigattn.so (or $SIGATTN_LIB, e.g. a trace build); raises if missing (no fallback)."""
    global _lib, LIB_PATH
    if _lib is not None:
        return _lib
    LIB_PATH = os.environ.get("SIGATTN_LIB", LIB_PATH)
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2604_27124_b200.build` "
                          "or __graft_entry__.build() -- there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(SigattnParams)
    vp = ctypes.c_void_p
    lib.sigattn_fwd.argtypes = [P, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.sigattn_fwd.restype = ctypes.c_int
    lib.sigattn_fwd_workspace_bytes.argtypes = [P]
    lib.sigattn_fwd_workspace_bytes.restype = ctypes.c_size_t
    lib.sigattn_bwd.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.sigattn_bwd.restype = ctypes.c_int
    lib.sigattn_bwd_workspace_bytes.argtypes = [P]
    lib.sigattn_bwd_workspace_bytes.restype = ctypes.c_size_t
    lib.sigattn_mask_to_seqlens.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
    lib.sigattn_mask_to_seqlens.restype = ctypes.c_int
    lib.sigattn_valid_flops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int]
    lib.sigattn_valid_flops.restype = ctypes.c_int64
    lib.sigattn_worklist_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          vp, vp, vp, ctypes.c_int64]
    lib.sigattn_worklist_host.restype = ctypes.c_int64
    lib.sigattn_launch_count.restype = ctypes.c_int64
    lib.sigattn_set_profile_events.argtypes = [vp, vp, vp, vp]
    lib.sigattn_set_profile_events.restype = None
    lib.sigattn_set_trace_buffer.argtypes = [vp]
    lib.sigattn_set_trace_buffer.restype = None
    # newer entry points: typed when present (an older experimental build loaded through $SIGATTN_LIB
    # for an A/B may predate them; test_abi_cpu checks that the in-tree library exports every one)
    if hasattr(lib, "sigattn_set_debug_counters"):
        lib.sigattn_set_debug_counters.argtypes = [vp]
        lib.sigattn_set_debug_counters.restype = None
    if hasattr(lib, "sigattn_mask_to_index"):
        lib.sigattn_mask_to_index.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        lib.sigattn_mask_to_index.restype = ctypes.c_int
    if hasattr(lib, "sigattn_permute_rows"):
        lib.sigattn_permute_rows.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, vp]
        lib.sigattn_permute_rows.restype = ctypes.c_int
    if hasattr(lib, "sigattn_copy_valid_rows"):
        lib.sigattn_copy_valid_rows.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                                ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int64)]
        lib.sigattn_copy_valid_rows.restype = ctypes.c_int
    if hasattr(lib, "sigattn_fwd_cp"):
        CP = ctypes.POINTER(SigattnCpParams)
        lib.sigattn_fwd_cp.argtypes = [P, CP, vp, vp, vp, vp, ctypes.c_size_t, vp]
        lib.sigattn_fwd_cp.restype = ctypes.c_int
        lib.sigattn_bwd_cp.argtypes = [P, CP, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
        lib.sigattn_bwd_cp.restype = ctypes.c_int
        lib.sigattn_bwd_cp_workspace_bytes.argtypes = [P]
        lib.sigattn_bwd_cp_workspace_bytes.restype = ctypes.c_size_t
        lib.sigattn_cp_finalize.argtypes = [P, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        lib.sigattn_cp_finalize.restype = ctypes.c_int
        lib.sigattn_ipc_handle_bytes.argtypes = []
        lib.sigattn_ipc_handle_bytes.restype = ctypes.c_size_t
        lib.sigattn_ipc_export.argtypes = [vp, vp]
        lib.sigattn_ipc_export.restype = ctypes.c_int
        lib.sigattn_ipc_import.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
        lib.sigattn_ipc_import.restype = ctypes.c_int
        lib.sigattn_ipc_close.argtypes = [vp]
        lib.sigattn_ipc_close.restype = ctypes.c_int
    lib.sigattn_last_error.restype = ctypes.c_char_p
    lib.sigattn_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(status: int):
    if status != SIGATTN_OK:
        raise SigattnError(status, load().sigattn_last_error().decode())


def make_params(B, H, Nq, Nk, d, dtype_code, seqlens_q_ptr, seqlens_k_ptr, scale, bias, bias_ptr, flags,
                dbias_ptr=None):
    return SigattnParams(int(B), int(H), int(Nq), int(Nk), int(d), int(dtype_code), seqlens_q_ptr or None,
                         seqlens_k_ptr or None, float(scale), float(bias), bias_ptr or None, int(flags),
                         dbias_ptr or None)
