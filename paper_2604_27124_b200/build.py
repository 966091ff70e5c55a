"""Build libsigattn.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsigattn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC,-O2",
    "-I", os.path.join(ROOT, "include"),
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "sigattn.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, extra=None) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [NVCC] + NVCC_FLAGS + (list(extra) if extra else []) + [os.path.join(CSRC, "sigattn.cu"), "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_trace() -> str:
    """Debug build with -DSIGATTN_TRACE=1 (clock64 pipeline timestamps) -> libsigattn_trace.so."""
    out = os.path.join(PKG, "libsigattn_trace.so")
    cmd = [NVCC] + NVCC_FLAGS + ["-DSIGATTN_TRACE=1", os.path.join(CSRC, "sigattn.cu"), "-o", out]
    subprocess.check_call(cmd)
    return out


def build_variant(name: str, defines) -> str:
    """Experimental build with extra -D flags -> libsigattn_<name>.so (selected with $SIGATTN_LIB).
    Timing-only SIGATTN_DBG_* switches (wrong results, csrc/debug.cuh) get -DSIGATTN_DEBUG_BUILD."""
    out = os.path.join(PKG, f"libsigattn_{name}.so")
    defines = list(defines)
    if any(d.startswith("SIGATTN_DBG_") for d in defines):
        defines.append("SIGATTN_DEBUG_BUILD")
    cmd = [NVCC] + NVCC_FLAGS + [f"-D{d}" for d in defines] + [os.path.join(CSRC, "sigattn.cu"), "-o", out]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
