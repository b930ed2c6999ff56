"""Build libwsb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libwsb200.so")
CHECK_LIB = os.path.join(PKG, "libwsb200_check.so")   # the bounds-check build (-DWS_CHECK, ws_check_read)
SRCS = [os.path.join(PKG, "csrc", f) for f in ("ws_api.cu", "ws_kernels.cu", "ws_validate.cu")]
DEPS = SRCS + [os.path.join(PKG, "csrc", "ws_internal.cuh"), os.path.join(ROOT, "include", "ws.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-I" + os.path.join(ROOT, "include")]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force=False, verbose=False, extra=(), out=None):
    if not force and not stale() and out is None:
        return LIB
    cmd = [NVCC] + FLAGS + list(extra) + (["-Xptxas", "-v"] if verbose else []) + ["-o", out or LIB] + SRCS
    subprocess.check_call(cmd)
    return LIB


def build_check(force=False):
    """The bounds-check build of the same sources (tests/test_bounds_check.py loads it via WS_LIB)."""
    if force or not os.path.exists(CHECK_LIB) or any(os.path.getmtime(d) > os.path.getmtime(CHECK_LIB) for d in DEPS):
        build(force=True, extra=["-DWS_CHECK"], out=CHECK_LIB)
    return CHECK_LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
