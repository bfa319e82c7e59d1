"""Build libzs.so (sm_100a) in-tree with nvcc.

    python -m paper_2603_17435_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libzs.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["zs_api.cu", "zs_decompress.cu", "zs_gemm.cu", "zs_encode_gpu.cu", "zs_peer.cu"]
CPP_SOURCES = ["zs_encode.cpp"]
HEADERS = ["zs_device.cuh", "zs_kernels.h", "zs_host.h", "zs_lut.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile libzs.so (or, with `defines`, a debug variant at `lib`, e.g. -DZS_TRACE=1)."""
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CPP_SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "zs.h"), __file__]
    if not force and not _stale(lib, deps):
        return lib
    objdir = os.path.join(PKG, "build" if lib == LIB else "build_" + os.path.basename(lib).split(".")[0])
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if s.endswith(".cu"):
            cmd = [NVCC, *ARCH, *COMMON, *defines, "-Xptxas", "-v" if verbose else "-O3", "-c", s, "-o", o]
        else:
            cmd = [NVCC, *ARCH, *COMMON, "-x", "c++", "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs,
                           "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-lcublas", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--trace2" in sys.argv:  # MMA-warp timeline (events 7..11 = MMA loop steps)
        build(force=True, verbose=True, defines=["-DZS_TRACE=2"], lib=os.path.join(PKG, "libzs_trace2.so"))
    elif "--trace" in sys.argv:   # timeline build for scripts/trace_gemm.py (ZS_LIB=...libzs_trace.so)
        build(force=True, verbose=True, defines=["-DZS_TRACE=1"], lib=os.path.join(PKG, "libzs_trace.so"))
    else:
        build(force="--force" in sys.argv, verbose=True)
