"""Build libgvom.so (the C-ABI CUDA library) in-tree for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false ...
-fmad=false (plus explicit _rn intrinsics in the kernels) keeps every float
step that decides an integer bit-identical to the oracle's float32 rule.
The static CUDA runtime is linked in; torch is not needed to build.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libgvom.so")
SOURCES = ["k_integrate.cu", "k_maps.cu", "k_slab.cu", "k_roll.cu", "gvom_api.cu"]
HEADERS = ["gvom_internal.cuh", "gvom_device.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-fvisibility=hidden",
    "-I", INCLUDE,
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "gvom.h"),
                                                                os.path.abspath(__file__)]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), "-shared", "-cudart", "static",
                           "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp])
    os.replace(tmp, LIB)
    return LIB


PROBE_SRC = os.path.join(CSRC, "probe", "l2_red_probe.cu")
PROBE_LIB = os.path.join(LIBDIR, "libgvom_probe.so")


def build_probe(force: bool = False) -> str:
    """The L2-reduction microbenchmark (a measurement tool for bench.py's
    roofline, not part of the gvom ABI)."""
    if not force and os.path.exists(PROBE_LIB) and \
            os.path.getmtime(PROBE_LIB) >= os.path.getmtime(PROBE_SRC):
        return PROBE_LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = PROBE_LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *NVCC_FLAGS, "-shared", "-cudart", "static", PROBE_SRC,
                           "-o", tmp])
    os.replace(tmp, PROBE_LIB)
    return PROBE_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
