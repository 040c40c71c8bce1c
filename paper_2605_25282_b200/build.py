"""In-tree build of libvlbm_b200.so (sm_100a) with nvcc + g++.

The library is built IN the source tree (paper_2605_25282_b200/lib/) so it
travels to the GPU box with the gpurun snapshot.  Numerics flags:
``--fmad=false`` (no FMA contraction: bit parity with the reference's x86-64
build), IEEE div/sqrt (nvcc defaults; never --use_fast_math).
"""
from __future__ import annotations

import os
import shlex
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(PKG, "lib", "libvlbm_b200.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr", "-I", INCLUDE,
] + shlex.split(os.environ.get("VLBM_NVCC_EXTRA", ""))  # experiment hook (tools/ab variants)
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-I", INCLUDE,
             "-I", "/usr/local/cuda/include"]

CU_SOURCES = ["march.cu", "march_tiled.cu", "post.cu", "capi.cu", "metrics_ctx.cu"]
CPP_SOURCES = ["host_ic.cpp"]
HEADERS = ["vlbm_device.cuh", "march.cuh", "march_common.cuh", "rlmp.cuh", "rlmp_replay.cuh", "internal.h"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    if verbose and r.stderr.strip():
        sys.stderr.write(r.stderr)


def build(verbose: bool = False, ptxas_v: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "vlbm_b200.h"),
                                                         __file__]
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + common):
            flags = NVCC_FLAGS + (["-Xptxas", "-v"] if ptxas_v else [])
            _run([NVCC, *flags, "-c", s, "-o", o], verbose or ptxas_v)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + common):
            _run([CXX, *CXX_FLAGS, "-c", s, "-o", o], verbose)
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-lpthread",
              "-ldl"], verbose)
    return LIB


if __name__ == "__main__":
    build(verbose=True, ptxas_v="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
