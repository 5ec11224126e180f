#!/usr/bin/env python3
"""Build the two native libraries in-tree.

  oracle/liboracle_warp3d.so                 plain C oracle (gcc, -ffp-contract=off)
  paper_1811_11226_b200/libwarp3d.so         CUDA path for sm_100a (nvcc) + C-ABI host code

The two share no source file or header.  Usage: python build.py [oracle|cuda|all]
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_oracle(force=False):
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("oracle_warp3d.c", "oracle_resample.c")]
    hdr = os.path.join(ROOT, "oracle", "oracle_warp3d.h")
    out = os.path.join(ROOT, "oracle", "liboracle_warp3d.so")
    if force or _stale(out, srcs + [hdr]):
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
              "-shared", "-Wall", "-Wextra", "-D_GNU_SOURCE", "-o", out, *srcs, "-lm"])
    return out


CUDA_SOURCES = [
    "paper_1811_11226_b200/csrc/warp3d_host.cu",
    "paper_1811_11226_b200/csrc/warp3d_cube.cu",
    "paper_1811_11226_b200/csrc/warp3d_aux.cu",
    "paper_1811_11226_b200/csrc/warp3d_resample.cu",
]
CUDA_HEADERS = [
    "include/warp3d.h",
    "paper_1811_11226_b200/csrc/warp3d_internal.cuh",
    "paper_1811_11226_b200/csrc/philox.cuh",
]


def build_cuda(force=False):
    srcs = [os.path.join(ROOT, s) for s in CUDA_SOURCES]
    hdrs = [os.path.join(ROOT, h) for h in CUDA_HEADERS]
    out = os.path.join(ROOT, "paper_1811_11226_b200", "libwarp3d.so")
    if force or _stale(out, srcs + hdrs):
        # No --use_fast_math and -fmad=false: the coordinate contract (R4)
        # and the trilinear lerp nesting use explicit __fmaf_rn, never contraction.
        extra = os.environ.get("W3D_NVCC_EXTRA", "").split()  # experiment knobs (-DW3D_TZ=16)
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
              "-fmad=false", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), *extra,
              "-o", out, *srcs])
    return out


def main(argv):
    what = argv[1] if len(argv) > 1 else "all"
    force = "--force" in argv
    if what in ("oracle", "all"):
        build_oracle(force)
    if what in ("cuda", "all"):
        build_cuda(force)


if __name__ == "__main__":
    main(sys.argv)
