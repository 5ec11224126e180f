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


def build_oracle(force=False, sanitize=False):
    """The C oracle (test infrastructure).  sanitize=True: the same sources with
    AddressSanitizer + UndefinedBehaviorSanitizer (no recovery: the first report
    aborts) into oracle/liboracle_warp3d_asan.so, loaded with libasan preloaded."""
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("oracle_warp3d.c", "oracle_resample.c")]
    hdr = os.path.join(ROOT, "oracle", "oracle_warp3d.h")
    name = "liboracle_warp3d_asan.so" if sanitize else "liboracle_warp3d.so"
    out = os.path.join(ROOT, "oracle", name)
    san = (["-fsanitize=address,undefined", "-fno-sanitize-recover=all",
            "-fno-omit-frame-pointer", "-g"] if sanitize else [])
    if force or _stale(out, srcs + [hdr]):
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
              "-shared", "-Wall", "-Wextra", "-D_GNU_SOURCE", *san, "-o", out, *srcs, "-lm"])
    return out


CUDA_SOURCES = [
    "paper_1811_11226_b200/csrc/warp3d_host.cu",
    "paper_1811_11226_b200/csrc/warp3d_cube.cu",
    "paper_1811_11226_b200/csrc/cube_inst_f32_s.cu",
    "paper_1811_11226_b200/csrc/cube_inst_f32_l.cu",
    "paper_1811_11226_b200/csrc/cube_inst_i16_s.cu",
    "paper_1811_11226_b200/csrc/cube_inst_i16_l.cu",
    "paper_1811_11226_b200/csrc/warp3d_aux.cu",
    "paper_1811_11226_b200/csrc/warp3d_resample.cu",
]
CUDA_HEADERS = [
    "include/warp3d.h",
    "paper_1811_11226_b200/csrc/warp3d_internal.cuh",
    "paper_1811_11226_b200/csrc/philox.cuh",
    "paper_1811_11226_b200/csrc/cube_config.cuh",
    "paper_1811_11226_b200/csrc/cube_kernel.cuh",
]
PRODUCT_LIB = os.path.join(ROOT, "paper_1811_11226_b200", "libwarp3d.so")


def _flags(extra):
    # No --use_fast_math and -fmad=false: the coordinate contract (R4)
    # and the trilinear lerp nesting use explicit __fmaf_rn, never contraction.
    return [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-fmad=false",
            "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), *extra]


def build_cuda(force=False, out=None, extra=None):
    """Compile every CUDA unit to an object in parallel, then link the shared library.

    extra: additional nvcc flags (default: $W3D_NVCC_EXTRA, experiment knobs such as
    -DW3D_TZ=16).  The flags are recorded in a stamp file next to the library and a
    build with different flags always rebuilds, so a knob build can never be mistaken
    for the product build (or the reverse).  out: library path (default: the product
    library the package loads)."""
    import concurrent.futures as cf
    import hashlib
    import json
    extra = os.environ.get("W3D_NVCC_EXTRA", "").split() if extra is None else list(extra)
    out = out or PRODUCT_LIB
    srcs = [os.path.join(ROOT, s) for s in CUDA_SOURCES]
    hdrs = [os.path.join(ROOT, h) for h in CUDA_HEADERS]
    flags = _flags(extra)
    stamp = out + ".flags"
    want = json.dumps({"nvcc": NVCC, "flags": flags, "sources": CUDA_SOURCES})
    have = open(stamp).read() if os.path.exists(stamp) else None
    if not (force or have != want or _stale(out, srcs + hdrs)):
        return out
    tag = hashlib.sha1(want.encode()).hexdigest()[:10]
    objdir = os.path.join(ROOT, "build", "obj", tag)
    os.makedirs(objdir, exist_ok=True)

    def obj_of(src):
        return os.path.join(objdir, os.path.basename(src)[:-3] + ".o")

    def compile_one(src):
        o = obj_of(src)
        if force or _stale(o, [src] + hdrs):
            _run([NVCC, *flags, "-c", "-o", o, src])
        return o

    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    if os.path.exists(stamp):
        os.remove(stamp)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs])
    with open(stamp, "w") as f:
        f.write(want)
    return out


def main(argv):
    what = argv[1] if len(argv) > 1 else "all"
    force = "--force" in argv
    if what in ("oracle", "all"):
        build_oracle(force)
    if what == "oracle-asan":
        build_oracle(force, sanitize=True)
    if what in ("cuda", "all"):
        build_cuda(force)


if __name__ == "__main__":
    main(sys.argv)
