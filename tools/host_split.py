#!/usr/bin/env python3
"""Where the host time of one C2 call goes: the binding's Python (argument checks and
marshalling) vs the C entry point (parameter derivation, boxes, tensor maps, launch).
usage: python tools/host_split.py"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build  # noqa: E402
build.build_cuda()
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200 import _lib as L  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
shape = (160, 128, 128)
B = 1
params = build_params([synth.draw(synth.TRAIN, 0)], [0], shape, shape, FULL, seed=synth.MASTER_SEED)
img = torch.zeros((B, *shape), device=dev)
lbl = torch.zeros((B, *shape), dtype=torch.uint8, device=dev)
batch = W.AugmentBatch(img, lbl, params, fill=-1000.0)
lib = L.load()
args = (B, ctypes.c_void_p(img.data_ptr()), ctypes.c_void_p(lbl.data_ptr()), L.dims(shape), params,
        0, -1000.0, 0, ctypes.c_void_p(batch.out.data_ptr()),
        ctypes.c_void_p(batch.out_labels.data_ptr()), L.dims(shape), 0,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


def t(fn, n=200):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # keep the launches queued behind a long kernel
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return dt


print(f"batch.run()            {t(batch.run):7.2f} us per call")
print(f"raw C call (ctypes)    {t(lambda: lib.warp3d_affine_batched_ex(*args)):7.2f} us per call")
print(f"torch current_stream   {t(lambda: torch.cuda.current_stream().cuda_stream):7.2f} us")
