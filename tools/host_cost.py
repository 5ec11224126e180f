#!/usr/bin/env python3
"""Host-side cost of one warp3d_affine_batched call (argument marshalling, per-volume
parameter derivation, staging boxes, tensor-map encodes, launches) against its GPU time,
for a 16-volume (C3) and a 256-volume (C5) batch.  usage: python tools/host_cost.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build  # noqa: E402
build.build_cuda()
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
shape = (160, 128, 128)
for B in (1, 16, 256):
    vids = list(range(B))
    params = build_params([synth.draw(synth.TRAIN, v) for v in vids], vids, shape, shape, FULL,
                          seed=synth.MASTER_SEED)
    img = torch.zeros((B, *shape), dtype=torch.float32, device=dev)
    lbl = torch.zeros((B, *shape), dtype=torch.uint8, device=dev)
    batch = W.AugmentBatch(img, lbl, params, fill=-1000.0)
    for _ in range(3):
        batch.run()
    torch.cuda.synchronize()
    host, gpu = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(50_000_000)  # keep the GPU busy so the calls queue up
        e0.record()
        t0 = time.perf_counter()
        batch.run()
        host.append((time.perf_counter() - t0) * 1e3)
        e1.record()
        torch.cuda.synchronize()
        gpu.append(e0.elapsed_time(e1))
    print(f"B={B}: host {np.median(host):.3f} ms per call, GPU {np.median(gpu):.3f} ms per call")
