#!/usr/bin/env python3
"""End-to-end rate of the host FIFO pipeline (warp3d_pipeline_run, chained calls) on the C3
workload for several slot depths.  usage: python tools/e2e_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build  # noqa: E402
build.build_cuda()
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402
import synth  # noqa: E402

shape = (160, 128, 128)
B = 16
vids = list(range(B))
params = build_params([synth.draw(synth.TRAIN, v) for v in vids], vids, shape, shape, FULL,
                      seed=synth.MASTER_SEED)
rng = np.random.default_rng(0)
h_img = torch.from_numpy(rng.normal(0, 300, (B, *shape)).astype(np.float32)).pin_memory()
h_lbl = torch.from_numpy(rng.integers(0, 6, (B, *shape), dtype=np.uint8)).pin_memory()
h_out = torch.empty((B, *shape), dtype=torch.float32).pin_memory()
h_out_l = torch.empty((B, *shape), dtype=torch.uint8).pin_memory()
nvox = B * int(np.prod(shape))
for depth in (2, 3, 4, 6, 8):
    for chain in (False, True):
        pipe = W.Pipeline(shape, shape, depth=depth, labels=True, chain=chain)
        for _ in range(2):
            pipe.run(h_img, h_lbl, params, h_out, h_out_l, fill=-1000.0)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            pipe.run(h_img, h_lbl, params, h_out, h_out_l, fill=-1000.0)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        print(f"depth {depth} chain {int(chain)}: {nvox * 10 / (ms * 1e-3) / 1e9:.2f} GVoxel/s")
        pipe.close()
