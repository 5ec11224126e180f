#!/usr/bin/env python3
"""Diagnostic: per-voxel speed of the warp kernel on a C3-shaped batch whose boxes are
small (mild transforms: rotations <= ROT degrees, no shear, scale 1), so every volume's
16-row box fits the buffer of either occupancy build (-DW3D_MINB=3 or 4).  Prints the
kernel time per batch and the box sizes.  usage: ROT=5 python tools/occ_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402
import synth  # noqa: E402

rot = float(os.environ.get("ROT", "5"))
R = synth.AugmentRanges(rot_deg=(rot, rot, rot), scale=(1.0, 1.0), shear=0.0)
shape, B = (160, 128, 128), 16
vids = list(range(B))
params = build_params([synth.draw(R, v) for v in vids], vids, shape, shape, FULL,
                      seed=synth.MASTER_SEED)
img = torch.randn((B, *shape), device="cuda") * 100
lbl = torch.randint(0, 6, (B, *shape), dtype=torch.uint8, device="cuda")
batch = W.AugmentBatch(img, lbl, params, fill=-1000.0)
for _ in range(5):
    batch.run()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(50):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    batch.run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
print(f"rot {rot}: {ms * 1e3:.1f} us per batch, {B * 160 * 128 * 128 / ms / 1e6:.1f} GVoxel/s, "
      f"tiles {W.warp3d_tile_stats()}")
