#!/usr/bin/env python3
"""Small invocations of every kernel path through the product binding, for
compute-sanitizer (tools/sanitize.sh): memcheck / racecheck / synccheck / initcheck.

Cases: C1 (32^3, fixed affine, noise), C2 (one 128x128x160 CT volume, full chain),
a 3-volume slice of C3, the large-footprint case (2/4-part sub-tiles, gathered
parts, clamped boxes), int16 input, occlusion, nearest image, a ragged nx % 4 != 0
layout (gather-only), mixed-dims batches and the resampling kernels -- each on the
AUTO (TMA-staged), STAGED and GATHER variants where they differ.  Exits non-zero on
any CUDA error; the sanitizer's own error exit code does the rest."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402

QUICK = "--quick" in sys.argv  # racecheck: skip the largest cases


def batch(shape, B, ranges, flags=FULL, first=0, occl=False):
    base = [synth.phantom(shape, seed=synth.MASTER_SEED + k) for k in range(min(B, 2))]
    imgs = np.stack([base[i % len(base)][0] for i in range(B)])
    lbls = np.stack([base[i % len(base)][1] for i in range(B)])
    if ranges is None:
        ds = [synth.C1_DRAW] * B
    else:
        ds = [synth.draw(ranges, first + i, out_mz=shape[0] if occl else None) for i in range(B)]
    params = build_params(ds, list(range(first, first + B)), shape, shape, flags,
                          seed=synth.MASTER_SEED)
    return torch.from_numpy(imgs).cuda(), torch.from_numpy(lbls).cuda(), params


def run(name, img, lbl, params, variants=(0, 1, 2), **kw):
    for v in variants:
        W.warp3d_affine_batched(img, lbl, params, fill=-1000.0, label_fill=0, variant=v, **kw)
        torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    img, lbl, ps = batch((32, 32, 32), 1, None, flags=1)
    run("c1", img, lbl, ps)
    img, lbl, ps = batch((160, 128, 128), 1, synth.TRAIN)
    run("c2", img, lbl, ps, variants=(0, 1) if QUICK else (0, 1, 2))
    if not QUICK:
        img, lbl, ps = batch((160, 128, 128), 3, synth.TRAIN)
        run("c3x3", img, lbl, ps, variants=(0,))
        run("c3x3 int16", img.round().to(torch.int16), lbl, ps, variants=(0, 1))
    img, lbl, ps = batch((48, 40, 64), 2, synth.TRAIN_OCC, occl=True)
    run("occlusion", img, lbl, ps)
    run("nearest", img, lbl, ps, interp=W.INTERP_NEAREST)
    run("no labels", img, None, ps)
    # large footprints: y-parts, gathered parts, clamped (4x zoom-out) boxes
    shape = (96, 96, 96)
    img, lbl, _ = batch(shape, 1, synth.LARGE)
    ds = [synth.draw(synth.LARGE, 40 + i) for i in range(3)]
    ps = build_params(ds, [0, 1, 2], shape, shape, FULL, seed=synth.MASTER_SEED)
    zoom = W.volume_params(np.concatenate([4.0 * np.eye(3), [[-150.0], [-130.0], [-160.0]]],
                                          axis=1).astype(np.float32), ps[0].ph)
    allp = list(ps) + [zoom]
    run("large footprints", img.repeat(4, 1, 1, 1), lbl.repeat(4, 1, 1, 1), allp, variants=(2, 0))
    # ragged layout (nx % 4 != 0): gather-only
    img, lbl, ps = batch((23, 29, 37), 2, synth.TRAIN)
    run("ragged", img, lbl, ps)
    # volumes of different dims into one batch
    a, la, pa = batch((24, 32, 48), 1, synth.TRAIN)
    b, lb, pb = batch((20, 36, 40), 1, synth.TRAIN, first=1)
    W.warp3d_affine_batched_list([a[0], b[0]], [la[0], lb[0]], [pa[0], pb[0]], (24, 32, 32),
                                 fill=-1000.0)
    torch.cuda.synchronize()
    print("ok mixed dims", flush=True)
    # resampling (NEXT-3): fused lowpass + scale warp, and the per-axis passes
    vol = torch.from_numpy(synth.phantom((64, 48, 40))[0]).cuda()
    lv = torch.from_numpy(synth.phantom((64, 48, 40))[1]).cuda()
    W.warp3d_resample(vol, lv, (1.0, 1.0, 1.0), 3.0)
    W.warp3d_smooth3d(vol, (4.0, 0.0, 9.5))
    torch.cuda.synchronize()
    print("ok resample", flush=True)
    print("all cases ok")


if __name__ == "__main__":
    main()
