#!/usr/bin/env python3
"""Design aid (not a test): shared-memory wavefronts per corner LDS of the staged warp
kernel for the C3 batch, with the box pitches the host picks (cube_cp_box's residue
rule) against the best (W, H) padding per volume.  Lanes: 16 consecutive output x by 2
output z per warp; every thread walks the tile's 16 rows in y."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_11226_b200 as W  # noqa: E402
from paper_1811_11226_b200.augment import FULL, build_params  # noqa: E402
import synth  # noqa: E402

shape = (160, 128, 128)
nz, ny, nx = shape
B = 16
vids = list(range(B))
params = build_params([synth.draw(synth.TRAIN, v) for v in vids], vids, shape, shape, FULL,
                      seed=synth.MASTER_SEED)
CAP = (233472 // 3 - 1024 - 272) // 5 * 4  # image bytes of the staging buffer, roughly


def wavefronts(words):
    banks = words % 32
    best = np.ones(words.shape[0])
    for b in range(32):
        sel = banks == b
        for i in np.nonzero(sel.any(1))[0]:
            best[i] = max(best[i], len(np.unique(words[i][sel[i]])))
    return best


def model(A, Wp, Hp, rng, ntiles=24):
    Af = A.astype(np.float32)
    tiles = [(x, y, z) for z in range(0, nz, 16) for y in range(0, ny, 16) for x in range(0, nx, 16)]
    res = []
    for ti in rng.choice(len(tiles), ntiles, replace=False):
        ox, oy, oz = tiles[ti]
        lane = np.arange(32)
        X = ox + (lane & 15)
        wf = []
        for w in range(8):
            Z = oz + 2 * w + (lane >> 4)
            for y in range(oy, oy + 16, 3):
                p = [Af[k, 0] * X + Af[k, 1] * y + Af[k, 2] * Z + Af[k, 3] for k in range(3)]
                f = [np.floor(q).astype(np.int64) for q in p]
                idx = f[0] + Wp * f[1] + Wp * Hp * f[2]
                for off in (0, 1, Wp, Wp + 1):
                    wf.append(wavefronts((idx + off)[None, :])[0])
        res.append(np.mean(wf))
    return float(np.mean(res))


rng = np.random.default_rng(3)
tot_cur, tot_best = [], []
for i, p in enumerate(params):
    A = np.array(p.affine, dtype=np.float32).reshape(3, 4)
    span = np.array([15.0, 15.0, 15.0])
    ext = [float(np.sum(np.abs(A[k, :3]) * span)) for k in range(3)]
    d = [int(np.floor(e + 0.01)) + 3 for e in ext]
    W0, H0, D = (d[0] + 3 + 3) & ~3, d[1], d[2]
    cur = None
    cands = []
    for Wc in (W0, W0 + 4, W0 + 8):
        for h in range(H0, H0 + 8):
            if Wc * h * D * 4 > CAP:
                continue
            res = (Wc * h) & 31
            cands.append((Wc, h))
            if cur is None and Wc <= W0 + 4 and res in (12, 16, 20, 24):
                cur = (Wc, h)
    cur = cur or (W0, H0)
    r = np.random.default_rng(i)
    wc = model(A, *cur, r)
    scored = sorted((model(A, Wc, h, np.random.default_rng(i)), Wc, h) for Wc, h in cands)
    tot_cur.append(wc)
    tot_best.append(scored[0][0])
    print(f"vol {i:2d} box {W0}x{H0}x{D}: current {cur} {wc:.2f} wf/LDS, best {scored[0][1:]} "
          f"{scored[0][0]:.2f}, unpadded {model(A, W0, H0, np.random.default_rng(i)):.2f}")
print(f"mean current {np.mean(tot_cur):.3f}, best {np.mean(tot_best):.3f}")
