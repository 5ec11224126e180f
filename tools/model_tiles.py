#!/usr/bin/env python3
"""CPU model of the staged tile kernel's memory behaviour (design aid, not a test).

For the C3 workload's train transforms it estimates, per candidate tile shape /
lane mapping / shared-memory pitch rule:
  * inflation   = staged box voxels / output voxels (L2 -> smem traffic, capacity),
  * wavefronts  = shared-memory wavefronts per LDS instruction (bank conflicts) for
                  the 8 trilinear corners and the nearest label,
  * over_cap    = fraction of tiles whose box exceeds a capacity.
Coordinates are evaluated in float32 like the kernel (sufficient for a model).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402


def affines(n, ranges, shape):
    out = []
    for i in range(n):
        d = synth.draw(ranges, i)
        g = O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp)
        out.append(O.compose_affine(g, shape, shape)[1])
    return out


def wavefronts(words):
    """words: int array [warps, 32] of 4-byte word addresses -> wavefronts per warp."""
    banks = words % 32
    res = np.empty(words.shape[0])
    for w in range(words.shape[0]):
        m = 1
        for b in np.unique(banks[w]):
            m = max(m, len(np.unique(words[w][banks[w] == b])))
        res[w] = m
    return res


def model(A, shape, tile, lanes, pitch_rule, rng, n_tiles=60, cap=None):
    nz, ny, nx = shape
    TX, TY, TZ = tile
    LX, LY = lanes  # a warp = LX consecutive x times LY consecutive y
    infl, wf_img, wf_lbl, over = [], [], [], 0
    tiles = [(x, y, z) for z in range(0, nz, TZ) for y in range(0, ny, TY) for x in range(0, nx, TX)]
    pick = rng.choice(len(tiles), size=min(n_tiles, len(tiles)), replace=False)
    Af = A.astype(np.float32)
    for ti in pick:
        ox, oy, oz = tiles[ti]
        xs = np.arange(ox, min(ox + TX, nx))
        ys = np.arange(oy, min(oy + TY, ny))
        zs = np.arange(oz, min(oz + TZ, nz))
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        P = [Af[k, 0] * X + Af[k, 1] * Y + Af[k, 2] * Z + Af[k, 3] for k in range(3)]
        P = [p.astype(np.float32) for p in P]
        lo = [int(np.floor(np.clip(p.min(), -1, n))) for p, n in zip(P, (nx, ny, nz))]
        hi = [int(np.floor(np.clip(p.max(), -1, n))) + 1 for p, n in zip(P, (nx, ny, nz))]
        bx = lo[0] & ~3
        Wn = hi[0] - bx + 1
        H = hi[1] - lo[1] + 1
        D = hi[2] - lo[2] + 1
        W = pitch_rule(Wn)
        infl.append(W * H * D / X.size)
        if cap is not None and W * H * D > cap:
            over += 1
        F = [np.floor(np.clip(p, -1, n)) for p, n in zip(P, (nx, ny, nz))]
        T = [np.clip(p, -1, n) - f for p, f, n in zip(P, F, (nx, ny, nz))]
        li = (F[0] - bx) + W * (F[1] - lo[1]) + W * H * (F[2] - lo[2])
        li = li.astype(np.int64)
        ln = li + (T[0] >= 0.5) + W * (T[1] >= 0.5) + W * H * (T[2] >= 0.5)
        # group into warps: lanes = LX x-consecutive, LY y-consecutive
        sh = li.shape  # [z, y, x]
        if sh[2] % LX or sh[1] % LY:
            continue
        def warps(a):
            a = a.reshape(sh[0], sh[1] // LY, LY, sh[2] // LX, LX)
            return a.transpose(0, 1, 3, 2, 4).reshape(-1, LX * LY)
        for off in (0, 1, W, W + 1, W * H, W * H + 1, W * H + W, W * H + W + 1):
            wf_img.append(wavefronts(warps(li + off)).mean())
        wf_lbl.append(wavefronts(warps(ln) // 4).mean())
    return np.mean(infl), np.mean(wf_img), np.mean(wf_lbl), over / len(pick)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vols", type=int, default=6)
    ap.add_argument("--tiles", type=int, default=30)
    ap.add_argument("--ranges", default="train")
    args = ap.parse_args()
    shape = (160, 128, 128) if args.ranges == "train" else (512, 512, 512)
    ranges = synth.TRAIN if args.ranges == "train" else synth.LARGE
    As = affines(args.vols, ranges, shape)
    rules = {
        "r4": lambda w: (w + 3) & ~3,
        "r32": lambda w: (w + 31) & ~31,
        "r4+32odd": lambda w: ((w + 3) & ~3) if ((w + 3) & ~3) % 64 == 32 else (((w + 3) & ~3) // 32) * 32 + 32,
        "r8o": lambda w: ((w + 7) & ~7) + (8 if ((w + 7) & ~7) % 32 == 0 else 0),
    }
    configs = [
        ((32, 16, 8), (32, 1)),
        ((32, 8, 8), (32, 1)),
        ((16, 16, 16), (16, 2)),
        ((32, 16, 16), (32, 1)),
        ((16, 16, 8), (16, 2)),
        ((32, 32, 8), (32, 1)),
        ((32, 32, 4), (32, 1)),
        ((16, 32, 8), (16, 2)),
        ((8, 32, 16), (8, 4)),
    ]
    rng = np.random.default_rng(1)
    print(f"{'tile':>12} {'lanes':>7} {'pitch':>9} {'infl':>6} {'wf/LDS img':>10} {'wf lbl':>7} {'>14592':>7}")
    for tile, lanes in configs:
        for name, rule in rules.items():
            r = [model(A, shape, tile, lanes, rule, rng, args.tiles, cap=14592) for A in As]
            r = np.mean(np.array(r), axis=0)
            print(f"{str(tile):>12} {str(lanes):>7} {name:>9} {r[0]:6.2f} {r[1]:10.2f} {r[2]:7.2f} {r[3]:7.2f}")


if __name__ == "__main__":
    main()
