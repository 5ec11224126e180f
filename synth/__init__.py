"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no coordinate map, no
interpolation, no noise transform, no window).  It only

  * builds a synthetic HU phantom shaped like 3 mm^3 / 1 mm^3 abdominal CT
    (SURVEY.md Sec. 8.d), and
  * draws the per-volume random parameters the method samples "uniformly from
    user-specified ranges".

Both sides receive exactly these numbers; each composes its own affine matrix.
Per-volume draws come from numpy.random.default_rng([master_seed, global_index]),
so a volume's parameters do not depend on batch size, shard or rank.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASTER_SEED = 0x181111226  # recorded in every report
AIR_HU = -1000.0

# label codes (SPEC.md LabelMap: 0 other, 1 lung, 2 liver, 3 bone, 4 kidney, 5 bladder)
OTHER, LUNG, LIVER, BONE, KIDNEY, BLADDER = range(6)


def _ellipsoid(X, Y, Z, c, r):
    return ((X - c[0]) / r[0]) ** 2 + ((Y - c[1]) / r[1]) ** 2 + ((Z - c[2]) / r[2]) ** 2 <= 1.0


def phantom(shape_zyx, seed=MASTER_SEED, texture_sigma=15.0):
    """HU phantom (float32 [nz,ny,nx]) and labels (uint8), deterministic in (shape, seed).

    Air -1000 HU; body ellipsoid 40 HU; two lungs -800; spine shell 700 HU with
    200 HU marrow and a rib shell; liver 60; kidneys 30; bladder 10; iid N(0, 15 HU)
    texture; clipped to the 12-bit CT range [-1024, 3071].
    """
    nz, ny, nx = shape_zyx
    rng = np.random.default_rng([seed, nz, ny, nx])
    img = np.empty(shape_zyx, dtype=np.float32)
    lbl = np.empty(shape_zyx, dtype=np.uint8)
    xs = (np.arange(nx, dtype=np.float32) + 0.5) / nx
    ys = (np.arange(ny, dtype=np.float32) + 0.5) / ny
    X, Y = np.meshgrid(xs, ys, indexing="xy")  # [ny, nx]
    slab = max(1, (1 << 22) // max(1, nx * ny))
    for z0 in range(0, nz, slab):
        z1 = min(nz, z0 + slab)
        Zs = ((np.arange(z0, z1, dtype=np.float32) + 0.5) / nz)[:, None, None]
        Xs, Ys = X[None], Y[None]
        v = np.full((z1 - z0, ny, nx), AIR_HU, dtype=np.float32)
        L = np.zeros((z1 - z0, ny, nx), dtype=np.uint8)
        body = _ellipsoid(Xs, Ys, Zs, (0.5, 0.5, 0.5), (0.42, 0.32, 0.48))
        v[body] = 40.0
        # rib shell: thin ellipsoidal shell in the upper half, in bands along z
        rib = body & ~_ellipsoid(Xs, Ys, Zs, (0.5, 0.5, 0.5), (0.39, 0.29, 0.48)) & \
            (Zs > 0.45) & ((np.floor(Zs * 24.0) % 2) == 0)
        v[rib] = 700.0
        L[rib] = BONE
        for cx in (0.33, 0.67):
            lung = _ellipsoid(Xs, Ys, Zs, (cx, 0.45, 0.72), (0.12, 0.15, 0.2))
            v[lung] = -800.0
            L[lung] = LUNG
        liver = _ellipsoid(Xs, Ys, Zs, (0.36, 0.5, 0.45), (0.14, 0.12, 0.12))
        v[liver] = 60.0
        L[liver] = LIVER
        for cx in (0.35, 0.65):
            kid = _ellipsoid(Xs, Ys, Zs, (cx, 0.64, 0.38), (0.05, 0.06, 0.08))
            v[kid] = 30.0
            L[kid] = KIDNEY
        blad = _ellipsoid(Xs, Ys, Zs, (0.5, 0.45, 0.12), (0.08, 0.07, 0.06))
        v[blad] = 10.0
        L[blad] = BLADDER
        # spine: cylinder along z, cortical shell 700 HU around 200 HU marrow
        rr = np.sqrt(((Xs - 0.5) / 0.05) ** 2 + ((Ys - 0.74) / 0.05) ** 2)
        spine = (rr <= 1.0) & body
        spine = np.broadcast_to(spine, v.shape)
        v[spine] = np.where(np.broadcast_to(rr, v.shape)[spine] >= 0.6, 700.0, 200.0)
        L[spine] = BONE
        v += rng.standard_normal(v.shape, dtype=np.float32) * np.float32(texture_sigma)
        np.clip(v, -1024.0, 3071.0, out=v)
        img[z0:z1] = v
        lbl[z0:z1] = L
    return img, lbl


@dataclass(frozen=True)
class AugmentRanges:
    """User-specified uniform ranges."""
    rot_deg: tuple = (15.0, 15.0, 15.0)       # +- per axis (x, y, z)
    scale: tuple = (0.9, 1.1)
    shear: float = 0.1                        # +- for xy, xz, yz
    flip_p: tuple = (0.5, 0.5, 0.5)           # reflection probability per axis
    generic: float = 0.0                      # +- entries of G - I
    disp: tuple = (8.0, 8.0, 8.0)             # +- voxels
    window_lo: tuple = (-1000.0, -150.0)      # a ~ U (spans PAPER.md:458-459 presets)
    window_hi: tuple = (230.0, 1500.0)        # b ~ U
    gamma: tuple = (0.7, 1.5)
    sigma: tuple = (0.0, 20.0)                # HU
    occ_dmax: float = 0.0                     # occlusion prism height bound (output z
                                              # voxels); 0 = no occlusion


TRAIN = AugmentRanges()
LARGE = AugmentRanges(rot_deg=(45.0, 45.0, 180.0), scale=(0.8, 1.2), shear=0.0,
                      flip_p=(0.0, 0.0, 0.0), disp=(0.0, 0.0, 0.0))
# TRAIN plus random occlusion: prism height delta ~ U[0, 48] output
# planes (the paper gives no value; 48 of the 160 planes of a 3 mm volume)
TRAIN_OCC = AugmentRanges(occ_dmax=48.0)


@dataclass(frozen=True)
class VolumeDraw:
    rot_rad: tuple
    scale: tuple
    shear: tuple
    flip: tuple
    generic: tuple
    disp: tuple
    window: tuple
    gamma: float
    sigma: float
    occ_z0: float = 0.0        # occlusion prism start z (output voxels)
    occ_height: float = -1.0   # delta; < 0 = no occlusion


def draw(ranges: AugmentRanges, global_index: int, master_seed: int = MASTER_SEED,
         out_mz: int | None = None) -> VolumeDraw:
    """Per-volume random draws, keyed by (master_seed, GLOBAL volume index).

    Occlusion (ranges.occ_dmax > 0; needs the output depth out_mz): delta ~ U[0, dmax]
    and z0 ~ U[-dmax, z_max] with z_max = out_mz - 1, so that every output plane has the
    same chance of being occluded.  Drawn after every other value,
    so the other draws do not depend on whether occlusion is on."""
    rng = np.random.default_rng([master_seed, global_index])
    rot = tuple(float(rng.uniform(-r, r)) * math.pi / 180.0 for r in ranges.rot_deg)
    scale = tuple(float(rng.uniform(*ranges.scale)) for _ in range(3))
    shear = tuple(float(rng.uniform(-ranges.shear, ranges.shear)) for _ in range(3))
    flip = tuple(int(rng.uniform() < p) for p in ranges.flip_p)
    generic = tuple(float(rng.uniform(-ranges.generic, ranges.generic)) for _ in range(9))
    disp = tuple(float(rng.uniform(-d, d)) for d in ranges.disp)
    a = float(rng.uniform(*ranges.window_lo))
    b = float(rng.uniform(*ranges.window_hi))
    while not a < b:  # a < b by rejection (SPEC.md augment3d decisions)
        b = float(rng.uniform(*ranges.window_hi))
    gamma = float(rng.uniform(*ranges.gamma))
    sigma = float(rng.uniform(*ranges.sigma))
    occ_z0, occ_h = 0.0, -1.0
    if ranges.occ_dmax > 0.0:
        if out_mz is None:
            raise ValueError("occlusion draws need the output depth out_mz")
        occ_h = float(rng.uniform(0.0, ranges.occ_dmax))
        occ_z0 = float(rng.uniform(-ranges.occ_dmax, out_mz - 1.0))
    return VolumeDraw(rot, scale, shear, flip, generic, disp, (a, b), gamma, sigma, occ_z0,
                      occ_h)


# The fixed C1 transform: Rz 25, Ry -7, Rx 10 degrees,
# scale (1.1, 0.9, 1.05), shear_xy 0.05, d = (1.5, -2.25, 0.75); noise only, sigma 10 HU.
C1_DRAW = VolumeDraw(rot_rad=(math.radians(10.0), math.radians(-7.0), math.radians(25.0)),
                     scale=(1.1, 0.9, 1.05), shear=(0.05, 0.0, 0.0), flip=(0, 0, 0),
                     generic=(0.0,) * 9, disp=(1.5, -2.25, 0.75), window=(0.0, 1.0),
                     gamma=1.0, sigma=10.0)

# BASELINE.json configs, in order (shape is numpy [nz, ny, nx]).
CONFIGS = {
    "c1": dict(shape=(32, 32, 32), batch=1, ranges=None, photometric="noise"),
    "c2": dict(shape=(160, 128, 128), batch=1, ranges=TRAIN, photometric="full"),
    "c3": dict(shape=(160, 128, 128), batch=16, ranges=TRAIN, photometric="full"),
    "c4": dict(shape=(512, 512, 512), batch=1, ranges=LARGE, photometric="full"),
    "c5": dict(shape=(160, 128, 128), batch=256, ranges=TRAIN, photometric="full"),
}


def random_volume(shape_zyx, seed, lo=-1024.0, hi=3071.0):
    """Uniform random HU volume + random labels 0..5 (stress inputs for parity tests)."""
    rng = np.random.default_rng([seed, 7])
    img = rng.uniform(lo, hi, size=shape_zyx).astype(np.float32)
    lbl = rng.integers(0, 6, size=shape_zyx, dtype=np.uint8)
    return img, lbl
