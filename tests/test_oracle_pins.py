"""Pins for the oracle (CPU only): the oracle is checked against what the paper
and the mathematics fix, never against itself.  DESIGN.md "Oracle pins" maps
each test to the passage it follows (P1..P14 numbering from SURVEY.md Sec. 8.c).
"""
import itertools
import math
import os
from exact_p import p_fp32, p_fp32_grid

import numpy as np
import pytest

import oracle as O
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def _aff(M, b):
    A = np.zeros((3, 4), dtype=np.float32)
    A[:, :3] = M
    A[:, 3] = b
    return A


# ----------------------------------------------------------------------------- P8 Philox
def test_philox_known_answers():
    rows = _golden_rows("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for r in rows:
        v = [int(t, 16) for t in r]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert list(out) == v[6:10]


# ----------------------------------------------------------------------------- P9 noise
def test_noise_uniforms_exact_lattice():
    # u1 = odd multiple of 2^-24 in (0,1); s = multiple of 2^-23 in [-1, 1)
    shp = (5, 10, 7)
    for v in range(0, 350, 3):
        x, y, z = v % 7, (v // 7) % 10, v // 70
        u1, s = O.noise_uniforms(123, 4, shp, x, y, z)
        k = u1 * 2.0 ** 24
        assert 0 < u1 < 1 and k == int(k) and int(k) % 2 == 1
        assert -1.0 <= s < 1.0 and s * 2.0 ** 23 == int(s * 2.0 ** 23)
    # R10: voxels (x, 4g..4g+3, z) share one Philox block; rows (4g, 4g+1) and
    # (4g+2, 4g+3) share uniforms; neighbours along x use different blocks
    a = [O.noise_uniforms(9, 1, shp, 3, 4 + l, 2) for l in range(4)]
    assert a[0] == a[1] and a[2] == a[3] and a[0] != a[2]
    assert O.noise_uniforms(9, 1, shp, 4, 4, 2) != a[0]
    # the last (partial) y-group: my = 10 -> rows 8, 9 are lanes 0, 1 of their block
    b = [O.noise_uniforms(9, 1, shp, 0, 8 + l, 0) for l in range(2)]
    assert b[0] == b[1]


def test_noise_uniforms_come_from_philox_words():
    seed, vid = 0x1234_5678_9ABC, 0xDEAD_BEEF_01
    shp = (20, 30, 40)                    # (nz, ny, nx): mx = 40, my = 30 -> Gy = 8
    x, y, z = 17, 22, 13                  # y-group 5, lane 2
    q = x + 40 * (22 // 4 + 8 * 13)
    r = O.philox4x32_10([q & 0xFFFFFFFF, q >> 32, vid & 0xFFFFFFFF, vid >> 32],
                        [seed & 0xFFFFFFFF, seed >> 32])
    u1, s = O.noise_uniforms(seed, vid, shp, x, y, z)
    assert u1 == (2 * (int(r[2]) >> 9) + 1) / 2.0 ** 24
    assert s == 2 * ((int(r[3]) >> 8) / 2.0 ** 24) - 1
    # Box-Muller closed form: even row -> R cos(pi s), odd row -> R sin(pi s)
    R = math.sqrt(-2 * math.log(u1))
    assert O.noise_normal(seed, vid, shp, x, y, z) == pytest.approx(R * math.cos(math.pi * s),
                                                                    rel=1e-14, abs=1e-14)
    assert O.noise_normal(seed, vid, shp, x, y + 1, z) == pytest.approx(R * math.sin(math.pi * s),
                                                                        rel=1e-14, abs=1e-14)


def test_noise_statistics_1e6():
    # SPEC.md:381 / S:639: 1e6 samples at sigma=1: |mean|<0.004, |sd-1|<0.01, |lag-1 rho|<0.005
    f = O.noise_field((100, 100, 100), 1.0, 0x181111226, 3).astype(np.float64)
    n = f.ravel()
    assert abs(n.mean()) < 0.004
    assert abs(n.std() - 1.0) < 0.01
    # lag-1 correlation along every axis (x: different blocks; y: cos/sin partners
    # and block-mates; z: different blocks)
    for ax in range(3):
        a = np.moveaxis(f, ax, -1)
        rho = np.corrcoef(a[..., :-1].ravel(), a[..., 1:].ravel())[0, 1]
        assert abs(rho) < 0.005, (ax, rho)
    # cos/sin partners (rows 2k, 2k+1 of one Box-Muller pair) are uncorrelated
    assert abs(np.corrcoef(f[:, 0::2, :].ravel(), f[:, 1::2, :].ravel())[0, 1]) < 0.005
    # whole-distribution check against the standard normal CDF (Kolmogorov-Smirnov)
    from scipy import stats
    assert stats.kstest(n[::7], "norm").pvalue > 1e-3
    # tails: P(|n| > 3) = 0.0027
    assert abs(np.mean(np.abs(n) > 3.0) - 0.0027) < 0.0005


def test_noise_streams_differ_by_volume_and_seed():
    a = O.noise_field((8, 8, 8), 1.0, 5, 0)
    b = O.noise_field((8, 8, 8), 1.0, 5, 1)
    c = O.noise_field((8, 8, 8), 1.0, 6, 0)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
    assert abs(np.corrcoef(a.ravel(), b.ravel())[0, 1]) < 0.2
    # determinism
    assert np.array_equal(a, O.noise_field((8, 8, 8), 1.0, 5, 0))
    # sigma = 0 -> zeros
    assert not O.noise_field((4, 4, 4), 0.0, 5, 0).any()


# ----------------------------------------------------------------------------- P1 compose
def test_compose_center_guarantee():
    # b = c + d - A c guarantees A c + b = c + d.
    for idx in range(2000):
        d = synth.draw(synth.TRAIN if idx % 2 else synth.LARGE, idx)
        g = O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp)
        in_shape, out_shape = (160, 128, 128), ((160, 120, 120) if idx % 3 == 0 else (160, 128, 128))
        Ad, _ = O.compose_affine(g, in_shape, out_shape)
        c_in = (np.array(in_shape[::-1], dtype=np.float64) - 1) / 2
        c_out = (np.array(out_shape[::-1], dtype=np.float64) - 1) / 2
        err = Ad[:, :3] @ c_out + Ad[:, 3] - (c_in + np.array(d.disp))
        assert np.max(np.abs(err)) < 1e-9


def test_compose_factor_matrices_hand_derived():
    s2 = math.pi / 2
    # Rz(90) maps e_x to e_y (right-handed, R_z = [[c,-s,0],[s,c,0],[0,0,1]])
    Ad, _ = O.compose_affine(O.make_geom(rot=(0, 0, s2)), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    # Rx(90): e_y -> e_z ; Ry(90): e_z -> e_x
    Ad, _ = O.compose_affine(O.make_geom(rot=(s2, 0, 0)), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[1, 0, 0], [0, 0, -1], [0, 1, 0]], atol=1e-15)
    Ad, _ = O.compose_affine(O.make_geom(rot=(0, s2, 0)), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[0, 0, 1], [0, 1, 0], [-1, 0, 0]], atol=1e-15)
    # order F Rz Ry (R16): F=diag(-1,1,1), Rz(90), Ry(90) ->
    # F Rz Ry = [[0,1,0],[0,0,1],[-1,0,0]] (Rz Ry F or Ry Rz would differ)
    Ad, _ = O.compose_affine(O.make_geom(rot=(0, s2, s2), flip=(1, 0, 0)), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[0, 1, 0], [0, 0, 1], [-1, 0, 0]], atol=1e-15)
    # Sh S: shear_xy h applied after scale: (Sh S)[0][1] = h * s_y, not h * s_x
    Ad, _ = O.compose_affine(O.make_geom(scale=(2, 3, 5), shear=(0.25, 0.5, 0.125)), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[2, 0.75, 2.5], [0, 3, 0.625], [0, 0, 5]], atol=1e-15)
    # S G: generic acts first
    G = np.zeros((3, 3)); G[0, 1] = 0.5
    Ad, _ = O.compose_affine(O.make_geom(scale=(2, 1, 1), generic=G), (9, 9, 9))
    assert np.allclose(Ad[:, :3], [[2, 1, 0], [0, 1, 0], [0, 0, 1]], atol=1e-15)
    # identity with A = I, d = (5,0,0) -> b = (5,0,0)
    Ad, Af = O.compose_affine(O.make_geom(disp=(5, 0, 0)), (9, 9, 9))
    assert np.array_equal(Ad, _aff(np.eye(3), (5, 0, 0)).astype(np.float64))
    # flip x with center (n-1)/2 maps x -> n-1-x (R3): b_x = n - 1
    Ad, _ = O.compose_affine(O.make_geom(flip=(1, 0, 0)), (4, 6, 10))
    assert np.array_equal(Ad, _aff(np.diag([-1.0, 1, 1]), (9, 0, 0)).astype(np.float64))


def test_compose_rotation_orthonormal_and_det():
    for idx in range(200):
        d = synth.draw(synth.LARGE, idx)
        g = O.make_geom(rot=d.rot_rad)
        Ad, _ = O.compose_affine(g, (8, 8, 8))
        R = Ad[:, :3]
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-13)
        assert abs(np.linalg.det(R) - 1) < 1e-13
        d = synth.draw(synth.TRAIN, idx)
        g = O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp)
        Ad, _ = O.compose_affine(g, (8, 8, 8))
        sign = (-1) ** sum(d.flip)
        assert abs(np.linalg.det(Ad[:, :3]) - sign * np.prod(d.scale)) < 1e-12


# ----------------------------------------------------------------------------- P2/P3/P5 exact
def test_identity_is_exact():
    img, lbl = synth.random_volume((7, 9, 11), 1)
    out, out_l = O.warp_volume(img, lbl, _aff(np.eye(3), (0, 0, 0)))
    assert np.array_equal(out, img) and np.array_equal(out_l, lbl)
    out, _ = O.warp_volume(img, None, _aff(np.eye(3), (0, 0, 0)), interp=O.NEAREST)
    assert np.array_equal(out, img)


@pytest.mark.parametrize("shift", [(1, 0, 0), (0, -2, 0), (0, 0, 3), (2, -1, 1)])
def test_integer_translation_is_shift_with_fill(shift):
    img, lbl = synth.random_volume((6, 7, 8), 2)
    fill, lfill = -1000.0, 9
    out, out_l = O.warp_volume(img, lbl, _aff(np.eye(3), shift), fill=fill, label_fill=lfill)
    nz, ny, nx = img.shape
    for z, y, x in itertools.product(range(nz), range(ny), range(nx)):
        sx, sy, sz = x + shift[0], y + shift[1], z + shift[2]
        inside = 0 <= sx < nx and 0 <= sy < ny and 0 <= sz < nz
        assert out[z, y, x] == (img[sz, sy, sx] if inside else np.float32(fill))
        assert out_l[z, y, x] == (lbl[sz, sy, sx] if inside else lfill)


def test_flips_and_90_degree_rotations_are_permutations():
    img, lbl = synth.random_volume((6, 6, 6), 3)
    n = 6
    # flip x: p = (n-1-x, y, z)
    out, out_l = O.warp_volume(img, lbl, _aff(np.diag([-1.0, 1, 1]), (n - 1, 0, 0)))
    assert np.array_equal(out, img[:, :, ::-1]) and np.array_equal(out_l, lbl[:, :, ::-1])
    # flip z
    out, out_l = O.warp_volume(img, lbl, _aff(np.diag([1.0, 1, -1]), (0, 0, n - 1)))
    assert np.array_equal(out, img[::-1]) and np.array_equal(out_l, lbl[::-1])
    # 90 deg about z: p = (y, n-1-x, z)  ->  out[z,y,x] = img[z, n-1-x, y]
    M = np.array([[0, 1, 0], [-1, 0, 0], [0, 0, 1]], dtype=np.float32)
    out, out_l = O.warp_volume(img, lbl, _aff(M, (0, n - 1, 0)))
    ref = np.empty_like(img); refl = np.empty_like(lbl)
    for z, y, x in itertools.product(range(n), repeat=3):
        ref[z, y, x] = img[z, n - 1 - x, y]
        refl[z, y, x] = lbl[z, n - 1 - x, y]
    assert np.array_equal(out, ref) and np.array_equal(out_l, refl)
    # and equals numpy's rot90 in the (y, x) plane
    assert np.array_equal(out, np.rot90(img, k=-1, axes=(1, 2)))
    # 90 deg about x: p = (x, z, n-1-y)
    M = np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0]], dtype=np.float32)
    out, _ = O.warp_volume(img, lbl, _aff(M, (0, 0, n - 1)))
    for z, y, x in itertools.product(range(n), repeat=3):
        assert out[z, y, x] == img[n - 1 - y, z, x]


# ----------------------------------------------------------------------------- P4 closed forms
def test_constant_volume_stays_constant():
    img = np.full((9, 10, 11), 37.25, dtype=np.float32)
    for idx in range(20):
        d = synth.draw(synth.LARGE, idx)
        _, Af = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear), img.shape)
        out, _ = O.warp_volume(img, None, Af, fill=37.25)   # fill == constant -> everywhere
        assert np.all(out == np.float32(37.25))


def test_linear_ramp_closed_form():
    # trilinear interpolation reproduces affine functions exactly (interior samples)
    nz, ny, nx = 12, 13, 14
    al, be, ga, de = 0.5, -0.25, 2.0, 3.0  # dyadic coefficients
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    img = (al * x + be * y + ga * z + de).astype(np.float32)
    rng = np.random.default_rng(5)
    M = np.array([[0.9, 0.2, -0.1], [-0.15, 1.05, 0.1], [0.05, -0.1, 0.95]], dtype=np.float32)
    A = _aff(M, (0.7, 0.3, 0.45))
    xyz = rng.integers(0, [nx, ny, nz], size=(3000, 3)).astype(np.int32)
    vals, _ = O.warp_points(img, None, A, xyz)
    checked = 0
    for (X, Y, Z), v in zip(xyz, vals):
        p = _p_fp32(A, int(X), int(Y), int(Z))
        if all(0 <= p[k] <= n - 1 for k, n in enumerate((nx, ny, nz))):
            ref = al * p[0] + be * p[1] + ga * p[2] + de
            assert abs(float(v) - ref) <= 2.0 ** -23 * abs(ref)
            checked += 1
    assert checked > 1000


# ----------------------------------------------------------------------------- P6 OOB
def test_fully_out_of_bounds_is_fill():
    img, lbl = synth.random_volume((5, 6, 7), 4)
    for b in [(-1.0, 0, 0), (7.0, 0, 0), (0, -1.0, 0), (0, 6.0, 0), (0, 0, -3.5), (0, 0, 100)]:
        A = _aff(np.zeros((3, 3)), b)  # every output voxel maps to p = b
        out, out_l = O.warp_volume(img, lbl, A, fill=-1000.0, label_fill=7)
        assert np.all(out == np.float32(-1000.0))
        assert np.all(out_l == 7)
    # p in (-1, 0): blend of fill and voxel 0 (border-fill semantics, R6)
    A = _aff(np.zeros((3, 3)), (-0.25, 0, 0))
    out, out_l = O.warp_volume(img, lbl, A, fill=-1000.0, label_fill=7)
    assert np.allclose(out, np.float32(0.25 * -1000.0 + 0.75 * img[0, 0, 0]), rtol=1e-6)
    assert np.all(out_l == lbl[0, 0, 0])  # nearest of -0.25 is 0


# ----------------------------------------------------------------------------- P7 brute force
def _tent_brute(img, fill, p):
    nz, ny, nx = img.shape
    jz, jy, jx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    w = (np.maximum(0.0, 1 - np.abs(p[0] - jx)) * np.maximum(0.0, 1 - np.abs(p[1] - jy)) *
         np.maximum(0.0, 1 - np.abs(p[2] - jz)))
    return fill + np.sum((img.astype(np.float64) - fill) * w)


def _nearest_brute(n, p):
    """argmin over the integer lattice of (p - j)^2 per axis, ties -> larger index."""
    out = []
    for k in range(3):
        cands = range(int(math.floor(p[k])) - 3, int(math.floor(p[k])) + 4)
        best = min(cands, key=lambda j: ((p[k] - j) ** 2, -j))
        out.append(best)
    return out


def _p_fp32(A, x, y, z):
    return p_fp32(A, x, y, z)


def test_brute_force_8cubed():
    img, lbl = synth.random_volume((8, 8, 8), 6)
    fill, lfill = -1000.0, 6
    mats = []
    for idx in range(6):
        d = synth.draw(synth.LARGE, idx)
        mats.append(O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip,
                                                  disp=(1.5 * idx - 4, 0.5, -1)), img.shape)[1])
    mats.append(_aff(np.diag([2.0, 2.0, 0.5]), (-3.5, -3.5, 1.75)))   # scale-2 half ties
    mats.append(_aff(np.diag([-1.0, 2.0, 1.0]), (7.5, -4.5, 0.5)))    # flip + ties
    for A in mats:
        out, out_l = O.warp_volume(img, lbl, A, fill=fill, label_fill=lfill)
        for z, y, x in itertools.product(range(8), repeat=3):
            p = _p_fp32(A, x, y, z)
            ref = _tent_brute(img, fill, p)
            assert abs(float(out[z, y, x]) - ref) <= 2.0 ** -23 * max(abs(ref), 1.0), (p, ref)
            r = _nearest_brute(8, p)
            inside = all(0 <= r[k] < 8 for k in range(3))
            assert out_l[z, y, x] == (lbl[r[2], r[1], r[0]] if inside else lfill), p


def test_nearest_image_matches_nearest_label():
    img, lbl = synth.random_volume((8, 9, 10), 8)
    d = synth.draw(synth.TRAIN, 3)
    _, Af = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, disp=d.disp),
                             img.shape)
    out, _ = O.warp_volume(lbl.astype(np.float32), None, Af, interp=O.NEAREST, fill=99.0)
    _, out_l = O.warp_volume(img, lbl, Af, label_fill=99)
    assert np.array_equal(out.astype(np.uint8), out_l)


# ----------------------------------------------------------------------------- P10/P11/P14 window+gamma
def test_window_worked_values():
    for a, b, v, w in _golden_rows("window_worked_value.txt"):
        a, b, v, w = map(float, (a, b, v, w))
        img = np.full((2, 2, 4), v, dtype=np.float32)
        ph = O.photometric(O.WINDOW | O.CLAMP, window=(a, b))
        out, _ = O.warp_volume(img, None, _aff(np.eye(3), (0, 0, 0)), ph=ph)
        assert np.all(out == np.float32(w))


def test_window_range_and_monotone():
    v = np.linspace(-1500, 2500, 4 * 4 * 64, dtype=np.float32).reshape(4, 4, 64)
    ph = O.photometric(O.WINDOW | O.CLAMP, window=(-150.0, 230.0))
    out, _ = O.warp_volume(v, None, _aff(np.eye(3), (0, 0, 0)), ph=ph)
    o = out.ravel()
    assert o.min() >= 0 and o.max() <= 1 and np.all(np.diff(o) >= 0)
    # window without clamp is the plain intensity affine
    ph = O.photometric(O.WINDOW, window=(-150.0, 230.0))
    out, _ = O.warp_volume(v, None, _aff(np.eye(3), (0, 0, 0)), ph=ph)
    assert np.allclose(out.ravel(), (v.ravel().astype(np.float64) + 150) / 380, rtol=1e-7)


def test_gamma():
    img = np.full((2, 2, 4), 40.0, dtype=np.float32)  # w = 0.5 under (-150, 230)
    I = _aff(np.eye(3), (0, 0, 0))
    base = O.photometric(O.WINDOW | O.CLAMP, window=(-150.0, 230.0))
    g1 = O.photometric(O.WINDOW | O.CLAMP | O.GAMMA, window=(-150.0, 230.0), gamma=1.0)
    assert np.array_equal(O.warp_volume(img, None, I, ph=base)[0],
                          O.warp_volume(img, None, I, ph=g1)[0])
    g2 = O.photometric(O.WINDOW | O.CLAMP | O.GAMMA, window=(-150.0, 230.0), gamma=2.0)
    assert np.all(O.warp_volume(img, None, I, ph=g2)[0] == np.float32(0.25))
    g3 = O.photometric(O.WINDOW | O.CLAMP | O.GAMMA, window=(-150.0, 230.0), gamma=0.5)
    assert np.all(O.warp_volume(img, None, I, ph=g3)[0] == np.float32(math.sqrt(0.5)))
    # fixed points 0 and 1
    for v, w in ((-500.0, 0.0), (900.0, 1.0)):
        im = np.full((2, 2, 4), v, dtype=np.float32)
        for gam in (0.7, 1.5):
            g = O.photometric(O.WINDOW | O.CLAMP | O.GAMMA, window=(-150.0, 230.0), gamma=gam)
            assert np.all(O.warp_volume(im, None, I, ph=g)[0] == np.float32(w))


# ----------------------------------------------------------------------------- P12/P13 invariance
def test_labels_photometric_invariant_and_determinism():
    img, lbl = synth.phantom((20, 24, 28))
    d = synth.draw(synth.TRAIN, 11)
    _, Af = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, disp=d.disp),
                             img.shape)
    outs = []
    for sig, win, gam in ((0.0, (-150.0, 230.0), 1.0), (20.0, (-1000.0, 1500.0), 0.7),
                          (5.0, (-500.0, 300.0), 1.5)):
        ph = O.photometric(O.NOISE | O.WINDOW | O.CLAMP | O.GAMMA, window=win, gamma=gam,
                           sigma=sig, seed=1, volume_id=2)
        outs.append(O.warp_volume(img, lbl, Af, fill=-1000.0, ph=ph))
    for o in outs[1:]:
        assert np.array_equal(o[1], outs[0][1])
    ph = O.photometric(O.NOISE | O.WINDOW | O.CLAMP | O.GAMMA, window=(-500.0, 300.0),
                       gamma=1.5, sigma=5.0, seed=1, volume_id=2)
    again = O.warp_volume(img, lbl, Af, fill=-1000.0, ph=ph)
    assert np.array_equal(again[0], outs[2][0]) and np.array_equal(again[1], outs[2][1])


def test_noise_is_added_everywhere_including_fill():
    # R9: I_noise = I + n for every voxel; with a fully-OOB map the
    # output is fill + sigma * n(v)
    img = np.zeros((4, 4, 8), dtype=np.float32)
    ph = O.photometric(O.NOISE, sigma=10.0, seed=77, volume_id=5)
    out, _ = O.warp_volume(img, None, _aff(np.zeros((3, 3)), (-5, -5, -5)), fill=-1000.0, ph=ph)
    field = O.noise_field(img.shape, 10.0, 77, 5)
    assert np.allclose(out, np.float32(-1000.0) + field, atol=1e-4)


# ----------------------------------------------------------------------------- occlusion (NEXT-1)
def test_occlusion_full_height_is_zero_and_input_independent():
    img, lbl = synth.random_volume((6, 5, 8), 9)
    ph = O.photometric(O.OCCLUDE | O.NOISE | O.WINDOW | O.CLAMP, window=(-150.0, 230.0),
                       sigma=10.0, seed=1, volume_id=0, occ_z0=-2.0, occ_height=8.0)
    out, out_l = O.warp_volume(img, lbl, _aff(np.eye(3), (0, 0, 0)), ph=ph)
    assert np.all(out == 0.0)  # SPEC.md:371 (delta = nz -> all zeros)
    assert np.array_equal(out_l, lbl)  # labels untouched
    ph = O.photometric(O.OCCLUDE | O.WINDOW | O.CLAMP, window=(-150.0, 230.0),
                       occ_z0=1.5, occ_height=2.0)  # occludes z = 2, 3
    out, _ = O.warp_volume(img, lbl, _aff(np.eye(3), (0, 0, 0)), ph=ph)
    assert np.all(out[2:4] == 0.0)
    img2 = img + 500
    out2, _ = O.warp_volume(img2, lbl, _aff(np.eye(3), (0, 0, 0)), ph=ph)
    assert np.all(out2[2:4] == 0.0)
    assert np.all(out[[0, 1, 4, 5]] == np.clip((img[[0, 1, 4, 5]].astype(np.float64) + 150) / 380, 0, 1).astype(np.float32))


def test_exact_p_grid_equals_rational_fma():
    """The vectorised exact-p helper (used to count footprints in the GPU tests) gives
    the bits of the rational fp32 FMA chain (R4) at every voxel of a small grid."""
    for rname, idx in (("TRAIN", 1), ("LARGE", 2)):
        d = synth.draw(getattr(synth, rname), idx)
        A = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic,
                                         d.disp), (9, 7, 11), (5, 6, 7))[1]
        g = p_fp32_grid(A, (5, 6, 7))
        for z, y, x in itertools.product(range(5), range(6), range(7)):
            assert [float(v) for v in g[:, z, y, x]] == p_fp32(A, x, y, z)


def test_occlusion_draw_is_uniform_over_planes():
    """The occlusion draw (delta ~ U[0, dmax], z0 ~ U[-dmax, z_max])
    gives every output plane the same chance E[delta] / (z_max + dmax) of being
    occluded; the other draws do not change when occlusion is switched on."""
    mz, n = 64, 6000
    dmax = synth.TRAIN_OCC.occ_dmax
    hits = np.zeros(mz)
    z = np.arange(mz)
    for v in range(n):
        d = synth.draw(synth.TRAIN_OCC, v, out_mz=mz)
        assert 0.0 <= d.occ_height <= dmax and -dmax <= d.occ_z0 <= mz - 1
        hits += (z >= d.occ_z0) & (z <= d.occ_z0 + d.occ_height)
        if v < 20:
            base = synth.draw(synth.TRAIN, v)
            assert base.rot_rad == d.rot_rad and base.sigma == d.sigma and base.window == d.window
    p = (dmax / 2.0) / (mz - 1 + dmax)
    sd = np.sqrt(p * (1 - p) / n)
    assert np.all(np.abs(hits / n - p) < 5 * sd), (hits.min() / n, hits.max() / n, p)
