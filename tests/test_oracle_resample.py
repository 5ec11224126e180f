"""Pins of the resampling oracle: values the
paper and SPEC.md state, closed forms and invariants of the Gaussian lowpass, all
evaluated through code paths independent of oracle/oracle_resample.c."""
import math

import numpy as np
import pytest

import oracle as O


# ----------------------------------------------------------------------------- sigma
@pytest.mark.parametrize("u,expect", [
    (1.0, 2.0 / 3.0),    # SPEC.md:109 "u=(1,1,1), r=3 -> sigma=(2/3,2/3,2/3)"
    (3.0, 0.0),          # SPEC.md:110 "u=(3,3,3), r=3 -> sigma=(0,0,0)"
    (0.5, 5.0 / 3.0),    # (3/0.5 - 1)/3
    (1.5, 1.0 / 3.0),
    (5.0, 0.0),          # coarser than the target: max(., 0)
])
def test_sigma_worked_values(u, expect):
    s = O.resample_sigma((u, u, u), 3.0)
    assert np.allclose(s, expect, rtol=0, atol=1e-15)


def test_sigma_per_axis_order():
    s = O.resample_sigma((1.0, 3.0, 0.5), 3.0)
    assert np.allclose(s, (2.0 / 3.0, 0.0, 5.0 / 3.0), atol=1e-15)


# ----------------------------------------------------------------------------- dims
def test_dims_spec_example():
    # SPEC.md:111 "dims (240,240,480), u=(1.5,1.5,1.5), r=3 -> dims (120,120,240)"
    # (x, y, z) = (240, 240, 480) -> numpy shape (480, 240, 240)
    assert O.resample_dims((480, 240, 240), (1.5, 1.5, 1.5), 3.0) == (240, 120, 120)


def test_dims_degenerate_and_rounding():
    # a dim that would round to 0 is clamped to 1 (SPEC.md:108 errors clause)
    assert O.resample_dims((1, 1, 1), (0.1, 0.1, 0.1), 3.0) == (1, 1, 1)
    # 512 voxels of 0.7 mm -> 119.47 -> 119; 5 mm slices upsampled: 60 -> 100
    assert O.resample_dims((60, 512, 512), (0.7, 0.7, 5.0), 3.0) == (100, 119, 119)
    # exact half (n u / r = 10.5): rounds half up
    assert O.resample_dims((7, 7, 7), (4.5, 4.5, 4.5), 3.0) == (11, 11, 11)


# ----------------------------------------------------------------------------- smoothing
def _kernel(sigma):
    """Closed form of the normalised 1D factor of g(x) ~ exp(-x^2/sigma^2)."""
    if sigma <= 0:
        return np.ones(1)
    R = math.ceil(3 * sigma)
    i = np.arange(-R, R + 1, dtype=np.float64)
    w = np.exp(-(i * i) / (sigma * sigma))
    return w / w.sum()


def test_sigma_zero_is_identity():
    rng = np.random.default_rng(0)
    v = rng.normal(size=(6, 7, 9)).astype(np.float32)
    assert np.array_equal(O.smooth3d(v, (0.0, 0.0, 0.0)), v.astype(np.float64))


def test_constant_is_invariant():
    # SPEC.md:640 (10): "constant volumes invariant" (edge replication at the borders)
    v = np.full((11, 9, 10), -1000.0, np.float32)
    out = O.smooth3d(v, (2.0 / 3.0, 1.3, 0.4))
    assert np.max(np.abs(out + 1000.0)) < 1e-10


def test_impulse_response_is_the_product_kernel():
    sig = (0.8, 2.0 / 3.0, 1.4)
    n = 21
    v = np.zeros((n, n, n), np.float32)
    v[n // 2, n // 2, n // 2] = 1.0
    out = O.smooth3d(v, sig)
    kx, ky, kz = (_kernel(s) for s in sig)
    expect = np.zeros_like(out)
    c = n // 2
    Rx, Ry, Rz = len(kx) // 2, len(ky) // 2, len(kz) // 2
    expect[c - Rz:c + Rz + 1, c - Ry:c + Ry + 1, c - Rx:c + Rx + 1] = \
        kz[:, None, None] * ky[None, :, None] * kx[None, None, :]
    assert np.max(np.abs(out - expect)) < 1e-15


def test_kernel_variance_is_sigma_squared_over_two():
    """PAPER.md:487 writes exp(-x^2/sigma^2) (variance sigma^2/2, not sigma^2): the
    impulse response's second moment along each axis pins that form."""
    n = 41
    v = np.zeros((n, n, n), np.float32)
    v[n // 2, n // 2, n // 2] = 1.0
    sig = (2.0, 3.0, 2.5)
    out = O.smooth3d(v, sig)
    i = np.arange(n) - n // 2
    for axis, s in zip((2, 1, 0), sig):
        other = tuple(a for a in range(3) if a != axis)
        m = out.sum(axis=other)
        var = float(np.sum(m * i * i))
        assert abs(var - s * s / 2.0) / (s * s / 2.0) < 0.01, (axis, var)


def test_linear_ramp_preserved_in_the_interior():
    nz, ny, nx = 18, 17, 19
    Z, Y, X = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    v = (0.75 * X - 1.25 * Y + 0.5 * Z + 3.0).astype(np.float32)
    sig = (0.9, 2.0 / 3.0, 1.2)
    out = O.smooth3d(v, sig)
    R = [O.gauss_radius(s) for s in sig]
    inner = (slice(R[2], nz - R[2]), slice(R[1], ny - R[1]), slice(R[0], nx - R[0]))
    assert np.max(np.abs(out[inner] - v[inner])) < 1e-12


def test_one_axis_equals_row_convolution_with_edge_padding():
    rng = np.random.default_rng(3)
    v = rng.normal(size=(4, 5, 23)).astype(np.float32)
    k = _kernel(1.1)
    R = len(k) // 2
    out = O.smooth3d(v, (1.1, 0.0, 0.0))
    padded = np.pad(v.astype(np.float64), ((0, 0), (0, 0), (R, R)), mode="edge")
    expect = np.zeros_like(out)
    for t in range(2 * R + 1):
        expect += k[t] * padded[:, :, t:t + v.shape[2]]
    assert np.max(np.abs(out - expect)) < 1e-12


# ----------------------------------------------------------------------------- resample
def test_resample_affine_maps_centre_to_centre():
    A = O.resample_affine((480, 240, 240), (240, 120, 120), (1.5, 1.5, 1.5), 3.0).astype(np.float64)
    c_out = np.array([(120 - 1) / 2, (120 - 1) / 2, (240 - 1) / 2])
    c_in = np.array([(240 - 1) / 2, (240 - 1) / 2, (480 - 1) / 2])
    assert np.allclose(A[:, :3], 2.0 * np.eye(3))
    assert np.max(np.abs(A[:, :3] @ c_out + A[:, 3] - c_in)) < 1e-4


def test_resample_at_target_spacing_is_identity():
    rng = np.random.default_rng(5)
    img = rng.normal(size=(6, 8, 10)).astype(np.float32) * 100
    lbl = rng.integers(0, 6, size=img.shape, dtype=np.uint8)
    out, out_l = O.resample(img, lbl, (3.0, 3.0, 3.0), 3.0)
    assert np.array_equal(out, img) and np.array_equal(out_l, lbl)


def test_resample_downsample_by_two_matches_smoothed_samples():
    """u = 1.5 mm -> 3 mm: centre-aligned, output voxel j samples input 2j + 0.5 per axis
    (c_in = (n-1)/2, c_out = (n/2-1)/2): the trilinear average of the smoothed volume's
    2x2x2 block, labels the nearest voxel (round half up: 2j + 1)."""
    rng = np.random.default_rng(7)
    img = rng.normal(size=(8, 10, 12)).astype(np.float32)
    lbl = rng.integers(0, 6, size=img.shape, dtype=np.uint8)
    out, out_l = O.resample(img, lbl, (1.5, 1.5, 1.5), 3.0, fill=0.0)
    sm = O.smooth3d(img, O.resample_sigma((1.5, 1.5, 1.5), 3.0)).astype(np.float32)
    blocks = sm.astype(np.float64).reshape(4, 2, 5, 2, 6, 2).mean(axis=(1, 3, 5))
    assert out.shape == (4, 5, 6)
    assert np.max(np.abs(out - blocks)) < 1e-5
    assert np.array_equal(out_l, lbl[1::2, 1::2, 1::2])
