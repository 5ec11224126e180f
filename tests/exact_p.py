"""The pull-back coordinate p of DESIGN.md R4 in fp32, computed exactly in the test
(not by the oracle or the CUDA path): p_k = fma(A_k1, y, fma(A_k0, x, fma(A_k2, z, b_k)))
with every fma correctly rounded to fp32.  Scalar form by exact rational arithmetic;
grid form vectorised in float64 with a TwoSum exactness check per element (an inexact
double sum falls back to the rational form), so both give the same bits."""
from fractions import Fraction

import numpy as np


def fma32(a, x, c):
    """Correctly rounded fp32 fma(a, x, c) from exact rational arithmetic."""
    exact = Fraction(float(a)) * x + Fraction(float(c))
    f = np.float32(float(exact))
    best = f
    for cand in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        dc, db = abs(Fraction(float(cand)) - exact), abs(Fraction(float(best)) - exact)
        if dc < db or (dc == db and (int(cand.view(np.uint32)) & 1) == 0):
            best = cand
    return np.float32(best)


def p_fp32(A, x, y, z):
    """p (x, y, z components) of output voxel (x, y, z), fp32 R4 nesting."""
    return [float(fma32(A[k, 1], y, fma32(A[k, 0], x, fma32(A[k, 2], z, A[k, 3]))))
            for k in range(3)]


def _fma32_vec(a, x, c):
    """fp32 fma of an fp32 scalar a, an integer array x and an fp32 array c."""
    a64 = np.float64(np.float32(a))
    prod = a64 * x.astype(np.float64)          # exact: 24-bit x small-integer product
    c64 = c.astype(np.float64)
    s = prod + c64
    bb = s - prod                              # TwoSum error of prod + c64
    err = (prod - (s - bb)) + (c64 - bb)
    out = s.astype(np.float32)                 # one rounding of the exact sum
    bad = np.nonzero(err != 0.0)
    for i in zip(*bad):
        out[i] = fma32(a, int(x[i]), c[i])
    return out


def p_fp32_grid(A, out_shape_zyx):
    """p of every output voxel: float32 array [3, mz, my, mx] (x, y, z components)."""
    mz, my, mx = out_shape_zyx
    Z, Y, X = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    A = np.asarray(A, dtype=np.float32)
    out = np.empty((3, mz, my, mx), np.float32)
    for k in range(3):
        t = _fma32_vec(A[k, 2], Z, np.full(Z.shape, A[k, 3], np.float32))
        t = _fma32_vec(A[k, 0], X, t)
        out[k] = _fma32_vec(A[k, 1], Y, t)
    return out
