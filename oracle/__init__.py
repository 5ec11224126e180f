"""Oracle for the arXiv 1811.11226 Sec. IV augmentation path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It loads
``oracle/liboracle_warp3d.so`` (plain C, fp64, built by ``build.py``) with ctypes
and wraps it for numpy arrays.  It never imports ``paper_1811_11226_b200`` and
shares no code with it.

Parity status per function:
  philox4x32_10    pinned: Random123 known-answer vectors
  noise_normal     pinned: moments / lag correlation / closed-form uniforms
  compose_affine   pinned: Ac+b=c+d, hand-derived factor products
  warp_volume      pinned: identity, permutations, constant/ramp closed forms,
                   OOB fill, tent-kernel brute force, window worked value, gamma
  resample_sigma   pinned: PAPER.md:488-490 worked values (u=1 -> 2/3, u=3 -> 0)
  resample_dims    pinned: SPEC.md example (240,240,480) at 1.5 mm -> (120,120,240)
  smooth3d         pinned: constant invariance, sigma=0 identity, interior impulse
                   response = outer product of the normalised 1D kernels, linear ramp
                   preserved in the interior (symmetric kernel)
  resample         composition of the above with warp_volume (scale-only affine)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# W3D_ORACLE_LIB: the same C sources built with -fsanitize=address,undefined
# (build.py oracle-asan; tests/test_oracle_sanitized.py runs the pins against it)
LIB_PATH = os.environ.get("W3D_ORACLE_LIB") or os.path.join(_HERE, "liboracle_warp3d.so")

NOISE, WINDOW, CLAMP, GAMMA, OCCLUDE = 1, 2, 4, 8, 16
LINEAR, NEAREST = 0, 1


class Photometric(ctypes.Structure):
    _fields_ = [
        ("flags", ctypes.c_uint32),
        ("window_lo", ctypes.c_float),
        ("window_hi", ctypes.c_float),
        ("gamma", ctypes.c_float),
        ("noise_sigma", ctypes.c_float),
        ("_pad0", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("volume_id", ctypes.c_uint64),
        ("occ_z0", ctypes.c_float),
        ("occ_height", ctypes.c_float),
    ]


class Geom(ctypes.Structure):
    _fields_ = [
        ("rot_rad", ctypes.c_double * 3),
        ("scale", ctypes.c_double * 3),
        ("shear", ctypes.c_double * 3),
        ("flip", ctypes.c_int32 * 3),
        ("_pad0", ctypes.c_int32),
        ("generic", ctypes.c_double * 9),
        ("disp", ctypes.c_double * 3),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle library not built: {LIB_PATH} (run python build.py)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        I32 = ctypes.c_int32
        L.oracle_noise_uniforms.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P, I32, I32, I32,
                                            P, P]
        L.oracle_noise_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P, I32, I32, I32]
        L.oracle_noise_normal.restype = ctypes.c_double
        L.oracle_compose_affine.argtypes = [P, P, P, P, P]
        L.oracle_warp_volume.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_float,
                                         ctypes.c_uint8, P, P, P, P]
        L.oracle_warp_points.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_float,
                                         ctypes.c_uint8, P, P, P, ctypes.c_int64, P, P]
        L.oracle_noise_field.argtypes = [P, P, ctypes.c_float, ctypes.c_uint64, ctypes.c_uint64]
        D = ctypes.c_double
        L.oracle_resample_sigma.argtypes = [P, D, P]
        L.oracle_resample_dims.argtypes = [P, P, D, P]
        L.oracle_gauss_radius.argtypes = [D]
        L.oracle_gauss_radius.restype = ctypes.c_int32
        L.oracle_smooth3d.argtypes = [P, P, P, P]
        L.oracle_resample_affine.argtypes = [P, P, P, D, P]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dims(shape_zyx):
    """numpy shape (nz, ny, nx) -> int32[3] (nx, ny, nz)."""
    nz, ny, nx = shape_zyx
    return np.array([nx, ny, nz], dtype=np.int32)


def photometric(flags=0, window=(0.0, 1.0), gamma=1.0, sigma=0.0, seed=0, volume_id=0,
                occ_z0=0.0, occ_height=0.0):
    return Photometric(flags, window[0], window[1], gamma, sigma, 0, seed, volume_id,
                       occ_z0, occ_height)


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def noise_uniforms(seed, volume_id, shape_zyx, x, y, z):
    u1, s = ctypes.c_double(), ctypes.c_double()
    lib().oracle_noise_uniforms(seed, volume_id, _ptr(_dims(shape_zyx)), x, y, z,
                                ctypes.byref(u1), ctypes.byref(s))
    return u1.value, s.value


def noise_normal(seed, volume_id, shape_zyx, x, y, z):
    return lib().oracle_noise_normal(seed, volume_id, _ptr(_dims(shape_zyx)), x, y, z)


def noise_field(shape_zyx, sigma, seed, volume_id):
    out = np.empty(shape_zyx, dtype=np.float32)
    lib().oracle_noise_field(_ptr(out), _ptr(_dims(shape_zyx)), sigma, seed, volume_id)
    return out


def make_geom(rot=(0, 0, 0), scale=(1, 1, 1), shear=(0, 0, 0), flip=(0, 0, 0), generic=None,
              disp=(0, 0, 0)):
    g = Geom()
    g.rot_rad[:] = list(map(float, rot))
    g.scale[:] = list(map(float, scale))
    g.shear[:] = list(map(float, shear))
    g.flip[:] = [int(bool(f)) for f in flip]
    g.generic[:] = [0.0] * 9 if generic is None else list(map(float, np.ravel(generic)))
    g.disp[:] = list(map(float, disp))
    return g


def compose_affine(geom, in_shape_zyx, out_shape_zyx=None):
    """Returns (affine_double[3,4], affine_f32[3,4])."""
    out_shape_zyx = in_shape_zyx if out_shape_zyx is None else out_shape_zyx
    d = np.zeros(12, dtype=np.float64)
    f = np.zeros(12, dtype=np.float32)
    lib().oracle_compose_affine(ctypes.byref(geom), _ptr(_dims(in_shape_zyx)),
                                _ptr(_dims(out_shape_zyx)), _ptr(d), _ptr(f))
    return d.reshape(3, 4), f.reshape(3, 4)


def warp_volume(image, labels, affine, out_shape_zyx=None, interp=LINEAR, fill=0.0,
                label_fill=0, ph=None):
    """One volume.  image float32 [nz,ny,nx]; labels uint8 or None; affine [3,4] float32."""
    image = np.ascontiguousarray(image, dtype=np.float32)
    labels = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)
    out_shape_zyx = image.shape if out_shape_zyx is None else tuple(out_shape_zyx)
    A = np.ascontiguousarray(affine, dtype=np.float32).reshape(12)
    out = np.empty(out_shape_zyx, dtype=np.float32)
    out_l = None if labels is None else np.empty(out_shape_zyx, dtype=np.uint8)
    lib().oracle_warp_volume(_ptr(image), _ptr(labels), _ptr(_dims(image.shape)), _ptr(A),
                             interp, fill, label_fill,
                             None if ph is None else ctypes.byref(ph),
                             _ptr(out), _ptr(out_l), _ptr(_dims(out_shape_zyx)))
    return out, out_l


def warp_points(image, labels, affine, xyz, out_shape_zyx=None, interp=LINEAR, fill=0.0,
                label_fill=0, ph=None):
    """Oracle at selected output voxels; xyz int32 [n,3] as (x, y, z)."""
    image = np.ascontiguousarray(image, dtype=np.float32)
    labels = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)
    out_shape_zyx = image.shape if out_shape_zyx is None else tuple(out_shape_zyx)
    A = np.ascontiguousarray(affine, dtype=np.float32).reshape(12)
    xyz = np.ascontiguousarray(xyz, dtype=np.int32)
    n = xyz.shape[0]
    vals = np.empty(n, dtype=np.float32)
    lbls = None if labels is None else np.empty(n, dtype=np.uint8)
    lib().oracle_warp_points(_ptr(image), _ptr(labels), _ptr(_dims(image.shape)), _ptr(A),
                             interp, fill, label_fill,
                             None if ph is None else ctypes.byref(ph),
                             _ptr(_dims(out_shape_zyx)), _ptr(xyz), n, _ptr(vals), _ptr(lbls))
    return vals, lbls


# ----------------------------------------------------------------------------- resampling
def resample_sigma(spacing_mm, target_mm=3.0):
    """sigma_k = max(r/u_k - 1, 0)/3, as (x, y, z)."""
    u = np.ascontiguousarray(spacing_mm, dtype=np.float64)
    out = np.zeros(3, dtype=np.float64)
    lib().oracle_resample_sigma(_ptr(u), float(target_mm), _ptr(out))
    return out


def resample_dims(in_shape_zyx, spacing_mm, target_mm=3.0):
    """Output numpy shape (nz, ny, nx) of the resampling; spacing_mm is (x, y, z)."""
    u = np.ascontiguousarray(spacing_mm, dtype=np.float64)
    out = np.zeros(3, dtype=np.int32)
    lib().oracle_resample_dims(_ptr(_dims(in_shape_zyx)), _ptr(u), float(target_mm), _ptr(out))
    return (int(out[2]), int(out[1]), int(out[0]))


def gauss_radius(sigma):
    return int(lib().oracle_gauss_radius(float(sigma)))


def smooth3d(volume, sigma_xyz):
    """Direct 3D Gaussian smoothing (float64 result) of a float32 [nz,ny,nx] volume."""
    v = np.ascontiguousarray(volume, dtype=np.float32)
    s = np.ascontiguousarray(sigma_xyz, dtype=np.float64)
    out = np.empty(v.shape, dtype=np.float64)
    lib().oracle_smooth3d(_ptr(v), _ptr(_dims(v.shape)), _ptr(s), _ptr(out))
    return out


def resample_affine(in_shape_zyx, out_shape_zyx, spacing_mm, target_mm=3.0):
    u = np.ascontiguousarray(spacing_mm, dtype=np.float64)
    A = np.zeros(12, dtype=np.float32)
    lib().oracle_resample_affine(_ptr(_dims(in_shape_zyx)), _ptr(_dims(out_shape_zyx)), _ptr(u),
                                 float(target_mm), _ptr(A))
    return A.reshape(3, 4)


def resample(image, labels, spacing_mm, target_mm=3.0, fill=-1000.0, label_fill=0):
    """Smooth the image (never the labels), round the smoothed volume to float32,
    then trilinear (image) / nearest (labels) at spacing target_mm, centre-aligned."""
    out_shape = resample_dims(image.shape, spacing_mm, target_mm)
    sm = smooth3d(image, resample_sigma(spacing_mm, target_mm)).astype(np.float32)
    A = resample_affine(image.shape, out_shape, spacing_mm, target_mm)
    img, _ = warp_volume(sm, None, A, out_shape, LINEAR, fill, 0, None)
    lbl = None
    if labels is not None:
        _, lbl = warp_volume(image, labels, A, out_shape, LINEAR, fill, label_fill, None)
    return img, lbl
