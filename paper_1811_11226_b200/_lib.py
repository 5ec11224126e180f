"""ctypes view of include/warp3d.h (libwarp3d.so, built in-tree by build.py).

Argument marshalling only: every step of the augmentation runs in the CUDA
library.  There is no fallback: if the shared library is missing, loading
raises, and on a machine without a GPU the compute entry points return
W3D_ERR_CUDA.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwarp3d.so")

W3D_OK, W3D_ERR_INVALID_ARG, W3D_ERR_UNSUPPORTED, W3D_ERR_CUDA, W3D_ERR_INTERNAL = range(5)
STATUS_NAMES = {0: "W3D_OK", 1: "W3D_ERR_INVALID_ARG", 2: "W3D_ERR_UNSUPPORTED",
                3: "W3D_ERR_CUDA", 4: "W3D_ERR_INTERNAL"}
INTERP_LINEAR, INTERP_NEAREST = 0, 1
KERNEL_AUTO, KERNEL_GATHER, KERNEL_STAGED = range(3)
PH_NOISE, PH_WINDOW, PH_CLAMP, PH_GAMMA, PH_OCCLUDE = 1, 2, 4, 8, 16

# every symbol include/warp3d.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "warp3d_affine", "warp3d_affine_batched", "warp3d_affine_batched_ex",
    "warp3d_compose_affine", "warp3d_noise", "warp3d_philox4x32_10",
    "warp3d_footprint_batched", "warp3d_launch_count", "warp3d_last_error",
    "warp3d_abi_version", "warp3d_tile_stats", "warp3d_pipeline_create", "warp3d_pipeline_run",
    "warp3d_pipeline_destroy", "warp3d_resample_sigma", "warp3d_resample_dims",
    "warp3d_resample_affine", "warp3d_smooth3d", "warp3d_resample",
    "warp3d_affine_batched_i16", "warp3d_affine_batched_i16_ex", "warp3d_affine_batched_v",
    "warp3d_pipeline_create_ex", "warp3d_pipeline_vols_per_job", "warp3d_compose_params_batched",
    "warp3d_params_from_arrays",
)


class Dims(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32)]


class Photometric(ctypes.Structure):
    _fields_ = [
        ("flags", ctypes.c_uint32),
        ("window_lo", ctypes.c_float),
        ("window_hi", ctypes.c_float),
        ("gamma", ctypes.c_float),
        ("noise_sigma", ctypes.c_float),
        ("_reserved", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("volume_id", ctypes.c_uint64),
        ("occ_z0", ctypes.c_float),
        ("occ_height", ctypes.c_float),
    ]


class VolumeParams(ctypes.Structure):
    _fields_ = [("affine", ctypes.c_float * 12), ("ph", Photometric)]


class Geom(ctypes.Structure):
    _fields_ = [
        ("rot_rad", ctypes.c_double * 3),
        ("scale", ctypes.c_double * 3),
        ("shear", ctypes.c_double * 3),
        ("flip", ctypes.c_int32 * 3),
        ("_reserved", ctypes.c_int32),
        ("generic", ctypes.c_double * 9),
        ("disp", ctypes.c_double * 3),
    ]


assert ctypes.sizeof(Photometric) == 48 and ctypes.sizeof(VolumeParams) == 96


class Warp3DError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA library not built: {LIB_PATH} (run python build.py)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, F = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                           ctypes.c_float)
    L.warp3d_affine.argtypes = [P, Dims, P, I32, F, P, P, Dims, P]
    L.warp3d_affine_batched.argtypes = [I32, P, P, Dims, P, I32, F, ctypes.c_uint8, P, P, Dims, P]
    L.warp3d_affine_batched_ex.argtypes = [I32, P, P, Dims, P, I32, F, ctypes.c_uint8, P, P, Dims,
                                           I32, P]
    L.warp3d_compose_affine.argtypes = [P, Dims, Dims, P]
    L.warp3d_compose_params_batched.argtypes = [I32, P, P, Dims, Dims, P]
    L.warp3d_params_from_arrays.argtypes = [I32, Dims, Dims, P, P, P, P, P, P, ctypes.c_uint32,
                                            P, P, P, U64, P, P, P, P]
    L.warp3d_noise.argtypes = [P, Dims, F, U64, U64, P]
    L.warp3d_philox4x32_10.argtypes = [P, U64, P, I64, P]
    L.warp3d_footprint_batched.argtypes = [I32, Dims, P, Dims, P, P, P]
    L.warp3d_pipeline_create.argtypes = [I32, Dims, Dims, I32, ctypes.POINTER(ctypes.c_void_p)]
    L.warp3d_pipeline_create_ex.argtypes = [I32, I32, Dims, Dims, I32,
                                            ctypes.POINTER(ctypes.c_void_p)]
    L.warp3d_pipeline_create_ex.restype = ctypes.c_int
    L.warp3d_pipeline_vols_per_job.argtypes = [P]
    L.warp3d_pipeline_vols_per_job.restype = I32
    L.warp3d_pipeline_run.argtypes = [P, I32, P, P, P, I32, F, ctypes.c_uint8, P, P, P]
    L.warp3d_pipeline_destroy.argtypes = [P]
    for name in ("warp3d_pipeline_create", "warp3d_pipeline_run", "warp3d_pipeline_destroy"):
        getattr(L, name).restype = ctypes.c_int
    L.warp3d_affine_batched_i16.argtypes = [I32, P, P, Dims, P, I32, F, ctypes.c_uint8, P, P,
                                            Dims, P]
    L.warp3d_affine_batched_i16_ex.argtypes = [I32, P, P, Dims, P, I32, F, ctypes.c_uint8, P, P,
                                               Dims, I32, P]
    L.warp3d_affine_batched_i16.restype = ctypes.c_int
    L.warp3d_affine_batched_v.argtypes = [I32, I32, P, P, P, P, I32, F, ctypes.c_uint8, P, P, Dims,
                                          P]
    L.warp3d_affine_batched_v.restype = ctypes.c_int
    L.warp3d_affine_batched_i16_ex.restype = ctypes.c_int
    D = ctypes.c_double
    L.warp3d_resample_sigma.argtypes = [P, D, P]
    L.warp3d_resample_dims.argtypes = [Dims, P, D, ctypes.POINTER(Dims)]
    L.warp3d_resample_affine.argtypes = [Dims, Dims, P, D, P]
    L.warp3d_smooth3d.argtypes = [P, Dims, P, P, P, P]
    L.warp3d_resample.argtypes = [P, P, Dims, P, D, F, ctypes.c_uint8, P, P, Dims, P, P]
    for name in ("warp3d_resample_sigma", "warp3d_resample_dims", "warp3d_resample_affine",
                 "warp3d_smooth3d", "warp3d_resample"):
        getattr(L, name).restype = ctypes.c_int
    L.warp3d_tile_stats.argtypes = [P]
    L.warp3d_tile_stats.restype = ctypes.c_int
    L.warp3d_launch_count.restype = U64
    L.warp3d_launch_count.argtypes = []
    L.warp3d_last_error.restype = ctypes.c_char_p
    L.warp3d_last_error.argtypes = []
    L.warp3d_abi_version.restype = ctypes.c_int
    L.warp3d_abi_version.argtypes = []
    for name in ("warp3d_affine", "warp3d_affine_batched", "warp3d_affine_batched_ex",
                 "warp3d_compose_affine", "warp3d_noise", "warp3d_philox4x32_10",
                 "warp3d_footprint_batched"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(status):
    if status != W3D_OK:
        raise Warp3DError(status, load().warp3d_last_error().decode())


def dims(shape_zyx):
    nz, ny, nx = (int(s) for s in shape_zyx)
    return Dims(nx, ny, nz)
