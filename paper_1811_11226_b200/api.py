"""Python entry points with the C-ABI's names (include/warp3d.h).

PyTorch provides device memory and the current CUDA stream; every step of
the augmentation runs in libwarp3d.so.  Tensors are passed
as raw device pointers; shapes are numpy-style [batch, nz, ny, nx].
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L
from ._lib import (INTERP_LINEAR, INTERP_NEAREST, KERNEL_AUTO, KERNEL_GATHER, KERNEL_STAGED,
                   PH_CLAMP, PH_GAMMA, PH_NOISE, PH_OCCLUDE, PH_WINDOW, Geom, Photometric,
                   VolumeParams, Warp3DError)

__all__ = [
    "warp3d_affine", "warp3d_affine_batched", "warp3d_compose_affine", "warp3d_noise",
    "warp3d_philox4x32_10", "warp3d_footprint_batched", "warp3d_launch_count",
    "warp3d_tile_stats", "Pipeline", "warp3d_resample_sigma", "warp3d_resample_dims",
    "warp3d_resample_affine", "warp3d_smooth3d", "warp3d_resample", "warp3d_affine_batched_list",
    "warp3d_abi_version", "photometric", "volume_params", "make_geom", "Warp3DError",
    "INTERP_LINEAR", "INTERP_NEAREST", "KERNEL_AUTO", "KERNEL_GATHER", "KERNEL_STAGED",
    "PH_NOISE", "PH_WINDOW", "PH_CLAMP", "PH_GAMMA", "PH_OCCLUDE",
]


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(device=None):
    """The caller's current CUDA stream as a raw handle (the launches go there)."""
    if _raw_stream is not None:
        idx = torch.cuda.current_device() if device is None else device.index
        return ctypes.c_void_p(_raw_stream(idx))
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev(t, dtype, name, shape=None, device=None):
    """Device pointer of a contiguous CUDA tensor, after checking its dtype, shape and
    device (the C side trusts the sizes it derives from dims and batch)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    return ctypes.c_void_p(t.data_ptr())


def _host(t, dtype, name, shape):
    """Address of a contiguous HOST tensor of exactly this dtype and shape."""
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a host (CPU) tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def photometric(flags=0, window=(0.0, 1.0), gamma=1.0, sigma=0.0, seed=0, volume_id=0,
                occ_z0=0.0, occ_height=0.0) -> Photometric:
    return Photometric(int(flags), float(window[0]), float(window[1]), float(gamma),
                       float(sigma), 0, int(seed), int(volume_id), float(occ_z0),
                       float(occ_height))


def make_geom(rot=(0, 0, 0), scale=(1, 1, 1), shear=(0, 0, 0), flip=(0, 0, 0), generic=None,
              disp=(0, 0, 0)) -> Geom:
    g = Geom()
    g.rot_rad[:] = [float(v) for v in rot]
    g.scale[:] = [float(v) for v in scale]
    g.shear[:] = [float(v) for v in shear]
    g.flip[:] = [int(bool(v)) for v in flip]
    g.generic[:] = [0.0] * 9 if generic is None else [float(v) for v in np.ravel(generic)]
    g.disp[:] = [float(v) for v in disp]
    return g


def warp3d_compose_affine(geom: Geom, in_shape_zyx, out_shape_zyx=None) -> np.ndarray:
    """Host-only: [A|b] (float32 [3,4]) for a w3d_geom."""
    out_shape_zyx = in_shape_zyx if out_shape_zyx is None else out_shape_zyx
    out = (ctypes.c_float * 12)()
    L.check(L.load().warp3d_compose_affine(ctypes.byref(geom), L.dims(in_shape_zyx),
                                           L.dims(out_shape_zyx), out))
    return np.array(out, dtype=np.float32).reshape(3, 4)


def volume_params(affine, ph: Photometric | None = None) -> VolumeParams:
    p = VolumeParams()
    p.affine[:] = [float(v) for v in np.asarray(affine, dtype=np.float32).ravel()]
    if ph is not None:
        p.ph = ph
    return p


def warp3d_affine(inp: torch.Tensor, affine, interp=INTERP_LINEAR, fill=0.0, ph=None,
                  out_shape=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """One volume: inp float32 [nz,ny,nx] on the GPU -> out float32 [mz,my,mx]."""
    if inp.dim() != 3:
        raise ValueError("inp must be [nz, ny, nx]")
    out_shape = tuple(inp.shape) if out_shape is None else tuple(out_shape)
    if out is None:
        out = torch.empty(out_shape, dtype=torch.float32, device=inp.device)
    A = (ctypes.c_float * 12)(*[float(v) for v in np.asarray(affine, dtype=np.float32).ravel()])
    L.check(L.load().warp3d_affine(_dev(inp, torch.float32, "inp"), L.dims(inp.shape), A,
                                   int(interp), float(fill),
                                   None if ph is None else ctypes.byref(ph),
                                   _dev(out, torch.float32, "out", out_shape, inp.device),
                                   L.dims(out.shape), _stream()))
    return out


def warp3d_affine_batched(inp: torch.Tensor, labels: torch.Tensor | None, params,
                          interp=INTERP_LINEAR, fill=0.0, label_fill=0, out_shape=None,
                          out: torch.Tensor | None = None, out_labels: torch.Tensor | None = None,
                          variant=KERNEL_AUTO):
    """Batch: inp float32 or int16 (HU) [B,nz,ny,nx], labels uint8 [B,nz,ny,nx] or None,
    params: sequence of B VolumeParams (or a ctypes array of them).  Output float32."""
    if inp.dim() != 4:
        raise ValueError("inp must be [batch, nz, ny, nx]")
    B = inp.shape[0]
    out_shape = tuple(inp.shape[1:]) if out_shape is None else tuple(out_shape)
    if out is None:
        out = torch.empty((B, *out_shape), dtype=torch.float32, device=inp.device)
    if labels is not None and out_labels is None:
        out_labels = torch.empty((B, *out_shape), dtype=torch.uint8, device=inp.device)
    if len(params) != B:  # before the ctypes array (which would zero-pad a short list)
        raise ValueError(f"{len(params)} params for a batch of {B}")
    arr = params if isinstance(params, ctypes.Array) else (VolumeParams * B)(*params)
    if (labels is None) != (out_labels is None):
        raise ValueError("out_labels must be given exactly when labels are")
    dev, oshape = inp.device, (B, *out_shape)
    if inp.dtype == torch.int16:  # NEXT-4: int16 HU input, float32 output
        fn, src = L.load().warp3d_affine_batched_i16_ex, _dev(inp, torch.int16, "inp")
    else:
        fn, src = L.load().warp3d_affine_batched_ex, _dev(inp, torch.float32, "inp")
    L.check(fn(
        B, src,
        None if labels is None else _dev(labels, torch.uint8, "labels", inp.shape, dev),
        L.dims(inp.shape[1:]), arr, int(interp), float(fill), int(label_fill),
        _dev(out, torch.float32, "out", oshape, dev),
        None if out_labels is None else _dev(out_labels, torch.uint8, "out_labels", oshape, dev),
        L.dims(out_shape), int(variant), _stream()))
    return out, out_labels


def prepared_batched_call(inp, labels, params, fill, label_fill, out, out_labels,
                          variant=KERNEL_AUTO):
    """A no-argument callable that repeats one (already validated) warp3d_affine_batched
    launch on the caller's current stream: the ctypes arguments are marshalled once.
    The tensors must stay alive and unchanged in shape; `params` must be a ctypes array
    (its contents may change between calls)."""
    if not isinstance(params, ctypes.Array):
        raise TypeError("params must be a ctypes array of VolumeParams")
    fn = (L.load().warp3d_affine_batched_i16_ex if inp.dtype == torch.int16
          else L.load().warp3d_affine_batched_ex)
    fixed = (int(inp.shape[0]), ctypes.c_void_p(inp.data_ptr()),
             None if labels is None else ctypes.c_void_p(labels.data_ptr()),
             L.dims(inp.shape[1:]), params, INTERP_LINEAR, float(fill), int(label_fill),
             ctypes.c_void_p(out.data_ptr()),
             None if out_labels is None else ctypes.c_void_p(out_labels.data_ptr()),
             L.dims(out.shape[1:]), int(variant))
    device = inp.device
    check = L.check

    def call():
        check(fn(*fixed, _stream(device)))
    return call


def warp3d_affine_batched_list(inputs, labels, params, out_shape, interp=INTERP_LINEAR,
                               fill=0.0, label_fill=0):
    """Volumes of different shapes (list of float32 or int16 [nz,ny,nx] CUDA tensors, one
    dtype) and their labels (list or None) into one [B, *out_shape] batch (NEXT-4)."""
    B = len(inputs)
    if B == 0 or (labels is not None and len(labels) != B) or len(params) != B:
        raise ValueError("inputs, labels and params must have the same non-zero length")
    i16 = inputs[0].dtype == torch.int16
    dt = torch.int16 if i16 else torch.float32
    dev = inputs[0].device
    ptrs = (ctypes.c_void_p * B)(*[_dev(t, dt, f"inputs[{i}]").value for i, t in enumerate(inputs)])
    dims = (L.Dims * B)(*[L.dims(t.shape) for t in inputs])
    lptrs = None
    if labels is not None:
        lptrs = (ctypes.c_void_p * B)(*[_dev(t, torch.uint8, f"labels[{i}]").value
                                        for i, t in enumerate(labels)])
    out = torch.empty((B, *out_shape), dtype=torch.float32, device=dev)
    out_l = None if labels is None else torch.empty((B, *out_shape), dtype=torch.uint8, device=dev)
    arr = params if isinstance(params, ctypes.Array) else (VolumeParams * B)(*params)
    L.check(L.load().warp3d_affine_batched_v(
        B, 1 if i16 else 0, ptrs, lptrs, dims, arr, int(interp), float(fill), int(label_fill),
        _dev(out, torch.float32, "out"), None if out_l is None else _dev(out_l, torch.uint8, "out_labels"),
        L.dims(out_shape), _stream()))
    return out, out_l


def warp3d_noise(shape_zyx, sigma, seed, volume_id, device="cuda") -> torch.Tensor:
    out = torch.empty(tuple(shape_zyx), dtype=torch.float32, device=device)
    L.check(L.load().warp3d_noise(_dev(out, torch.float32, "out"), L.dims(shape_zyx),
                                  float(sigma), int(seed), int(volume_id), _stream()))
    return out


def warp3d_philox4x32_10(ctr: torch.Tensor, key: int) -> torch.Tensor:
    """ctr: int32/uint32 CUDA tensor [n,4] (bit pattern) -> out same shape."""
    if ctr.dim() != 2 or ctr.shape[1] != 4:
        raise ValueError("ctr must be [n, 4]")
    out = torch.empty_like(ctr)
    L.check(L.load().warp3d_philox4x32_10(_dev(ctr, ctr.dtype, "ctr"), int(key),
                                          _dev(out, ctr.dtype, "out"), ctr.shape[0], _stream()))
    return out


def warp3d_footprint_batched(params, in_shape_zyx, out_shape_zyx=None, device="cuda"):
    """(#F_img, #F_lbl): distinct input voxels the warp reads (measurement only)."""
    out_shape_zyx = in_shape_zyx if out_shape_zyx is None else out_shape_zyx
    arr = params if isinstance(params, ctypes.Array) else (VolumeParams * len(params))(*params)
    B = len(arr)
    nin = int(np.prod(in_shape_zyx))
    marks = torch.empty(2 * B * nin, dtype=torch.uint8, device=device)
    counts = torch.zeros(2, dtype=torch.int64, device=device)
    L.check(L.load().warp3d_footprint_batched(B, L.dims(in_shape_zyx), arr, L.dims(out_shape_zyx),
                                              ctypes.c_void_p(marks.data_ptr()),
                                              ctypes.c_void_p(counts.data_ptr()), _stream()))
    c = counts.cpu().tolist()
    return int(c[0]), int(c[1])


class Pipeline:
    """FIFO host pipeline (include/warp3d.h warp3d_pipeline_*):
    H2D of job j+1, the warp of job j and the D2H of job j-1 overlap (a job is
    `vols_per_job` consecutive volumes; 0 lets the library choose).
    Host tensors should be pinned (tensor.pin_memory())."""

    def __init__(self, in_shape_zyx, out_shape_zyx=None, depth=3, labels=True, chain=False,
                 vols_per_job=0):
        """chain=True: W3D_PIPE_CHAIN (calls ordered after the previous calls on this
        pipeline only, so consecutive batches' transfers overlap; see warp3d.h)."""
        self.in_shape = tuple(in_shape_zyx)
        self.out_shape = self.in_shape if out_shape_zyx is None else tuple(out_shape_zyx)
        self._h = ctypes.c_void_p()
        flags = (1 if labels else 0) | (2 if chain else 0)
        L.check(L.load().warp3d_pipeline_create_ex(int(depth), int(vols_per_job),
                                                   L.dims(self.in_shape), L.dims(self.out_shape),
                                                   flags, ctypes.byref(self._h)))
        self.vols_per_job = int(L.load().warp3d_pipeline_vols_per_job(self._h))

    def run(self, inp: torch.Tensor, labels, params, out: torch.Tensor, out_labels=None,
            interp=INTERP_LINEAR, fill=0.0, label_fill=0):
        """inp/out (and labels) are CPU tensors [B, nz, ny, nx]; returns immediately,
        results valid after torch.cuda.current_stream() completes."""
        if inp.dim() != 4:
            raise ValueError("inp must be [batch, nz, ny, nx]")
        B = inp.shape[0]
        if len(params) != B:
            raise ValueError(f"{len(params)} params for a batch of {B}")
        if (labels is None) != (out_labels is None):
            raise ValueError("out_labels must be given exactly when labels are")
        ishape, oshape = (B, *self.in_shape), (B, *self.out_shape)
        arr = params if isinstance(params, ctypes.Array) else (VolumeParams * B)(*params)
        L.check(L.load().warp3d_pipeline_run(
            self._h, B, _host(inp, torch.float32, "inp", ishape),
            None if labels is None else _host(labels, torch.uint8, "labels", ishape), arr,
            int(interp), float(fill), int(label_fill), _host(out, torch.float32, "out", oshape),
            None if out_labels is None else _host(out_labels, torch.uint8, "out_labels", oshape),
            _stream()))
        return out, out_labels

    def close(self):
        if self._h:
            L.load().warp3d_pipeline_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


# ----------------------------------------------------------------------------- resampling
def _u(spacing_mm):
    u = (ctypes.c_double * 3)(*[float(v) for v in spacing_mm])
    return u


def warp3d_resample_sigma(spacing_mm, target_mm=3.0):
    """sigma_k = max(r/u_k - 1, 0)/3; spacing_mm = (u_x, u_y, u_z)."""
    out = (ctypes.c_double * 3)()
    L.check(L.load().warp3d_resample_sigma(_u(spacing_mm), float(target_mm), out))
    return tuple(out)


def warp3d_resample_dims(in_shape_zyx, spacing_mm, target_mm=3.0):
    """numpy-order output shape (nz, ny, nx) of warp3d_resample."""
    d = L.Dims()
    L.check(L.load().warp3d_resample_dims(L.dims(in_shape_zyx), _u(spacing_mm), float(target_mm),
                                          ctypes.byref(d)))
    return (d.nz, d.ny, d.nx)


def warp3d_resample_affine(in_shape_zyx, out_shape_zyx, spacing_mm, target_mm=3.0):
    A = (ctypes.c_float * 12)()
    L.check(L.load().warp3d_resample_affine(L.dims(in_shape_zyx), L.dims(out_shape_zyx),
                                            _u(spacing_mm), float(target_mm), A))
    return np.array(A, dtype=np.float32).reshape(3, 4)


def warp3d_smooth3d(inp: torch.Tensor, sigma_xyz) -> torch.Tensor:
    """Separable Gaussian lowpass of a float32 [nz, ny, nx] CUDA tensor."""
    out = torch.empty_like(inp)
    tmp = torch.empty_like(inp)
    s = (ctypes.c_double * 3)(*[float(v) for v in sigma_xyz])
    L.check(L.load().warp3d_smooth3d(_dev(inp, torch.float32, "inp"), L.dims(inp.shape), s,
                                     _dev(out, torch.float32, "out"),
                                     _dev(tmp, torch.float32, "tmp"), _stream()))
    return out


def warp3d_resample(inp: torch.Tensor, labels, spacing_mm, target_mm=3.0, fill=-1000.0,
                    label_fill=0):
    """Resample one volume (float32 [nz, ny, nx]) and its labels (uint8 or None) to
    target_mm spacing: Gaussian lowpass then trilinear / nearest."""
    out_shape = warp3d_resample_dims(inp.shape, spacing_mm, target_mm)
    out = torch.empty(out_shape, dtype=torch.float32, device=inp.device)
    out_l = None if labels is None else torch.empty(out_shape, dtype=torch.uint8,
                                                    device=inp.device)
    tmp = torch.empty(2 * inp.numel(), dtype=torch.float32, device=inp.device)
    L.check(L.load().warp3d_resample(
        _dev(inp, torch.float32, "inp"), None if labels is None else _dev(labels, torch.uint8,
                                                                             "labels", inp.shape,
                                                                             inp.device),
        L.dims(inp.shape), _u(spacing_mm), float(target_mm), float(fill), int(label_fill),
        _dev(out, torch.float32, "out"), None if out_l is None else _dev(out_l, torch.uint8,
                                                                         "out_labels"),
        L.dims(out_shape), _dev(tmp, torch.float32, "tmp"), _stream()))
    return out, out_l


def warp3d_launch_count() -> int:
    return int(L.load().warp3d_launch_count())


def warp3d_tile_stats():
    """(staged tiles, gather tiles, staged by TMA, staged in y-parts) so far in this
    process (diagnostic)."""
    out = (ctypes.c_uint64 * 4)()
    L.check(L.load().warp3d_tile_stats(out))
    return tuple(int(v) for v in out)


def warp3d_abi_version() -> int:
    return int(L.load().warp3d_abi_version())
