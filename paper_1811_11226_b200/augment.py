"""Per-volume parameter assembly for a training batch.

A "draw" is any object with the fields of synth.VolumeDraw (rot_rad, scale,
shear, flip, generic, disp, window, gamma, sigma): the random numbers the
method samples per training example.
The affine is composed by the library's own warp3d_compose_affine.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from . import api
from ._lib import PH_CLAMP, PH_GAMMA, PH_NOISE, PH_OCCLUDE, PH_WINDOW, VolumeParams

FULL = PH_NOISE | PH_WINDOW | PH_CLAMP | PH_GAMMA


def photometric_from_draw(draw, flags, seed, volume_id):
    """w3d_photometric of one draw; a draw with an occlusion prism (occ_height >= 0,
    PAPER.md:420-438) adds W3D_PH_OCCLUDE."""
    occ = getattr(draw, "occ_height", -1.0)
    if occ is not None and occ >= 0.0:
        flags |= PH_OCCLUDE
    else:
        occ = 0.0
    return api.photometric(flags, window=draw.window, gamma=draw.gamma, sigma=draw.sigma,
                           seed=seed, volume_id=volume_id,
                           occ_z0=getattr(draw, "occ_z0", 0.0), occ_height=occ)


def _col(x, n, k, dtype):
    """x as a C-contiguous [n, k] (or [n]) array of dtype, scalars broadcast."""
    shape = (n,) if k == 1 else (n, k)
    if isinstance(x, np.ndarray) and x.dtype == dtype and x.shape == shape and x.flags.c_contiguous:
        return x
    a = np.asarray(x, dtype=dtype)
    if a.shape != shape:
        a = np.broadcast_to(a, shape)
    return np.ascontiguousarray(a)


def _ptr(a):
    # (ndarray.ctypes builds a helper object per call: ~10x the cost of the interface)
    return None if a is None else a.__array_interface__["data"][0]


def params_from_arrays(in_shape_zyx, rot_rad, scale, shear=None, flip=None, disp=None,
                       generic=None, *, out_shape_zyx=None, flags=FULL, window=(0.0, 1.0),
                       gamma=1.0, sigma=0.0, seed=0, volume_ids=None, occ_z0=None,
                       occ_height=None):
    """ctypes array of n VolumeParams from per-volume arrays (x, y, z columns): rot_rad,
    scale, shear, disp [n, 3] float, flip [n, 3] bool, generic [n, 9] (G - I, row-major,
    the w3d_geom convention) or None (G = I), window [n, 2] or one pair, gamma / sigma
    [n] or scalars, volume_ids [n] (default 0..n-1), occ_z0 / occ_height [n] or None (an
    occ_height >= 0 sets PH_OCCLUDE for that volume).  One library call
    (warp3d_params_from_arrays) composes the affines and fills the photometrics; no
    per-volume Python."""
    out_shape_zyx = in_shape_zyx if out_shape_zyx is None else out_shape_zyx
    rot = np.ascontiguousarray(np.asarray(rot_rad, dtype=np.float64).reshape(-1, 3))
    n = rot.shape[0]
    keep = [rot, _col(scale, n, 3, np.float64),
            None if shear is None else _col(shear, n, 3, np.float64),
            None if flip is None else _col(np.asarray(flip, dtype=bool), n, 3, np.uint8),
            None if disp is None else _col(disp, n, 3, np.float64),
            None if generic is None else _col(np.asarray(generic, np.float64).reshape(n, 9), n, 9,
                                              np.float64),
            _col(window, n, 2, np.float64), _col(gamma, n, 1, np.float64),
            _col(sigma, n, 1, np.float64),
            None if volume_ids is None else _col(volume_ids, n, 1, np.uint64),
            None if occ_z0 is None else _col(occ_z0, n, 1, np.float64),
            None if occ_height is None else _col(occ_height, n, 1, np.float64)]
    out = (VolumeParams * n)()
    L.check(L.load().warp3d_params_from_arrays(
        n, L.dims(in_shape_zyx), L.dims(out_shape_zyx), *[_ptr(k) for k in keep[:6]],
        int(flags), *[_ptr(k) for k in keep[6:9]], int(seed), *[_ptr(k) for k in keep[9:]],
        out))
    return out


def build_params(draws, volume_ids, in_shape_zyx, out_shape_zyx=None, flags=FULL, seed=0,
                 sigma_override=None):
    """ctypes array of VolumeParams, volume i keyed by GLOBAL volume_ids[i]."""
    generic = None
    if any(d.generic is not None for d in draws):
        generic = [np.zeros(9) if d.generic is None else np.asarray(d.generic, dtype=np.float64)
                   for d in draws]
    occ_h = [getattr(d, "occ_height", -1.0) for d in draws]
    occ_h = [(-1.0 if h is None else h) for h in occ_h]
    return params_from_arrays(
        in_shape_zyx, [d.rot_rad for d in draws], [d.scale for d in draws],
        [d.shear for d in draws], [d.flip for d in draws], [d.disp for d in draws], generic,
        out_shape_zyx=out_shape_zyx, flags=flags, window=[d.window for d in draws],
        gamma=[d.gamma for d in draws],
        sigma=[d.sigma for d in draws] if sigma_override is None else float(sigma_override),
        seed=seed, volume_ids=list(volume_ids), occ_z0=[getattr(d, "occ_z0", 0.0) for d in draws],
        occ_height=occ_h)


class AugmentBatch:
    """Device-resident batch: inputs, outputs and per-volume params."""

    def __init__(self, image, labels, params, out_shape=None, fill=-1000.0, label_fill=0,
                 variant=api.KERNEL_AUTO):
        import torch
        self.image, self.labels, self.params = image, labels, params
        B = image.shape[0]
        self.out_shape = tuple(image.shape[1:]) if out_shape is None else tuple(out_shape)
        self.out = torch.empty((B, *self.out_shape), dtype=torch.float32, device=image.device)
        self.out_labels = None if labels is None else torch.empty(
            (B, *self.out_shape), dtype=torch.uint8, device=image.device)
        self.fill, self.label_fill, self.variant = fill, label_fill, variant

        # the first run goes through the checked entry point (validates every buffer);
        # later runs reuse its marshalled arguments: the buffers are fixed for the life
        # of the batch and `params` is the same ctypes array (updated in place between
        # training steps if the caller draws new transforms)
        self._call = None

    def set_params(self, params):
        """Next step's per-volume parameters (a ctypes array of the same length, e.g. from
        params_from_arrays), copied into the array the prepared call reads."""
        if len(params) != len(self.params):
            raise ValueError(f"{len(params)} params for a batch of {len(self.params)}")
        if not isinstance(self.params, ctypes.Array):
            self.params = (VolumeParams * len(self.params))(*self.params)
            self._call = None
        ctypes.memmove(self.params, (VolumeParams * len(params))(*params)
                       if not isinstance(params, ctypes.Array) else params,
                       ctypes.sizeof(VolumeParams) * len(params))

    def run(self):
        if self._call is None:
            api.warp3d_affine_batched(self.image, self.labels, self.params, fill=self.fill,
                                      label_fill=self.label_fill, out_shape=self.out_shape,
                                      out=self.out, out_labels=self.out_labels,
                                      variant=self.variant)
            self._call = api.prepared_batched_call(
                self.image, self.labels, self.params, self.fill, self.label_fill, self.out,
                self.out_labels, self.variant)
            return self.out, self.out_labels
        self._call()
        return self.out, self.out_labels
