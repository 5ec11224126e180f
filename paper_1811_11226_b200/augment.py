"""Per-volume parameter assembly for a training batch.

A "draw" is any object with the fields of synth.VolumeDraw (rot_rad, scale,
shear, flip, generic, disp, window, gamma, sigma): the random numbers the
method samples per training example.
The affine is composed by the library's own warp3d_compose_affine.
"""
from __future__ import annotations

import ctypes

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


def build_params(draws, volume_ids, in_shape_zyx, out_shape_zyx=None, flags=FULL, seed=0,
                 sigma_override=None):
    """ctypes array of VolumeParams, volume i keyed by GLOBAL volume_ids[i]."""
    out_shape_zyx = in_shape_zyx if out_shape_zyx is None else out_shape_zyx
    arr = (VolumeParams * len(draws))()
    for i, (d, vid) in enumerate(zip(draws, volume_ids)):
        g = api.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp)
        A = api.warp3d_compose_affine(g, in_shape_zyx, out_shape_zyx)
        ph = photometric_from_draw(d, flags, seed, vid)
        if sigma_override is not None:
            ph.noise_sigma = float(sigma_override)
        arr[i] = api.volume_params(A, ph)
    return arr


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
