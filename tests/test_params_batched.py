"""Host-only (no GPU): the batched parameter builder (augment.params_from_arrays over
warp3d_compose_params_batched) gives the same VolumeParams bytes as composing volume by
volume through warp3d_compose_affine, for every draw family the benches use."""
import ctypes
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build  # noqa: E402
import synth  # noqa: E402


@pytest.fixture(scope="module")
def W():
    build.build_cuda()
    import paper_1811_11226_b200 as W
    return W


def _per_volume(W, draws, vids, shape, flags, seed):
    from paper_1811_11226_b200.augment import photometric_from_draw
    from paper_1811_11226_b200._lib import VolumeParams
    out = (VolumeParams * len(draws))()
    for i, (d, v) in enumerate(zip(draws, vids)):
        g = W.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp)
        A = W.warp3d_compose_affine(g, shape, shape)
        out[i] = W.volume_params(A, photometric_from_draw(d, flags, seed, v))
    return out


@pytest.mark.parametrize("ranges", ["TRAIN", "LARGE", "TRAIN_OCC"])
def test_batched_params_equal_per_volume(W, ranges):
    from paper_1811_11226_b200.augment import FULL, build_params
    shape = (160, 128, 128)
    R = getattr(synth, ranges)
    vids = list(range(1000, 1064))
    draws = [synth.draw(R, v, out_mz=shape[0]) for v in vids]
    a = build_params(draws, vids, shape, shape, FULL, seed=0x181111226)
    b = _per_volume(W, draws, vids, shape, FULL, 0x181111226)
    assert bytes(a) == bytes(b)


def test_params_from_arrays_validates(W):
    from paper_1811_11226_b200.augment import params_from_arrays
    from paper_1811_11226_b200._lib import Warp3DError
    with pytest.raises(Warp3DError):   # scale <= 0
        params_from_arrays((8, 8, 8), [[0, 0, 0]], [[1, 0, 1]])
    with pytest.raises(Warp3DError):   # gamma <= 0
        params_from_arrays((8, 8, 8), [[0, 0, 0]], [[1, 1, 1]], gamma=0.0)
    p = params_from_arrays((8, 8, 8), np.zeros((3, 3)), np.ones((3, 3)))
    assert len(p) == 3 and list(p[2].affine)[:4] == [1.0, 0.0, 0.0, 0.0]
    assert ctypes.sizeof(p) == 3 * 96
