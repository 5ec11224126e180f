"""C-ABI library tests that need no GPU: the library loads, exports every symbol
include/warp3d.h declares, validates arguments before launching, and its host
composition agrees with the oracle's."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def W():
    build.build_cuda()
    import paper_1811_11226_b200 as W
    return W


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "warp3d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(warp3d_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported(W):
    from paper_1811_11226_b200 import _lib
    L = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == declared
    assert W.warp3d_abi_version() == 3


def test_struct_sizes_match_header(W):
    from paper_1811_11226_b200 import _lib
    assert ctypes.sizeof(_lib.Photometric) == 48
    assert ctypes.sizeof(_lib.VolumeParams) == 96
    assert ctypes.sizeof(_lib.Geom) == 8 * 21 + 16


def test_compose_matches_oracle(W):
    import oracle as O
    import synth
    for idx in range(300):
        d = synth.draw(synth.TRAIN if idx % 2 else synth.LARGE, idx)
        shp_in, shp_out = (160, 128, 128), ((160, 120, 120) if idx % 3 == 0 else (160, 128, 128))
        ours = W.warp3d_compose_affine(
            W.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp), shp_in, shp_out)
        _, ref = O.compose_affine(
            O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic, d.disp), shp_in, shp_out)
        # both evaluate the same double expression then round once to fp32: allow 1 ulp
        # for a different double summation order
        ulp = np.spacing(np.maximum(np.abs(ref), np.float32(1e-30)))
        assert np.all(np.abs(ours - ref) <= ulp), (idx, ours - ref)


def _call_batched(W, **kw):
    from paper_1811_11226_b200 import _lib
    L = _lib.load()
    args = dict(batch=1, inp=0x10000, lbl=None, in_dims=(4, 4, 4), params=None, interp=0,
                fill=0.0, label_fill=0, out=0x20000, out_lbl=None, out_dims=(4, 4, 4), variant=0)
    args.update(kw)
    params = args["params"]
    if params is None:
        params = (_lib.VolumeParams * max(1, args["batch"]))()
        for p in params:
            p.affine[:] = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
    st = L.warp3d_affine_batched_ex(args["batch"], ctypes.c_void_p(args["inp"]),
                                    None if args["lbl"] is None else ctypes.c_void_p(args["lbl"]),
                                    _lib.Dims(*args["in_dims"]), params, args["interp"],
                                    args["fill"], args["label_fill"],
                                    ctypes.c_void_p(args["out"]),
                                    None if args["out_lbl"] is None else ctypes.c_void_p(args["out_lbl"]),
                                    _lib.Dims(*args["out_dims"]), args["variant"], None)
    return st, L.warp3d_last_error().decode()


def _params(W, **ph):
    from paper_1811_11226_b200 import _lib
    p = (_lib.VolumeParams * 1)()
    p[0].affine[:] = [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]
    for k, v in ph.items():
        setattr(p[0].ph, k, v)
    return p


@pytest.mark.parametrize("case", [
    dict(batch=0),
    dict(inp=0),
    dict(out=0),
    dict(inp=0x10002),                        # misaligned float pointer
    dict(in_dims=(0, 4, 4)),
    dict(out_dims=(4, -1, 4)),
    dict(in_dims=(1 << 23, 1, 1)),
    dict(interp=7),
    dict(fill=float("nan")),
    dict(fill=float("inf")),
    dict(lbl=0x30000),                        # labels in without labels out
    dict(out_lbl=0x30000),
    dict(variant=9),
    dict(out=0x10000 + 64),                   # out overlaps in
])
def test_invalid_arguments_rejected_before_launch(W, case):
    st, msg = _call_batched(W, **case)
    assert st == 1, (case, st, msg)
    assert msg


@pytest.mark.parametrize("ph", [
    dict(flags=64),
    dict(flags=4),                            # CLAMP without WINDOW
    dict(flags=2 | 8),                        # GAMMA without CLAMP
    dict(flags=2, window_lo=1.0, window_hi=1.0),
    dict(flags=2, window_lo=float("nan"), window_hi=1.0),
    dict(flags=2 | 4 | 8, window_lo=0.0, window_hi=1.0, gamma=0.0),
    dict(flags=2 | 4 | 8, window_lo=0.0, window_hi=1.0, gamma=-1.0),
    dict(flags=1, noise_sigma=-1.0),
    dict(flags=1, noise_sigma=float("inf")),
    dict(flags=16, occ_z0=0.0, occ_height=-1.0),
    dict(_reserved=1),
])
def test_invalid_photometric_rejected(W, ph):
    st, msg = _call_batched(W, params=_params(W, **ph))
    assert st == 1, (ph, msg)


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), 2.0 ** 21])
def test_invalid_affine_rejected(W, bad):
    p = _params(W)
    p[0].affine[1] = bad
    st, msg = _call_batched(W, params=p)
    assert st == 1 and "affine" in msg


def test_too_many_voxels_unsupported(W):
    st, msg = _call_batched(W, in_dims=(2048, 2048, 1024), out=1 << 45)
    assert st == 2, msg


def test_compose_rejects_bad_geom(W):
    g = W.make_geom(scale=(1, 0, 1))
    with pytest.raises(W.Warp3DError):
        W.warp3d_compose_affine(g, (4, 4, 4))
    g = W.make_geom(rot=(math.nan, 0, 0))
    with pytest.raises(W.Warp3DError):
        W.warp3d_compose_affine(g, (4, 4, 4))


def test_hooks_validate(W):
    from paper_1811_11226_b200 import _lib
    L = _lib.load()
    assert L.warp3d_noise(None, _lib.Dims(4, 4, 4), 1.0, 0, 0, None) == 1
    assert L.warp3d_noise(ctypes.c_void_p(0x1000), _lib.Dims(4, 4, 4), -1.0, 0, 0, None) == 1
    assert L.warp3d_philox4x32_10(None, 0, ctypes.c_void_p(0x1000), 4, None) == 1
    assert L.warp3d_philox4x32_10(ctypes.c_void_p(0x1004), 0, ctypes.c_void_p(0x2000), 4, None) == 1
    assert L.warp3d_philox4x32_10(ctypes.c_void_p(0x1000), 0, ctypes.c_void_p(0x2000), 0, None) == 0


def test_no_gpu_means_cuda_error_not_fallback(W):
    """On a machine without a GPU the compute entry points fail loudly (W3D_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, msg = _call_batched(W)
    assert st == 3, msg


def test_pipeline_create_validates(W):
    from paper_1811_11226_b200 import _lib
    L = _lib.load()
    h = ctypes.c_void_p()
    assert L.warp3d_pipeline_create(0, _lib.Dims(4, 4, 4), _lib.Dims(4, 4, 4), 1, ctypes.byref(h)) == 1
    assert L.warp3d_pipeline_create(9, _lib.Dims(4, 4, 4), _lib.Dims(4, 4, 4), 1, ctypes.byref(h)) == 1
    assert L.warp3d_pipeline_create(2, _lib.Dims(0, 4, 4), _lib.Dims(4, 4, 4), 1, ctypes.byref(h)) == 1
    assert L.warp3d_pipeline_create(2, _lib.Dims(4, 4, 4), _lib.Dims(4, 4, 4), 4, ctypes.byref(h)) == 1
    assert L.warp3d_pipeline_run(None, 1, None, None, None, 0, 0.0, 0, None, None, None) == 1
    assert L.warp3d_pipeline_destroy(None) == 0
    d = _lib.Dims(4, 4, 4)
    assert L.warp3d_pipeline_create_ex(2, -1, d, d, 1, ctypes.byref(h)) == 1   # vols_per_job < 0
    assert L.warp3d_pipeline_create_ex(2, 105, d, d, 1, ctypes.byref(h)) == 1  # > 104
    assert L.warp3d_pipeline_create_ex(0, 1, d, d, 1, ctypes.byref(h)) == 1    # depth
    assert L.warp3d_pipeline_vols_per_job(None) == 0


def test_resample_host_functions_match_oracle(W):
    """NEXT-3 host side (no GPU): sigma, dims and the centre-aligned scale map agree
    with the oracle's independent implementations (dims / affine bit for bit)."""
    import oracle as O
    rng = np.random.default_rng(11)
    for _ in range(40):
        shape = tuple(int(v) for v in rng.integers(1, 600, size=3))
        u = tuple(float(v) for v in rng.uniform(0.3, 6.0, size=3))
        r = float(rng.choice([3.0, 2.0, 1.5]))
        assert np.allclose(W.warp3d_resample_sigma(u, r), O.resample_sigma(u, r), rtol=0,
                           atol=1e-15)
        out_shape = W.warp3d_resample_dims(shape, u, r)
        assert out_shape == O.resample_dims(shape, u, r)
        assert np.array_equal(W.warp3d_resample_affine(shape, out_shape, u, r),
                              O.resample_affine(shape, out_shape, u, r))
    with pytest.raises(W.Warp3DError):
        W.warp3d_resample_sigma((1.0, 0.0, 1.0), 3.0)


def test_product_library_is_the_default_build():
    """The library the package loads was built with the default flags (the flag stamp
    written by build.py; a knob build with other flags always rebuilds)."""
    import json
    import build
    build.build_cuda()
    with open(build.PRODUCT_LIB + ".flags") as f:
        stamp = json.load(f)
    extra = [a for a in stamp["flags"] if a not in build._flags([])]
    assert stamp["flags"] == build._flags([]) and not extra, extra
    assert stamp["sources"] == build.CUDA_SOURCES
