"""Image tolerance of the parity tests.

north_star: image voxels agree within 1e-5 relative or 1e-3 HU absolute.
Without a window the output is in HU and the bound is max(1e-5 |r|, 1e-3).
With window (and gamma) the output is f(v) = clamp((v - a) s)^gamma of an HU
value v; a 1e-3 HU error in v maps to the exact image of the interval
[v - 1e-3, v + 1e-3] under f, so the bound is

    max(1e-5 |r|,  max(|f(v + eps) - f(v)|, |f(v) - f(v - eps)|)),  eps = 1e-3 HU,

evaluated from the oracle's own output r (w = r^(1/gamma) recovers the window value).
"""
import numpy as np

EPS_HU = 1e-3
REL = 1e-5


def image_tol(ref, window=None, gamma=1.0, clamp=True):
    r = np.asarray(ref, dtype=np.float64)
    if window is None:
        return np.maximum(REL * np.abs(r), EPS_HU)
    a, b = window
    s = 1.0 / (float(b) - float(a))
    g = float(gamma)
    if g != 1.0:
        w = np.power(np.clip(r, 0.0, 1.0), 1.0 / g)
    else:
        w = r
    d = s * EPS_HU
    hi = w + d
    lo = w - d
    if clamp:
        hi = np.clip(hi, 0.0, 1.0)
        lo = np.clip(lo, 0.0, 1.0)
        ww = np.clip(w, 0.0, 1.0)
    else:
        ww = w
    if g != 1.0:
        f = lambda t: np.power(t, g)  # noqa: E731
    else:
        f = lambda t: t  # noqa: E731
    band = np.maximum(np.abs(f(hi) - f(ww)), np.abs(f(ww) - f(lo)))
    return np.maximum(REL * np.abs(r), band)


def assert_image_close(gpu, ref, window=None, gamma=1.0, clamp=True, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tol = image_tol(ref, window, gamma, clamp)
    err = np.abs(gpu - ref)
    bad = err > tol
    if bad.any():
        i = np.flatnonzero(bad.ravel())[:8]
        raise AssertionError(
            f"{what}: {int(bad.sum())} of {bad.size} image voxels outside tolerance; "
            f"first idx {i.tolist()} gpu {gpu.ravel()[i].tolist()} ref {ref.ravel()[i].tolist()} "
            f"tol {tol.ravel()[i].tolist()}")
    return float(np.max(err / tol)) if err.size else 0.0
