"""B200-native (sm_100a) 3D CT augmentation hot path of Rister et al., arXiv 1811.11226.

Batched pull-back affine warp (trilinear image, nearest label) fused with
Philox/Box-Muller noise, window/clamp and gamma, as a C-ABI
CUDA library (include/warp3d.h) with a thin ctypes binding.  See DESIGN.md.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
from .augment import AugmentBatch, build_params, photometric_from_draw  # noqa: F401
