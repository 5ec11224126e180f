// cube_config.cuh -- tile shape and staging-buffer constants of the warp kernel
// (shared by the kernel instantiations, cube_kernel.cuh, and the host-side box
// sizing in warp3d_cube.cu).  Experiment knobs: -DW3D_TZ, -DW3D_TY, -DW3D_MINB,
// -DW3D_GMINB, -DW3D_PRE (build.py W3D_NVCC_EXTRA).
#pragma once
#include <cstdint>

namespace w3d {
namespace cube {

// Tile 16 x kTY x TZ output voxels; a warp = 16 x by 2 z, so TZ / 2 warps.
#ifndef W3D_TZ
#define W3D_TZ 16
#endif
#ifndef W3D_PRE  // Philox blocks computed before the staging wait: 1, 2 or 4
#define W3D_PRE 4
#endif
constexpr int TX = 16, TZ = W3D_TZ, THREADS = 16 * TZ;
// CTAs per SM: 3 (80 registers, 76 KB of staging each: every C3 volume's
// fixed-dims image AND label boxes fit, so both come by TMA; measured 242.6
// GVoxel/s vs 228.3 at 4 CTAs/SM, where 6 of 16 volumes fall back to per-tile
// boxes with cp.async labels)
#ifndef W3D_MINB
#define W3D_MINB (TZ > 16 ? 2 : 3)
#endif
#ifndef W3D_TY
#define W3D_TY 16
#endif
// the gather kernel has no staging buffer: more resident CTAs hide its L2 latency
#ifndef W3D_GMINB
#define W3D_GMINB 4  // C4 gather: 144.7 GVoxel/s at 4 (64 registers) vs 140.4 at 3, 124.2 at 6
#endif
constexpr int kTY = W3D_TY, kMinB = W3D_MINB, kGMinB = W3D_GMINB;
// staging buffer (voxels of 5 B): kMinB * (kCapVox * 5 B + 256 + 1 KB) <= 228 KB
constexpr int kCapVox = (233472 / kMinB - 1024 - 272) / 5;

}  // namespace cube
}  // namespace w3d
