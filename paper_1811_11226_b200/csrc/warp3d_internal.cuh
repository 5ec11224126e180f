// warp3d_internal.cuh -- launch-argument structs shared by the host entry
// points (warp3d_host.cu) and the kernels (warp3d_cube.cu, warp3d_aux.cu).
#pragma once
#include <cstddef>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "warp3d.h"

namespace w3d {

// Effective per-volume flags after host-side simplification.
enum : uint32_t {
  kNoise = 1u,    // sigma > 0
  kWindow = 2u,
  kClamp = 4u,
  kGamma = 8u,    // gamma != 1
  kOcclude = 16u  // non-empty integer z range
};

// Per-volume parameters as the kernels see them (derived on the host from
// w3d_volume_params).  Disabled photometric
// steps get neutral values, so the kernel evaluates the chain branch-free:
//   v = fma(sigma, n, v); w = fma(v, win_s, win_off); w = min(max(w, lo), hi);
//   out = (flags & kGamma) ? w^gamma : w
struct alignas(16) VolDev {
  float A[12];        // [A | b] row-major, R4
  uint32_t flags;     // kNoise (sigma > 0) | kGamma (gamma != 1) | kOcclude
  float sigma;        // HU; 0 without NOISE
  float win_s;        // fp32(1 / (b - a)); 1 without WINDOW
  float win_off;      // fp32(-a * s);      0 without WINDOW
  float clamp_lo;     // 0 with CLAMP, else -inf
  float clamp_hi;     // 1 with CLAMP, else +inf
  float gamma;
  // cp.async staging box of this volume's tiles (host-computed from A,
  // cube_cp_box): tiles in y-parts of cp_rows rows (kTY, kTY/2 or kTY/4; 0 =
  // the footprint does not fit: per-tile boxes / gathers), box cp_w x cp_h x
  // cp_d elements with plane pitch cp_p, origin as the TMA box (box_mlo)
  uint16_t cp_w, cp_h, cp_d, cp_rows;
  int32_t cp_p;
  uint16_t cp_w_bytes, cp_p_bytes;  // cp_w, cp_p in bytes of the image element type
  int32_t occ_lo, occ_hi;  // occluded output z in [occ_lo, occ_hi]
  // TMA boxes of this volume's tiles: box_w != 0 when tm[2 vi] holds the image
  // map (box cp_w x cp_h x cp_d); box_wl != 0 when tm[2 vi + 1] holds the label
  // map (box box_wl x box_h x cp_d bytes), else the labels go by cp.async
  uint16_t box_w, box_h, box_d, box_wl;
  uint32_t rk0[10], rk1[10];  // Philox round keys k + r * (W0, W1), host-precomputed
  uint32_t ph_K0, ph_K1, ph_K2, ph_U3;  // PhiloxPrefix (philox.cuh), host-precomputed
  // box origin of a full tile (TMA and cp.async): floor(p(tile origin voxel) +
  // box_mlo[k]) with box_mlo[k] = sum_j min(0, A_kj span_j) - rounding margin
  // (cube_box_mlo); a y-part of r rows adds -min(0, A_k1) (kTY - r)
  float box_mlo[3];
  // fix-up test of a full tile: every trilinear corner and nearest voxel lies
  // inside the volume iff floor(p0 + box_mlo[k]) >= 0 and p0 + box_mhi[k] <
  // n_k - 1 (box_mhi[k] = sum_j max(0, A_kj span_j) + the same margin)
  float box_mhi[3];
  int32_t cp_abs;       // cp_rows != 0 only with 1: the staged index kM + fx + W fy + P fz
                        // (absolute volume coordinates) is exact for every tile not
                        // entirely outside the volume (cube_cp_box)
  int32_t out_slot;     // output volume index in the caller's batch (out + slot * out_stride)
  uint64_t in_addr;     // device address of this volume's image (float32 or int16)
  uint64_t lbl_addr;    // device address of its labels (0 without labels)
};
static_assert(sizeof(VolDev) == 256, "VolDev layout");

constexpr int kMaxVolPerLaunch = 104;  // sizeof(WarpArgs) < 32764 B of kernel parameters
// Volumes per launch when TMA staging is used: the tensor maps must lie in the
// first 4 KB of the kernel parameters (measured: TMA on a __grid_constant__
// map at a larger parameter offset faults).
constexpr int kTmaVolPerLaunch = 16;

// NV = volumes the parameter block holds.  Launches of at most kSmallVol
// volumes pass WarpArgsT<kSmallVol> (~8.4 KB of parameters instead of ~31 KB:
// the launch's parameter upload costs ~2.5 us more at 31 KB,
// tools/probes/param_probe.cu); the kernels read it through the WarpArgs prefix
// (same layout up to vol[NV], vol last) and never index past nvol <= NV.
template <int NV>
struct alignas(64) WarpArgsT {
  // per volume i: tm[2i] 3D (nx, ny, nz) image map (float32 or int16), box
  // (cp_w, cp_h, cp_d); tm[2i+1] uint8 label map, box (box_wl, box_h, cp_d)
  CUtensorMap tm[2 * kTmaVolPerLaunch];
  const float* in;        // non-null: float32 image input (per-volume addresses in vol[i])
  const int16_t* in16;    // non-null: int16 HU image input (NEXT-4)
  const uint8_t* in_lbl;  // may be null
  float* out;
  uint8_t* out_lbl;       // null iff in_lbl null
  int32_t nx, ny, nz;     // input dims
  int32_t mx, my, mz;     // output dims
  int64_t in_stride;      // voxels per input volume
  int64_t out_stride;     // voxels per output volume
  int64_t out_row_bytes;  // 4 * mx: the float output row pitch in bytes, and mx: the
  int64_t out_lrow_bytes; // label row pitch (kernel parameters, so the per-row pointer
                          // steps are plain 64-bit adds of a parameter, not IMAD.WIDE)
  float fill;
  uint32_t label_fill;
  uint32_t fill16_pair;   // int16 input: (int16)fill in both halves (staged boxes)
  int32_t interp;         // W3D_INTERP_*
  int32_t nvol;           // volumes in this launch
  int32_t use_tma;        // tensor maps valid for the volumes with box_w > 0
  int32_t in_aligned;     // every volume's image (labels) 16 B (8 B) aligned: staged paths
  int32_t pdl;            // host only: launch as a programmatic dependent of the previous
                          // chunk of the same call (independent volumes: no data dependency)
  int32_t tile_rows;      // output rows per tile (kTY = 16, or 8 for launches whose
                          // 16-row boxes do not fit: large rotations, AUTO); the
                          // per-volume boxes and offsets are computed for it
  int32_t brick;          // 0, or the tile order in bricks of 2^sx x 2^sy x 2^sz tiles
                          // (bit 31 set; sx, sy, sz, log2 bricks per row / column in
                          // 4-bit fields from bit 0): consecutive CTAs cover compact
                          // output regions, so a wave's input footprint stays in L2
  int32_t prefetch_ahead; // > 0: each CTA of the fixed-box path also prefetches into L2
                          // the boxes of the tile this many CTAs later in launch order
                          // (same volume; 8-row launches, W3D_PREFETCH)
  // Philox round keys shared by every volume of the launch (all seeds equal;
  // required by the kPhFull kernels: fixed parameter offsets, so the round
  // function reads them as constant-bank operands)
  uint32_t rk0[10], rk1[10];
  VolDev vol[NV];
};
using WarpArgs = WarpArgsT<kMaxVolPerLaunch>;
constexpr int kSmallVol = 16;
using WarpArgsSmall = WarpArgsT<kSmallVol>;
static_assert(sizeof(WarpArgs) <= 32764, "kernel parameter space");
static_assert(offsetof(WarpArgs, vol) == offsetof(WarpArgsSmall, vol), "WarpArgs prefix layout");

// Launchers.  All return cudaGetLastError() of the launch.
// warp3d_cube.cu (the warp): cube_supported() = the staged layout requirements.
bool cube_supported(const WarpArgs& a);
bool cube_tma_supported(const WarpArgs& a);
// staging box (TMA image box and cp.async boxes) of one volume's tiles and its
// origin offsets (out = output dims x, y, z: the rounding margin scales with
// the largest |p|)
void cube_cp_box(const float A[12], VolDev& P, int elem_bytes, const int in[3], const int out[3],
                 int tile_rows);
cudaError_t launch_cube(const WarpArgs& a, bool gather_only, cudaStream_t s);
cudaError_t read_cube_stats(unsigned long long out[4]);
// warp3d_resample.cu (NEXT-3): one separable Gaussian pass along `axis` (0 x, 1 y, 2 z)
constexpr int kMaxTaps = 63;  // radius ceil(3 sigma) <= 31
int gauss_radius(double sigma);
cudaError_t launch_smooth_axis(int axis, const float* in, float* out, int nx, int ny, int nz,
                               double sigma, cudaStream_t s);
// all three passes in one kernel (radius <= 8 per axis), bit-identical to the passes
bool smooth_fusable(const double sigma[3]);
// mask (optional): 3 x kSmoothMaskMax / 32 words, bit i of axis k (x, y, z) set = output
// coordinate i is needed; the others are neither computed nor stored (dims <= kSmoothMaskMax)
constexpr int kSmoothMaskMax = 4096;
cudaError_t launch_smooth_fused(const float* in, float* out, int nx, int ny, int nz,
                                const double sigma[3], cudaStream_t s,
                                const uint32_t* mask = nullptr);
// warp3d_aux.cu (test hooks, measurement)
cudaError_t launch_noise(float* out, int mx, int my, int mz, float sigma, uint32_t k0,
                         uint32_t k1, uint32_t v0, uint32_t v1, cudaStream_t s);
cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                          int64_t n, cudaStream_t s);
cudaError_t launch_footprint(const WarpArgs& a, uint8_t* marks, cudaStream_t s);
cudaError_t launch_count_marks(const uint8_t* marks, int64_t n, unsigned long long* counts,
                               cudaStream_t s);

void note_launch(int n = 1);

}  // namespace w3d
