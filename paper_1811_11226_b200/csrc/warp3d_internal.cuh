// warp3d_internal.cuh -- launch-argument structs shared by the host entry
// points (warp3d_host.cu) and the kernels (warp3d_kernels.cu).
#pragma once
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
  uint32_t key0, key1;  // Philox key = seed
  uint32_t vid0, vid1;  // Philox counter words 2,3 = volume_id
  int32_t occ_lo, occ_hi;  // occluded output z in [occ_lo, occ_hi]
  uint32_t _pad[2];
  uint32_t rk0[10], rk1[10];  // Philox round keys k + r * (W0, W1), host-precomputed
  uint32_t _pad2[4];
};
static_assert(sizeof(VolDev) == 208, "VolDev layout");

constexpr int kMaxVolPerLaunch = 112;

// TMA staging: the box is loaded with
// cp.async.bulk.tensor boxes of kTmaRowsImg image rows x WI floats and
// kTmaRowsLbl label rows x WL bytes; WI / WL come from these width classes
// (one tensor map per class; WI*kTmaRowsImg*4 and WL*kTmaRowsLbl must be
// multiples of 128 B so consecutive boxes stay 128 B aligned in smem).
constexpr int kTmaRowsImg = 4, kTmaRowsLbl = 8;
constexpr int kNumImgCls = 10, kNumLblCls = 7;
__host__ __device__ constexpr int img_cls_width(int c) {
  return c < 7 ? 16 + 8 * c : (c == 7 ? 80 : (c == 8 ? 96 : 128));
}
__host__ __device__ constexpr int lbl_cls_width(int c) { return c < 6 ? 16 * (c + 1) : 128; }

// Persistent kernel: two buffers of kPersCapVox voxels (5 B each) per SM.
constexpr int kPersCapVox = 11008;  // 2 CTAs/SM x 2 buffers x (55 KB + 1 KB reserve)

struct alignas(64) WarpArgs {
  CUtensorMap tm_img[kNumImgCls];  // 4D (nx, ny, nz, nvol) float32, box (w, 4, 1, 1)
  CUtensorMap tm_lbl[kNumLblCls];  // 4D uint8, box (w, 8, 1, 1)
  int32_t use_tma;                 // tensor maps valid
  int32_t _pad_tma[15];
  const float* in;
  const uint8_t* in_lbl;  // may be null
  float* out;
  uint8_t* out_lbl;       // null iff in_lbl null
  int32_t nx, ny, nz;     // input dims
  int32_t mx, my, mz;     // output dims
  int64_t in_stride;      // voxels per input volume
  int64_t out_stride;     // voxels per output volume
  float fill;
  uint32_t label_fill;
  int32_t interp;         // W3D_INTERP_*
  int32_t nvol;           // volumes in this launch
  VolDev vol[kMaxVolPerLaunch];
};

// Launchers (warp3d_kernels.cu).  All return cudaGetLastError() of the launch.
cudaError_t launch_gather(const WarpArgs& a, cudaStream_t s);
cudaError_t launch_staged(const WarpArgs& a, cudaStream_t s);
cudaError_t launch_auto(const WarpArgs& a, cudaStream_t s);
cudaError_t launch_tma(const WarpArgs& a, cudaStream_t s);
cudaError_t launch_bulk(const WarpArgs& a, cudaStream_t s);
cudaError_t launch_persistent_api(const WarpArgs& a, cudaStream_t s);
bool tma_supported(const WarpArgs& a);
cudaError_t encode_tensor_maps(WarpArgs& a);
cudaError_t launch_noise(float* out, int mx, int my, int mz, float sigma, uint32_t k0,
                         uint32_t k1, uint32_t v0, uint32_t v1, cudaStream_t s);
bool staged_supported(const WarpArgs& a);
cudaError_t read_tile_stats(unsigned long long out[2]);
cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                          int64_t n, cudaStream_t s);
cudaError_t launch_footprint(const WarpArgs& a, uint8_t* marks, cudaStream_t s);
cudaError_t launch_count_marks(const uint8_t* marks, int64_t n, unsigned long long* counts,
                               cudaStream_t s);

void note_launch(int n = 1);

}  // namespace w3d
