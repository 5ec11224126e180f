// warp3d_aux.cu -- test hooks and the measurement helper of the warp3d library:
//   warp3d_noise_kernel     the noise field alone (R10), checked against the oracle
//   warp3d_philox_kernel    raw Philox4x32-10 words (known-answer tests)
//   warp3d_footprint_kernel touched input footprint (algorithmic bytes)
//   warp3d_count_kernel     sum of a byte array
// None of these is on the hot path.
#include <cuda_runtime.h>

#include <cstdint>

#include "philox.cuh"
#include "warp3d_internal.cuh"

namespace w3d {

__global__ void __launch_bounds__(256) warp3d_noise_kernel(float* __restrict__ out, int mx,
                                                           int my, int mz, float sigma,
                                                           uint32_t k0, uint32_t k1,
                                                           uint32_t v0, uint32_t v1) {
  // one thread per Philox block (x, y/4, z) (R10)
  const int Gy = (my + 3) >> 2;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= static_cast<int64_t>(mx) * Gy * mz) return;
  const int x = static_cast<int>(q % mx);
  const int64_t r = q / mx;
  const int gy = static_cast<int>(r % Gy), z = static_cast<int>(r / Gy);
  const uint4 w = philox4x32_10(
      make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), v0, v1), k0, k1);
  const float4 n = box_muller4(w);
  const float nn[4] = {n.x, n.y, n.z, n.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int y = 4 * gy + k;
    if (y < my) out[(static_cast<int64_t>(z) * my + y) * mx + x] = sigma * nn[k];
  }
}

cudaError_t launch_noise(float* out, int mx, int my, int mz, float sigma, uint32_t k0,
                         uint32_t k1, uint32_t v0, uint32_t v1, cudaStream_t s) {
  const int64_t blocks = static_cast<int64_t>(mx) * ((my + 3) / 4) * mz;
  warp3d_noise_kernel<<<static_cast<unsigned>((blocks + 255) / 256), 256, 0, s>>>(
      out, mx, my, mz, sigma, k0, k1, v0, v1);
  note_launch();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) warp3d_philox_kernel(const uint4* __restrict__ ctr,
                                                            uint32_t k0, uint32_t k1,
                                                            uint4* __restrict__ out, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox4x32_10(ctr[i], k0, k1);
}

cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, int64_t n,
                          cudaStream_t s) {
  warp3d_philox_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(ctr), k0, k1, reinterpret_cast<uint4*>(out), n);
  note_launch();
  return cudaGetLastError();
}

// Footprint measurement (not on the hot path): marks[0][vol][in] = 1 for every
// in-volume trilinear corner of a not-fully-OOB sample, marks[1][vol][in] = 1
// for every in-volume nearest voxel.  Same coordinate contract as the warp
// (R4).  Benign races: every writer stores 1.
__global__ void __launch_bounds__(256) warp3d_footprint_kernel(const __grid_constant__ WarpArgs a,
                                                               uint8_t* __restrict__ marks) {
  const int vi = blockIdx.y;
  const VolDev& P = a.vol[vi];
  const int64_t nvox = static_cast<int64_t>(a.mx) * a.my * a.mz;
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nvox) return;
  const int64_t total_in = a.in_stride * a.nvol;
  uint8_t* mimg = marks + vi * a.in_stride;
  uint8_t* mlbl = marks + total_in + vi * a.in_stride;
  const int x = static_cast<int>(v % a.mx);
  const int64_t yz = v / a.mx;
  const int y = static_cast<int>(yz % a.my), z = static_cast<int>(yz / a.my);
  const float X = static_cast<float>(x), Y = static_cast<float>(y), Z = static_cast<float>(z);
  float p[3];
  for (int k = 0; k < 3; ++k)
    p[k] = __fmaf_rn(P.A[4 * k + 1], Y,
                     __fmaf_rn(P.A[4 * k], X, __fmaf_rn(P.A[4 * k + 2], Z, P.A[4 * k + 3])));
  const int n[3] = {a.nx, a.ny, a.nz};
  bool near_in = true, any_in = true;
  int fl[3], r[3];
  for (int k = 0; k < 3; ++k) {
    near_in &= (p[k] >= -0.5f) & (p[k] < static_cast<float>(n[k]) - 0.5f);
    any_in &= (p[k] > -1.0f) & (p[k] < static_cast<float>(n[k]));
  }
  if (near_in) {
    for (int k = 0; k < 3; ++k) {
      const float f = floorf(p[k]);
      r[k] = static_cast<int>(f) + (__fsub_rn(p[k], f) >= 0.5f);
    }
    mlbl[(static_cast<int64_t>(r[2]) * a.ny + r[1]) * a.nx + r[0]] = 1;
  }
  const bool occluded = (P.flags & kOcclude) && z >= P.occ_lo && z <= P.occ_hi;
  if (!any_in || occluded) return;
  if (a.interp == W3D_INTERP_NEAREST) {
    if (near_in) mimg[(static_cast<int64_t>(r[2]) * a.ny + r[1]) * a.nx + r[0]] = 1;
    return;
  }
  for (int k = 0; k < 3; ++k) fl[k] = static_cast<int>(floorf(p[k]));
  for (int c = 0; c < 8; ++c) {
    const int jx = fl[0] + (c & 1), jy = fl[1] + ((c >> 1) & 1), jz = fl[2] + (c >> 2);
    if (jx < 0 || jy < 0 || jz < 0 || jx >= a.nx || jy >= a.ny || jz >= a.nz) continue;
    mimg[(static_cast<int64_t>(jz) * a.ny + jy) * a.nx + jx] = 1;
  }
}

cudaError_t launch_footprint(const WarpArgs& a, uint8_t* marks, cudaStream_t s) {
  const int64_t nvox = static_cast<int64_t>(a.mx) * a.my * a.mz;
  const dim3 grid(static_cast<unsigned>((nvox + 255) / 256), static_cast<unsigned>(a.nvol));
  warp3d_footprint_kernel<<<grid, 256, 0, s>>>(a, marks);
  note_launch();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) warp3d_count_kernel(const uint8_t* __restrict__ marks,
                                                           int64_t n,
                                                           unsigned long long* counts) {
  unsigned long long acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc += marks[i];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(counts, acc);
}

cudaError_t launch_count_marks(const uint8_t* marks, int64_t n, unsigned long long* counts,
                               cudaStream_t s) {
  warp3d_count_kernel<<<148 * 8, 256, 0, s>>>(marks, n, counts);
  note_launch();
  return cudaGetLastError();
}

}  // namespace w3d
