// warp3d_kernels.cu -- sm_100a kernels of the Sec. IV augmentation path
// (Rister et al., arXiv 1811.11226).
//
// One pass per output voxel, in the paper's order:
//   occlusion test -> p = A x + b -> image/label sample -> noise -> window -> gamma
// The arithmetic contract is DESIGN.md readings R1-R21.  Compiled without
// fast-math and with -fmad=false: every FMA below is an explicit __fmaf_rn.
#include <cuda_runtime.h>

#include <cstdint>

#include "philox.cuh"
#include "warp3d_internal.cuh"

namespace w3d {

// ----------------------------------------------------------------------------
// Shared per-voxel pieces
// ----------------------------------------------------------------------------

// lerp(a, b, t) = a + t (b - a), one rounding for the difference, one FMA (R5).
__device__ __forceinline__ float lerp(float a, float b, float t) {
  return __fmaf_rn(t, __fsub_rn(b, a), a);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Photometric tail for one voxel (PAPER.md:440-467 + gamma, R9-R14).
// n is the standard normal of this voxel (ignored without kNoise).
__device__ __forceinline__ float photometric(float v, float n, const VolDev& P) {
  const uint32_t f = P.flags;
  if (f & kNoise) v = __fmaf_rn(P.sigma, n, v);
  if (f & kWindow) {
    v = __fmaf_rn(v, P.win_s, P.win_off);  // (v - a) / (b - a)
    if (f & kClamp) v = __saturatef(v);    // min(max(., 0), 1)
  }
  if (f & kGamma) v = ex2_approx(P.gamma * lg2_approx(v));  // w^gamma on [0,1]
  return v;
}

// Normals for the 4 voxels of Philox block q (lanes 0..3, R10).
__device__ __forceinline__ void normals4(uint32_t q, const VolDev& P, float n[4]) {
  const uint4 r = philox4x32_10(make_uint4(q, 0u, P.vid0, P.vid1), P.key0, P.key1);
  const float2 a = box_muller(r.x, r.y);
  const float2 b = box_muller(r.z, r.w);
  n[0] = a.x; n[1] = a.y; n[2] = b.x; n[3] = b.y;
}

// p_k = fma(A_k0, x, fma(A_k1, y, fma(A_k2, z, b_k))) (R4).  The (y, z) part is
// the row base: the caller hoists it and adds A_k0 * x with one FMA per axis.
__device__ __forceinline__ void row_base(const VolDev& P, float Y, float Z, float rb[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    rb[k] = __fmaf_rn(P.A[4 * k + 1], Y, __fmaf_rn(P.A[4 * k + 2], Z, P.A[4 * k + 3]));
}

// ----------------------------------------------------------------------------
// Gather sampling: corners read through L1/L2 with per-corner bounds (R6).
// ----------------------------------------------------------------------------
struct Sample {
  float img;
  uint32_t lbl;
};

__device__ __forceinline__ Sample sample_gather(const WarpArgs& a, const float* __restrict__ vin,
                                                const uint8_t* __restrict__ lin, float px,
                                                float py, float pz, bool want_img) {
  Sample s;
  s.img = a.fill;
  s.lbl = a.label_fill;
  const float fnx = static_cast<float>(a.nx), fny = static_cast<float>(a.ny),
              fnz = static_cast<float>(a.nz);
  const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
  const float tx = __fsub_rn(px, fx), ty = __fsub_rn(py, fy), tz = __fsub_rn(pz, fz);
  // nearest (R7): floor(p) + (frac >= 0.5); in bounds iff -0.5 <= p < n - 0.5 (R8)
  const bool near_in = (px >= -0.5f) & (px < fnx - 0.5f) & (py >= -0.5f) & (py < fny - 0.5f) &
                       (pz >= -0.5f) & (pz < fnz - 0.5f);
  int64_t near_idx = 0;
  if (near_in) {
    const int rx = static_cast<int>(fx) + (tx >= 0.5f);
    const int ry = static_cast<int>(fy) + (ty >= 0.5f);
    const int rz = static_cast<int>(fz) + (tz >= 0.5f);
    near_idx = (static_cast<int64_t>(rz) * a.ny + ry) * a.nx + rx;
    if (lin) s.lbl = __ldg(lin + near_idx);
  }
  if (!want_img) return s;
  if (a.interp == W3D_INTERP_NEAREST) {
    if (near_in) s.img = __ldg(vin + near_idx);
    return s;
  }
  // fully out of bounds (every corner outside) -> fill, NaN-safe (R6)
  const bool any_in = (px > -1.0f) & (px < fnx) & (py > -1.0f) & (py < fny) & (pz > -1.0f) &
                      (pz < fnz);
  if (!any_in) return s;
  const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
  const bool x0 = ix >= 0, x1 = ix + 1 < a.nx;
  const bool y0 = iy >= 0, y1 = iy + 1 < a.ny;
  const bool z0 = iz >= 0, z1 = iz + 1 < a.nz;
  const int64_t sy = a.nx, sz = static_cast<int64_t>(a.nx) * a.ny;
  const float* b = vin + (static_cast<int64_t>(iz) * sz + static_cast<int64_t>(iy) * sy + ix);
  const float f = a.fill;
  const float c000 = (x0 & y0 & z0) ? __ldg(b) : f;
  const float c100 = (x1 & y0 & z0) ? __ldg(b + 1) : f;
  const float c010 = (x0 & y1 & z0) ? __ldg(b + sy) : f;
  const float c110 = (x1 & y1 & z0) ? __ldg(b + sy + 1) : f;
  const float c001 = (x0 & y0 & z1) ? __ldg(b + sz) : f;
  const float c101 = (x1 & y0 & z1) ? __ldg(b + sz + 1) : f;
  const float c011 = (x0 & y1 & z1) ? __ldg(b + sz + sy) : f;
  const float c111 = (x1 & y1 & z1) ? __ldg(b + sz + sy + 1) : f;
  const float c00 = lerp(c000, c100, tx), c10 = lerp(c010, c110, tx);
  const float c01 = lerp(c001, c101, tx), c11 = lerp(c011, c111, tx);
  s.img = lerp(lerp(c00, c10, ty), lerp(c01, c11, ty), tz);
  return s;
}

// ----------------------------------------------------------------------------
// Kernel 1: gather.  One thread = one Philox block = 4 consecutive output
// voxels (v = 4q .. 4q+3).  grid = (quads / 256, volumes).
// kAligned: mx % 4 == 0 and 16 B aligned outputs -> the 4 voxels are one
// x-run of one row: hoisted row base, 16 B image store, 4 B label store.
// ----------------------------------------------------------------------------
template <bool kAligned>
__global__ void __launch_bounds__(256) warp3d_gather_kernel(const __grid_constant__ WarpArgs a) {
  const int vi = blockIdx.y;
  const VolDev& P = a.vol[vi];
  const int64_t nvox = static_cast<int64_t>(a.mx) * a.my * a.mz;
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (static_cast<int64_t>(q) * 4 >= nvox) return;

  const float* __restrict__ vin = a.in + vi * a.in_stride;
  const uint8_t* __restrict__ lin = a.in_lbl ? a.in_lbl + vi * a.in_stride : nullptr;
  float* __restrict__ vout = a.out + vi * a.out_stride;
  uint8_t* __restrict__ lout = a.out_lbl ? a.out_lbl + vi * a.out_stride : nullptr;

  float n[4] = {0.f, 0.f, 0.f, 0.f};
  if (P.flags & kNoise) normals4(q, P, n);

  if (kAligned) {
    const uint32_t v0 = q * 4u;
    const uint32_t x0 = v0 % static_cast<uint32_t>(a.mx);
    const uint32_t yz = v0 / static_cast<uint32_t>(a.mx);
    const uint32_t y = yz % static_cast<uint32_t>(a.my), z = yz / static_cast<uint32_t>(a.my);
    const bool occluded = (P.flags & kOcclude) && static_cast<int>(z) >= P.occ_lo &&
                          static_cast<int>(z) <= P.occ_hi;
    float rb[3];
    row_base(P, static_cast<float>(y), static_cast<float>(z), rb);
    float o[4];
    uint32_t l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float X = static_cast<float>(x0 + j);
      const float px = __fmaf_rn(P.A[0], X, rb[0]);
      const float py = __fmaf_rn(P.A[4], X, rb[1]);
      const float pz = __fmaf_rn(P.A[8], X, rb[2]);
      const Sample s = sample_gather(a, vin, lin, px, py, pz, !occluded);
      o[j] = occluded ? 0.0f : photometric(s.img, n[j], P);
      l[j] = s.lbl;
    }
    reinterpret_cast<float4*>(vout)[q] = make_float4(o[0], o[1], o[2], o[3]);
    if (lout)
      reinterpret_cast<uint32_t*>(lout)[q] = l[0] | (l[1] << 8) | (l[2] << 16) | (l[3] << 24);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t v = static_cast<int64_t>(q) * 4 + j;
      if (v >= nvox) break;
      const uint32_t x = static_cast<uint32_t>(v % a.mx);
      const uint32_t yz = static_cast<uint32_t>(v / a.mx);
      const uint32_t y = yz % static_cast<uint32_t>(a.my), z = yz / static_cast<uint32_t>(a.my);
      const bool occluded = (P.flags & kOcclude) && static_cast<int>(z) >= P.occ_lo &&
                            static_cast<int>(z) <= P.occ_hi;
      float rb[3];
      row_base(P, static_cast<float>(y), static_cast<float>(z), rb);
      const float X = static_cast<float>(x);
      const float px = __fmaf_rn(P.A[0], X, rb[0]);
      const float py = __fmaf_rn(P.A[4], X, rb[1]);
      const float pz = __fmaf_rn(P.A[8], X, rb[2]);
      const Sample s = sample_gather(a, vin, lin, px, py, pz, !occluded);
      vout[v] = occluded ? 0.0f : photometric(s.img, n[j], P);
      if (lout) lout[v] = static_cast<uint8_t>(s.lbl);
    }
  }
}

cudaError_t launch_gather(const WarpArgs& a, cudaStream_t s) {
  const int64_t nvox = static_cast<int64_t>(a.mx) * a.my * a.mz;
  const int64_t quads = (nvox + 3) / 4;
  const dim3 grid(static_cast<unsigned>((quads + 255) / 256), static_cast<unsigned>(a.nvol));
  const bool aligned = (a.mx % 4 == 0) && (reinterpret_cast<uintptr_t>(a.out) % 16 == 0) &&
                       (a.out_lbl == nullptr || reinterpret_cast<uintptr_t>(a.out_lbl) % 4 == 0);
  if (aligned)
    warp3d_gather_kernel<true><<<grid, 256, 0, s>>>(a);
  else
    warp3d_gather_kernel<false><<<grid, 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_staged(const WarpArgs& a, cudaStream_t s) {
  return launch_gather(a, s);  // replaced by the staged kernel
}

// ----------------------------------------------------------------------------
// Test hooks
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) warp3d_noise_kernel(float* __restrict__ out, int64_t n,
                                                           float sigma, uint32_t k0, uint32_t k1,
                                                           uint32_t v0, uint32_t v1) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q * 4 >= n) return;
  float nn[4];
  const uint4 r = philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32),
                                           v0, v1), k0, k1);
  const float2 a = box_muller(r.x, r.y), b = box_muller(r.z, r.w);
  nn[0] = a.x; nn[1] = a.y; nn[2] = b.x; nn[3] = b.y;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (q * 4 + j < n) out[q * 4 + j] = sigma * nn[j];
}

cudaError_t launch_noise(float* out, int64_t n, float sigma, uint32_t k0, uint32_t k1,
                         uint32_t v0, uint32_t v1, cudaStream_t s) {
  const int64_t quads = (n + 3) / 4;
  warp3d_noise_kernel<<<static_cast<unsigned>((quads + 255) / 256), 256, 0, s>>>(out, n, sigma, k0,
                                                                               k1, v0, v1);
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

// ----------------------------------------------------------------------------
// Footprint measurement (not on the hot path): marks[0][vol][in] = 1 for every
// in-volume trilinear corner of a not-fully-OOB sample, marks[1][vol][in] = 1
// for every in-volume nearest voxel.  Benign races: every writer stores 1.
// ----------------------------------------------------------------------------
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
  const uint32_t x = static_cast<uint32_t>(v % a.mx);
  const uint32_t yz = static_cast<uint32_t>(v / a.mx);
  const uint32_t y = yz % static_cast<uint32_t>(a.my), z = yz / static_cast<uint32_t>(a.my);
  float rb[3];
  row_base(P, static_cast<float>(y), static_cast<float>(z), rb);
  const float X = static_cast<float>(x);
  const float p[3] = {__fmaf_rn(P.A[0], X, rb[0]), __fmaf_rn(P.A[4], X, rb[1]),
                      __fmaf_rn(P.A[8], X, rb[2])};
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
  const bool occluded = (P.flags & kOcclude) && static_cast<int>(z) >= P.occ_lo &&
                        static_cast<int>(z) <= P.occ_hi;
  if (!any_in || occluded) return;
  for (int k = 0; k < 3; ++k) fl[k] = static_cast<int>(floorf(p[k]));
  for (int c = 0; c < 8; ++c) {
    const int jx = fl[0] + (c & 1), jy = fl[1] + ((c >> 1) & 1), jz = fl[2] + (c >> 2);
    if (jx < 0 || jy < 0 || jz < 0 || jx >= a.nx || jy >= a.ny || jz >= a.nz) continue;
    if (a.interp == W3D_INTERP_NEAREST) continue;
    mimg[(static_cast<int64_t>(jz) * a.ny + jy) * a.nx + jx] = 1;
  }
  if (a.interp == W3D_INTERP_NEAREST && near_in) {
    mimg[(static_cast<int64_t>(r[2]) * a.ny + r[1]) * a.nx + r[0]] = 1;
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
