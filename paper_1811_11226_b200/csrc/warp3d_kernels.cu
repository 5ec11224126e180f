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

// Normals of the 4 voxels (rows y = 4g .. 4g+3) of Philox block q (R10).
__device__ __forceinline__ void normals4(uint32_t q, const VolDev& P, float n[4]) {
  const uint4 r = philox4x32_10(make_uint4(q, 0u, P.vid0, P.vid1), P.key0, P.key1);
  const float2 a = box_muller(r.x, r.y);
  const float2 b = box_muller(r.z, r.w);
  n[0] = a.x; n[1] = a.y; n[2] = b.x; n[3] = b.y;
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
// Staged sampling: the CTA's source footprint box is in shared memory with
// `fill` / `label_fill` in its out-of-volume part, so no per-corner predicate is
// needed.  p is clamped to [-1, n] first: a clamped coordinate reads only pad
// voxels or gets weight 0 on in-volume ones, which reproduces the border-fill
// rule (R6) and the label rule (R8) exactly.
// ----------------------------------------------------------------------------
struct StageView {
  const float* img;     // [D][H][W] floats
  const uint8_t* lbl;   // [D][H][W] bytes, same index
  int W, HW;            // row and plane pitch (elements)
  float bx, by, bz;     // box origin (input voxel coords of element 0)
  float Wf, HWf;
  float nx, ny, nz;     // clamp bounds
};

__device__ __forceinline__ Sample sample_staged(const StageView& v, float px, float py, float pz,
                                                bool want_img, bool nearest_img,
                                                bool has_lbl) {
  Sample s;
  px = fminf(fmaxf(px, -1.0f), v.nx);
  py = fminf(fmaxf(py, -1.0f), v.ny);
  pz = fminf(fmaxf(pz, -1.0f), v.nz);
  const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
  const float tx = __fsub_rn(px, fx), ty = __fsub_rn(py, fy), tz = __fsub_rn(pz, fz);
  // local element index: all terms are small integers, exact in fp32
  const float lf = __fmaf_rn(__fsub_rn(fz, v.bz), v.HWf,
                             __fmaf_rn(__fsub_rn(fy, v.by), v.Wf, __fsub_rn(fx, v.bx)));
  const int li = __float2int_rz(lf);
  const int ln = li + (tx >= 0.5f ? 1 : 0) + (ty >= 0.5f ? v.W : 0) + (tz >= 0.5f ? v.HW : 0);
  s.lbl = has_lbl ? v.lbl[ln] : 0u;
  s.img = 0.0f;
  if (!want_img) return s;
  if (nearest_img) {
    s.img = v.img[ln];
    return s;
  }
  const float* b = v.img + li;
  const int W = v.W, HW = v.HW;
  const float c000 = b[0], c100 = b[1], c010 = b[W], c110 = b[W + 1];
  const float c001 = b[HW], c101 = b[HW + 1], c011 = b[HW + W], c111 = b[HW + W + 1];
  const float c00 = lerp(c000, c100, tx), c10 = lerp(c010, c110, tx);
  const float c01 = lerp(c001, c101, tx), c11 = lerp(c011, c111, tx);
  s.img = lerp(lerp(c00, c10, ty), lerp(c01, c11, ty), tz);
  return s;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ----------------------------------------------------------------------------
// Output tile loop shared by both paths.  Thread (lane, warp) of the CTA owns
// output column x = ox + lane at z = oz + warp and the kTY rows oy .. oy+kTY-1,
// i.e. kTY/4 Philox blocks (R10: block = (x, y/4, z), lane = y mod 4).  A warp
// writes 32 consecutive x of one row: 128 B image + 32 B label stores.
// ----------------------------------------------------------------------------
template <bool kStagedPath>
__device__ __forceinline__ void tile_compute(const WarpArgs& a, const VolDev& P,
                                             const float* __restrict__ vin,
                                             const uint8_t* __restrict__ lin,
                                             float* __restrict__ vout,
                                             uint8_t* __restrict__ lout, const StageView& sv,
                                             int ox, int oy, int oz) {
  const int X = ox + static_cast<int>(threadIdx.x & 31);
  const int Z = oz + static_cast<int>(threadIdx.x >> 5);
  if (X >= a.mx || Z >= a.mz) return;
  const float fX = static_cast<float>(X), fZ = static_cast<float>(Z);
  float cz[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) cz[k] = __fmaf_rn(P.A[4 * k + 2], fZ, P.A[4 * k + 3]);
  const bool occluded = (P.flags & kOcclude) && Z >= P.occ_lo && Z <= P.occ_hi;
  const bool nearest_img = a.interp == W3D_INTERP_NEAREST;
  const int Gy = (a.my + 3) >> 2;
  const int64_t zoff = static_cast<int64_t>(Z) * a.mx * a.my + X;
#pragma unroll
  for (int g = 0; g < kTY / 4; ++g) {
    const int Y0 = oy + 4 * g;
    if (Y0 >= a.my) break;
    float n[4] = {0.f, 0.f, 0.f, 0.f};
    if ((P.flags & kNoise) && !occluded) {
      const uint32_t q = static_cast<uint32_t>(X) +
                         static_cast<uint32_t>(a.mx) * static_cast<uint32_t>((Y0 >> 2) + Gy * Z);
      normals4(q, P, n);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int Y = Y0 + k;
      if (Y >= a.my) break;
      const float fY = static_cast<float>(Y);
      const float px = __fmaf_rn(P.A[0], fX, __fmaf_rn(P.A[1], fY, cz[0]));
      const float py = __fmaf_rn(P.A[4], fX, __fmaf_rn(P.A[5], fY, cz[1]));
      const float pz = __fmaf_rn(P.A[8], fX, __fmaf_rn(P.A[9], fY, cz[2]));
      Sample s;
      if (kStagedPath)
        s = sample_staged(sv, px, py, pz, !occluded, nearest_img, lout != nullptr);
      else
        s = sample_gather(a, vin, lin, px, py, pz, !occluded);
      const int64_t o = zoff + static_cast<int64_t>(Y) * a.mx;
      vout[o] = occluded ? 0.0f : photometric(s.img, n[k], P);
      if (lout) lout[o] = static_cast<uint8_t>(s.lbl);
    }
  }
}

// ----------------------------------------------------------------------------
// Kernel: one CTA per kTX x kTY x kTZ output tile; grid = (tiles, volumes),
// tiles x-fastest so CTAs of one volume run together (L2 holds ~1 volume).
// kStage: stage the tile's source footprint (bounding box of the 8 transformed
// tile corners -- exact, because p is monotone in each output coordinate) in
// shared memory with cp.async; tiles whose box exceeds cap_vox gather instead.
// ----------------------------------------------------------------------------
template <bool kStage>
__global__ void __launch_bounds__(kThreads, 4)
    warp3d_tile_kernel(const __grid_constant__ WarpArgs a, const int tiles_x, const int tiles_y,
                       const int cap_vox) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_box[8];
  const int vi = blockIdx.y;
  const VolDev& P = a.vol[vi];
  int t = blockIdx.x;
  const int ox = (t % tiles_x) * kTX;
  t /= tiles_x;
  const int oy = (t % tiles_y) * kTY;
  const int oz = (t / tiles_y) * kTZ;
  const float* __restrict__ vin = a.in + vi * a.in_stride;
  const uint8_t* __restrict__ lin = a.in_lbl ? a.in_lbl + vi * a.in_stride : nullptr;
  float* __restrict__ vout = a.out + vi * a.out_stride;
  uint8_t* __restrict__ lout = a.out_lbl ? a.out_lbl + vi * a.out_stride : nullptr;
  StageView sv;
  if (!kStage) {
    tile_compute<false>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
    return;
  }
  if (threadIdx.x < 32) {
    const int c = threadIdx.x & 7;
    const float X = static_cast<float>((c & 1) ? min(ox + kTX, a.mx) - 1 : ox);
    const float Y = static_cast<float>((c & 2) ? min(oy + kTY, a.my) - 1 : oy);
    const float Z = static_cast<float>((c & 4) ? min(oz + kTZ, a.mz) - 1 : oz);
    float mn[3], mxv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float p = __fmaf_rn(P.A[4 * k], X,
                                __fmaf_rn(P.A[4 * k + 1], Y, __fmaf_rn(P.A[4 * k + 2], Z, P.A[4 * k + 3])));
      mn[k] = p;
      mxv[k] = p;
    }
#pragma unroll
    for (int off = 1; off < 8; off <<= 1)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
        mxv[k] = fmaxf(mxv[k], __shfl_xor_sync(0xffffffffu, mxv[k], off));
      }
    if (threadIdx.x == 0) {
      const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                          static_cast<float>(a.nz)};
      int lo[3], hi[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lo[k] = static_cast<int>(floorf(fminf(fmaxf(mn[k], -1.0f), n[k])));
        hi[k] = static_cast<int>(floorf(fminf(fmaxf(mxv[k], -1.0f), n[k]))) + 1;
      }
      const int x0 = lo[0] >= 0 ? (lo[0] & ~3) : -4;
      const int W = (hi[0] + 1 - x0 + 3) & ~3;
      const int H = hi[1] - lo[1] + 1, D = hi[2] - lo[2] + 1;
      s_box[0] = x0; s_box[1] = lo[1]; s_box[2] = lo[2];
      s_box[3] = W; s_box[4] = H; s_box[5] = D;
      s_box[6] = (static_cast<int64_t>(W) * H * D <= cap_vox) ? 1 : 0;
    }
  }
  __syncthreads();
  if (!s_box[6]) {
    tile_compute<false>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
    return;
  }
  const int bx = s_box[0], by = s_box[1], bz = s_box[2];
  const int W = s_box[3], H = s_box[4], D = s_box[5];
  float* simg = reinterpret_cast<float*>(smem);
  uint8_t* slbl = smem + static_cast<size_t>(cap_vox) * 4;
  {
    // Stage rows of 16 B chunks (4 voxels): in-volume chunks by cp.async (image
    // 16 B + label 4 B), out-of-volume chunks set to fill.  nx % 4 == 0 and
    // x0 % 4 == 0, so a chunk is entirely inside or outside in x.
    const int CW = W >> 2;
    const int total = CW * H * D;
    const float inv_cw = 1.0f / static_cast<float>(CW);
    const float inv_h = 1.0f / static_cast<float>(H);
    const float f = a.fill;
    const uint32_t lf4 = a.label_fill * 0x01010101u;
    for (int i = threadIdx.x; i < total; i += kThreads) {
      // float-reciprocal division, exact: the quotient q = (i + 0.5) / CW has
      // relative error < 2^-22, i.e. absolute < (i + 0.5) 2^-22 / CW, below its
      // distance 0.5 / CW to the nearest integer while i + 0.5 < 2^21.
      const int row = __float2int_rz((static_cast<float>(i) + 0.5f) * inv_cw);
      const int c = i - row * CW;
      const int rz = __float2int_rz((static_cast<float>(row) + 0.5f) * inv_h);
      const int ry = row - rz * H;
      const int gx = bx + 4 * c, gy = by + ry, gz = bz + rz;
      const int li = row * W + 4 * c;
      const bool in = (gx >= 0) & (gx < a.nx) & (gy >= 0) & (gy < a.ny) & (gz >= 0) & (gz < a.nz);
      if (in) {
        const int64_t g = (static_cast<int64_t>(gz) * a.ny + gy) * a.nx + gx;
        cp_async16(simg + li, vin + g);
        if (lin) cp_async4(slbl + li, lin + g);
      } else {
        *reinterpret_cast<float4*>(simg + li) = make_float4(f, f, f, f);
        if (lin) *reinterpret_cast<uint32_t*>(slbl + li) = lf4;
      }
    }
    cp_async_wait_all();
  }
  __syncthreads();
  sv.img = simg;
  sv.lbl = slbl;
  sv.W = W;
  sv.HW = W * H;
  sv.bx = static_cast<float>(bx);
  sv.by = static_cast<float>(by);
  sv.bz = static_cast<float>(bz);
  sv.Wf = static_cast<float>(W);
  sv.HWf = static_cast<float>(W * H);
  sv.nx = static_cast<float>(a.nx);
  sv.ny = static_cast<float>(a.ny);
  sv.nz = static_cast<float>(a.nz);
  tile_compute<true>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
}

static int g_cap_vox = kDefaultCapVox;

int stage_capacity() { return g_cap_vox; }
void set_stage_capacity(int cap) { g_cap_vox = cap; }

static cudaError_t launch_tiles(const WarpArgs& a, bool staged, cudaStream_t s) {
  const int tiles_x = (a.mx + kTX - 1) / kTX, tiles_y = (a.my + kTY - 1) / kTY;
  const int tiles_z = (a.mz + kTZ - 1) / kTZ;
  const int64_t tiles = static_cast<int64_t>(tiles_x) * tiles_y * tiles_z;
  if (tiles >= (int64_t(1) << 31)) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(a.nvol));
  if (staged) {
    const int cap = g_cap_vox;
    const size_t smem = static_cast<size_t>(cap) * 5;
    static size_t configured = 0;
    if (configured != smem) {
      const cudaError_t e = cudaFuncSetAttribute(
          warp3d_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
          static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      configured = smem;
    }
    warp3d_tile_kernel<true><<<grid, kThreads, smem, s>>>(a, tiles_x, tiles_y, cap);
  } else {
    warp3d_tile_kernel<false><<<grid, kThreads, 0, s>>>(a, tiles_x, tiles_y, 0);
  }
  note_launch();
  return cudaGetLastError();
}

bool staged_supported(const WarpArgs& a) {
  return (a.nx % 4 == 0) && (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) &&
         (a.in_stride % 4 == 0) &&
         (a.in_lbl == nullptr || reinterpret_cast<uintptr_t>(a.in_lbl) % 4 == 0);
}

cudaError_t launch_gather(const WarpArgs& a, cudaStream_t s) { return launch_tiles(a, false, s); }

cudaError_t launch_staged(const WarpArgs& a, cudaStream_t s) {
  return launch_tiles(a, staged_supported(a), s);
}

// ----------------------------------------------------------------------------
// Test hooks
// ----------------------------------------------------------------------------
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
  const float2 a = box_muller(w.x, w.y), b = box_muller(w.z, w.w);
  const float nn[4] = {a.x, a.y, b.x, b.y};
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
  const int x = static_cast<int>(v % a.mx);
  const int64_t yz = v / a.mx;
  const int y = static_cast<int>(yz % a.my), z = static_cast<int>(yz / a.my);
  const float X = static_cast<float>(x), Y = static_cast<float>(y), Z = static_cast<float>(z);
  float p[3];
  for (int k = 0; k < 3; ++k)
    p[k] = __fmaf_rn(P.A[4 * k], X, __fmaf_rn(P.A[4 * k + 1], Y, __fmaf_rn(P.A[4 * k + 2], Z,
                                                                          P.A[4 * k + 3])));
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
