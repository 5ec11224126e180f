// warp3d_resample.cu -- resampling to r mm before the network (Rister et al.,
// arXiv 1811.11226, Sec. V.A):
// Gaussian lowpass g(x) ~ exp(-sum_k x_k^2 / sigma_k^2), sigma_k = (1/3)
// max(r/u_k - 1, 0), then interpolation at spacing r
// (trilinear image, nearest labels; labels are never smoothed).
//
// The 3D kernel is a product of 1D factors, so the smoothing runs as separable
// passes x, y, z (each an HBM-streaming stencil: every output voxel reads its
// 2R+1 neighbours along one axis through L1/L2, edge voxels replicated, fp32
// accumulation in tap order), and the interpolation is the warp kernel with a
// centre-aligned scale-only affine (warp3d_cube.cu).  Readings R22-R25.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "warp3d_internal.cuh"

namespace w3d {

namespace {

struct Taps {
  float w[kMaxTaps];  // w[0 .. 2R] for offsets -R .. R, normalised (sum 1 in double)
  int32_t R;
};

// out(x, y, z) = sum_t w[t] in(.., clamp(c + t - R), ..) along `Axis`.  One
// thread per output voxel, x fastest (coalesced for every axis).
template <int Axis>
__global__ void __launch_bounds__(256) smooth_axis_kernel(const float* __restrict__ in,
                                                          float* __restrict__ out, int nx, int ny,
                                                          int nz, const __grid_constant__ Taps t) {
  const int x = static_cast<int>(blockIdx.x) * 256 + static_cast<int>(threadIdx.x);
  const int y = static_cast<int>(blockIdx.y), z = static_cast<int>(blockIdx.z);
  if (x >= nx) return;
  const int n = Axis == 0 ? nx : (Axis == 1 ? ny : nz);
  const int c = Axis == 0 ? x : (Axis == 1 ? y : z);
  const int64_t stride = Axis == 0 ? 1 : (Axis == 1 ? int64_t(nx) : int64_t(nx) * ny);
  const int64_t base = (static_cast<int64_t>(z) * ny + y) * nx + x - int64_t(c) * stride;
  float acc = 0.0f;
  for (int k = 0; k <= 2 * t.R; ++k) {
    int j = c + k - t.R;
    j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
    acc = __fmaf_rn(t.w[k], __ldg(in + base + int64_t(j) * stride), acc);
  }
  out[(static_cast<int64_t>(z) * ny + y) * nx + x] = acc;
}

// Fused separable smoothing, z-marching (2.5D): a CTA owns a 32 x 8 NYT column of
// outputs and walks MZ output planes along z.  Each input plane's tile plus its x/y halo (edge voxels replicated by
// clamped coordinates) streams into a ring of shared-memory stages by cp.async,
// kStages - 1 planes ahead of the compute; per plane the x pass runs over the
// halo rows (shared memory -> shared memory), the y pass gives each thread its
// (x, y) value, and the z pass runs in registers over a window of the last
// 2 RM + 1 planes (the plane loop unrolled by 2 RM + 1, so the window is a fixed
// set of register slots).  The x pass reads 16 B words (4 outputs per thread)
// and writes one of two buffers, so the x pass of plane i and the y / z passes
// of plane i - 1 share one barrier interval.  Same passes, order and fp32 FMAs
// as smooth_axis_kernel (bit-identical results); HBM sees one read (+ the z
// halo of 2 RM planes per run) and one write per voxel.
#ifndef W3D_SM_STAGES
#define W3D_SM_STAGES 4
#endif
#ifndef W3D_SM_NYT2  // rows per thread at radius <= 2 (the 1 mm -> 3 mm case)
#define W3D_SM_NYT2 4
#endif
#ifndef W3D_SM_MZ
#define W3D_SM_MZ 64
#endif
#ifndef W3D_SM_THREADS  // threads per CTA (warps = rows of 32 columns x NYT)
#define W3D_SM_THREADS 256
#endif
#ifndef W3D_SM_MINB  // __launch_bounds__ minimum CTAs per SM (register cap)
#define W3D_SM_MINB 1
#endif
constexpr int kFuseR = 8, MX = 32, MZ = W3D_SM_MZ, kStages = W3D_SM_STAGES,
              kSmoothMaskWords = kSmoothMaskMax / 32,
              kSmThreads = W3D_SM_THREADS;
// planes loaded ahead of the compute; x-result buffers (two planes per barrier --
// four buffers, kStages - 2 ahead -- measured slower, profiles/round2/HISTORY.md)
constexpr int kLook = kStages - 1, kXBuf = 2;
struct Taps3 {
  float wx[2 * kFuseR + 1], wy[2 * kFuseR + 1], wz[2 * kFuseR + 1];
  int32_t rx, ry, rz;
  // optional output mask (warp3d_resample: only the voxels the 3 mm grid's trilinear
  // corners read are computed and stored): bit i of mask[k] = coordinate i of axis k
  int32_t masked;
  uint32_t mask[3][kSmoothMaskWords];
};

extern __shared__ __align__(128) float fuse_smem[];

__device__ __forceinline__ void cp_async4(float* s, const float* g) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(float* s, const float* g) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// ld.shared.v4 as written: the compiler narrows a float4 load whose outer words
// are unused to LDS.64 pieces, and two rows' LDS.64 halves (160 B apart) share
// banks -- a 2-way conflict the full-width load does not have.
__device__ __forceinline__ void lds128(const float* p, float* v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
      : "r"(a));
}

// RM: compile-time tap radius >= every axis' radius; an axis with a smaller
// radius has its weights centred and zero-padded (fma(0, v, acc) = acc exactly,
// so the result equals the per-axis passes bit for bit).  NYT: output rows per
// thread (warp w owns rows NYT w .. NYT w + NYT - 1 of the MY = 8 NYT rows).
// f(i0 + U, integral_constant<U>) for U = 0 .. P-1 while i0 + U < n (compile-time slots)
template <typename F, int... U>
__device__ __forceinline__ void for_each_slot(F& f, int i0, int n, std::integer_sequence<int, U...>) {
  ((i0 + U < n ? f(i0 + U, std::integral_constant<int, U>()) : void()), ...);
}

template <int RM, int NYT>
__global__ void __launch_bounds__(kSmThreads, W3D_SM_MINB)
    smooth_fused_kernel(const float* __restrict__ in, float* __restrict__ out, int nx, int ny, int nz,
                        const __grid_constant__ Taps3 t) {
  constexpr int NT = kSmThreads, NW = NT / 32;
  constexpr int MYT = NW * NYT;
  // plane tile: x range [ox - XP, ox + 32 + XP) (16 B aligned chunks), y halo RM
  constexpr int XP = RM <= 4 ? 4 : 8;
  constexpr int AX = MX + 2 * XP, AY = MYT + 2 * RM, PL = AX * AY;
  constexpr int CX = AX / 4, PC = CX * AY;   // 16 B chunks per row / plane
  constexpr int kPer = (PL + NT - 1) / NT;   // elements per thread (edge tiles)
  constexpr int kPerC = (PC + NT - 1) / NT;  // chunks per thread (interior tiles)
  constexpr int P = 2 * RM + 1;              // z window; the plane loop's unroll
  constexpr int NL = (XP + RM + 4 + 3) / 4;  // 16 B words per x-pass thread
  float* X = fuse_smem + kStages * PL;       // [kXBuf][AY][MX] x-pass results
  float wx[2 * RM + 1], wy[2 * RM + 1], wz[2 * RM + 1];
#pragma unroll
  for (int k = 0; k <= 2 * RM; ++k) {
    wx[k] = (k >= RM - t.rx && k <= RM + t.rx) ? t.wx[k - (RM - t.rx)] : 0.0f;
    wy[k] = (k >= RM - t.ry && k <= RM + t.ry) ? t.wy[k - (RM - t.ry)] : 0.0f;
    wz[k] = (k >= RM - t.rz && k <= RM + t.rz) ? t.wz[k - (RM - t.rz)] : 0.0f;
  }
  const int lx = static_cast<int>(threadIdx.x & 31), w = static_cast<int>(threadIdx.x >> 5);
  // x pass: 8 threads per row (4 outputs each), 32 rows per sweep
  const int xr = static_cast<int>(threadIdx.x) >> 3, xj = static_cast<int>(threadIdx.x) & 7;
  const size_t plane = static_cast<size_t>(nx) * static_cast<size_t>(ny);
  float ring[NYT][2 * RM + 1];  // z window: slot i mod P holds the y-pass value of plane i
#pragma unroll
  for (int q = 0; q < NYT; ++q)
#pragma unroll
    for (int k = 0; k <= 2 * RM; ++k) ring[q][k] = 0.0f;

  {
    const int ox = static_cast<int>(blockIdx.x) * MX, oy = static_cast<int>(blockIdx.y) * MYT,
              oz = static_cast<int>(blockIdx.z) * MZ;
    const int nout = min(MZ, nz - oz);
    const int nin = nout + 2 * RM;  // input planes oz - RM + i, i < nin
    // interior in x (whole aligned chunks inside the rows): 16 B copies, else 4 B
    // copies of clamped coordinates (edge replication)
    const bool chunked = ox - XP >= 0 && ox + MX + XP <= nx && (nx & 3) == 0 &&
                         (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    int soff[kPer];
    uint32_t goff[kPer];
    if (chunked) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int e = static_cast<int>(threadIdx.x) + NT * j;  // chunk index
        const int r = e / CX, c = e - r * CX;
        const int gy = min(max(oy - RM + r, 0), ny - 1);
        soff[j] = (j < kPerC && e < PC) ? r * AX + 4 * c : -1;
        goff[j] = static_cast<uint32_t>(gy) * static_cast<uint32_t>(nx) +
                  static_cast<uint32_t>(ox - XP + 4 * c);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int e = static_cast<int>(threadIdx.x) + NT * j;
        const int r = e / AX, c = e - r * AX;
        const int gx = min(max(ox - XP + c, 0), nx - 1), gy = min(max(oy - RM + r, 0), ny - 1);
        soff[j] = e < PL ? e : -1;
        goff[j] = static_cast<uint32_t>(gy) * static_cast<uint32_t>(nx) + static_cast<uint32_t>(gx);
      }
    }
    auto load_plane = [&](int i) {
      const int zc = min(max(oz - RM + i, 0), nz - 1);
      const float* src = in + static_cast<size_t>(zc) * plane;
      float* dst = fuse_smem + (i % kStages) * PL;
      if (chunked) {
#pragma unroll
        for (int j = 0; j < kPerC; ++j)
          if (soff[j] >= 0) cp_async16(dst + soff[j], src + goff[j]);
      } else {
#pragma unroll
        for (int j = 0; j < kPer; ++j)
          if (soff[j] >= 0) cp_async4(dst + soff[j], src + goff[j]);
      }
    };
    // prologue: the first kLook planes, one cp.async group each
#pragma unroll
    for (int i = 0; i < kLook; ++i) {
      if (i < nin) load_plane(i);
      cp_async_commit();
    }
    const int gx = ox + lx, gy0 = oy + NYT * w;
    float* po = out + (static_cast<size_t>(oz) * ny + gy0) * nx + gx;
    bool ok[NYT];  // store bounds per row (and the output mask's x / y bits)
    const bool xneed = !t.masked || (gx < nx && ((t.mask[0][gx >> 5] >> (gx & 31)) & 1u));
#pragma unroll
    for (int q = 0; q < NYT; ++q) {
      const int gy = gy0 + q;
      ok[q] = gx < nx && gy < ny && xneed &&
              (!t.masked || ((t.mask[1][gy >> 5] >> (gy & 31)) & 1u));
    }
    // x pass of plane i (its stage) into Xb
    auto xpass = [&](int i, float* Xb) {
      const float* A = fuse_smem + (i % kStages) * PL;
#ifndef W3D_SM_SCALAR_X
      // 4 outputs per thread from NL aligned 16 B loads (the taps of neighbouring
      // outputs overlap: ~1 LDS per output instead of 2 RM + 1); same FMA order
      // per output as the per-axis pass
#pragma unroll
      for (int r0 = 0; r0 < AY; r0 += 4 * NW) {
        const int r = r0 + xr;
        if (r0 + 4 * NW <= AY || r < AY) {
          float v[4 * NL];
#pragma unroll
          for (int l = 0; l < NL; ++l)  // whole 16 B words even where only half is
            lds128(A + r * AX + 4 * xj + 4 * l, v + 4 * l);  // used: no bank conflicts
          float o[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float acc = 0.0f;
#pragma unroll
            for (int k = 0; k <= 2 * RM; ++k) acc = __fmaf_rn(wx[k], v[c + k + XP - RM], acc);
            o[c] = acc;
          }
          *reinterpret_cast<float4*>(Xb + r * MX + 4 * xj) = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
#else
      for (int r = w; r < AY; r += NW) {  // A/B knob: one output per thread
        const float* a = A + r * AX + lx + (XP - RM);
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k <= 2 * RM; ++k) acc = __fmaf_rn(wx[k], a[k], acc);
        Xb[r * MX + lx] = acc;
      }
#endif
    };
    // y pass of plane j (x results in Xp) into ring slot S = j mod P, then, once the
    // window is full (j >= 2 RM), its z pass: output plane oz + j - 2 RM
    auto yzpass = [&](int j, auto slot_tag, const float* Xp) {
      constexpr int S = decltype(slot_tag)::value;
      float xv[NYT + 2 * RM];  // y pass: the thread's rows share their x-pass inputs
#pragma unroll
      for (int k = 0; k < NYT + 2 * RM; ++k) xv[k] = Xp[(NYT * w + k) * MX + lx];
#pragma unroll
      for (int q = 0; q < NYT; ++q) {
        float yv = 0.0f;
#pragma unroll
        for (int k = 0; k <= 2 * RM; ++k) yv = __fmaf_rn(wy[k], xv[q + k], yv);
        ring[q][S] = yv;
      }
      // output plane oz + j - 2 RM once the window is full; a masked-out plane skips
      // its z pass and stores (CTA-uniform)
      const int zo = oz + j - 2 * RM;
      if (j >= 2 * RM && (!t.masked || ((t.mask[2][zo >> 5] >> (zo & 31)) & 1u))) {
        float acc[NYT];
#pragma unroll
        for (int q = 0; q < NYT; ++q) {
          acc[q] = 0.0f;
#pragma unroll
          for (int k = 0; k <= 2 * RM; ++k)  // oldest (plane j - 2 RM: slot S + 1) first
            acc[q] = __fmaf_rn(wz[k], ring[q][(S + 1 + k) % P], acc[q]);
        }
        float* pq = po;
#pragma unroll
        for (int q = 0; q < NYT; ++q) {
          if (ok[q]) *pq = acc[q];
          pq += nx;
        }
      }
      if (j >= 2 * RM) po += plane;
    };
    // One barrier per plane: the x pass of plane i (into X buffer i & 1) and the y /
    // z passes of plane i - 1 (from buffer (i - 1) & 1) share a phase.  Behind the
    // barrier of step i: plane i has landed, buffer (i - 1) & 1 is complete, buffer
    // i & 1 was last read by the y pass of plane i - 2 (step i - 1), and the stage
    // the next load overwrites was last read by the x pass of plane i - 1.
    auto plane_step = [&](int i, auto slot_tag) {
      constexpr int u = decltype(slot_tag)::value;  // slot of plane i: u = i mod P
      cp_async_wait<kLook - 1>();
      __syncthreads();
      if (i < nin) xpass(i, X + (i & 1) * (AY * MX));
      if (i + kLook < nin) load_plane(i + kLook);  // into plane i-1's stage
      cp_async_commit();
      if (i >= 1)
        yzpass(i - 1, std::integral_constant<int, (u + P - 1) % P>(),
               X + ((i - 1) & 1) * (AY * MX));
    };
    for (int i0 = 0; i0 <= nin; i0 += P)
      for_each_slot(plane_step, i0, nin + 1, std::make_integer_sequence<int, P>());
  }
}

void make_taps(double sigma, int R, float* w) {
  double d[kMaxTaps], sum = 0.0;
  for (int i = -R; i <= R; ++i) {
    d[i + R] = sigma > 0.0 ? std::exp(-double(i) * double(i) / (sigma * sigma)) : 1.0;
    sum += d[i + R];
  }
  for (int i = 0; i <= 2 * R; ++i) w[i] = static_cast<float>(d[i] / sum);
}

}  // namespace

int gauss_radius(double sigma) { return sigma > 0.0 ? static_cast<int>(std::ceil(3.0 * sigma)) : 0; }

cudaError_t launch_smooth_axis(int axis, const float* in, float* out, int nx, int ny, int nz,
                               double sigma, cudaStream_t s) {
  Taps t;
  t.R = gauss_radius(sigma);
  make_taps(sigma, t.R, t.w);
  const dim3 grid(static_cast<unsigned>((nx + 255) / 256), static_cast<unsigned>(ny),
                  static_cast<unsigned>(nz));
  if (axis == 0)
    smooth_axis_kernel<0><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  else if (axis == 1)
    smooth_axis_kernel<1><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  else
    smooth_axis_kernel<2><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  note_launch();
  return cudaGetLastError();
}

bool smooth_fusable(const double sigma[3]) {
  for (int k = 0; k < 3; ++k)
    if (gauss_radius(sigma[k]) > kFuseR) return false;
  return true;
}

cudaError_t launch_smooth_fused(const float* in, float* out, int nx, int ny, int nz,
                                const double sigma[3], cudaStream_t s, const uint32_t* mask) {
  Taps3 t;
  t.masked = mask != nullptr;
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < kSmoothMaskWords; ++i) t.mask[k][i] = mask ? mask[k * kSmoothMaskWords + i] : 0u;
  t.rx = gauss_radius(sigma[0]);
  t.ry = gauss_radius(sigma[1]);
  t.rz = gauss_radius(sigma[2]);
  make_taps(sigma[0], t.rx, t.wx);
  make_taps(sigma[1], t.ry, t.wy);
  make_taps(sigma[2], t.rz, t.wz);
  const int rmax = max(t.rx, max(t.ry, t.rz));
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kernel, int RM, int nyt) {
    const int my = (kSmThreads / 32) * nyt, xp = RM <= 4 ? 4 : 8;
    const size_t smem =
        sizeof(float) * (size_t(kStages) * (MX + 2 * xp) * (my + 2 * RM) + kXBuf * size_t(my + 2 * RM) * MX);
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>((nx + MX - 1) / MX), static_cast<unsigned>((ny + my - 1) / my),
                    static_cast<unsigned>((nz + MZ - 1) / MZ));
    if (e == cudaSuccess) kernel<<<grid, kSmThreads, smem, s>>>(in, out, nx, ny, nz, t);
  };
  if (rmax <= 1) go(smooth_fused_kernel<1, 4>, 1, 4);
  else if (rmax <= 2) go(smooth_fused_kernel<2, W3D_SM_NYT2>, 2, W3D_SM_NYT2);
  else if (rmax <= 3) go(smooth_fused_kernel<3, 4>, 3, 4);
  else if (rmax <= 4) go(smooth_fused_kernel<4, 2>, 4, 2);
  else if (rmax <= 6) go(smooth_fused_kernel<6, 1>, 6, 1);
  else go(smooth_fused_kernel<8, 1>, 8, 1);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace w3d
