// cube_kernel.cuh -- the default sm_100a kernel of the Sec. IV augmentation path
// (Rister et al., arXiv 1811.11226).
//
// One CTA per 16 x TY x 16 output tile of one volume:
//   1. every warp transforms the tile's 8 corners (p is monotone in each output
//      coordinate, so their min/max bound every p of the tile exactly) and
//      derives the tile's source footprint box -- no barrier needed;
//   2. all threads stage the box into shared memory with cp.async (16 B image
//      + 4 B label chunks; out-of-volume chunks are written with fill /
//      label_fill, so the gathers need no per-corner predicate: R6, R8) while
//      computing their first Philox block;
//   3. thread = output column (x, z) (lane = 16 x by 2 z, half-warps on two
//      z-planes: fewest bank conflicts, tools/model_tiles.py), rows y in groups
//      of 4 (one Philox block each, R10), as y-pairs in packed fp32x2.
// Per voxel, in the paper's order:
//   p = A x + b (R4) -> floor / frac on the FMA pipe (magic-number add with
//   round-down; indices read back from the float bits, no XU conversions) ->
//   8 LDS + 7 lerps (R5) | nearest label (R7) -> noise (R9-R11) -> window /
//   clamp (R12, R14) -> gamma (R13) -> store.
// Tiles whose box exceeds the buffer are split into y-parts (whole Philox
// blocks); a part that still does not fit is gathered through L1/L2.
// Compiled without fast-math and with -fmad=false: every FMA is explicit.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>

#include "philox.cuh"
#include "warp3d_internal.cuh"
#include "cube_config.cuh"

namespace w3d {
namespace cube {

constexpr float kM = 12582912.0f;       // 1.5 * 2^23: rm(p + kM) = kM + floor(p), |p| < 2^22
constexpr int32_t kMbits = 0x4B400000;  // bit pattern of kM
constexpr int kPlaneRes = 20;           // plane pitch = 20 (mod 32) words (bank spread)
constexpr float kSane = 2097152.0f;     // 2^21: unclamped boxes only for |p| below this

extern __shared__ __align__(16) unsigned char cube_smem[];
#ifndef W3D_NO_ABS
constexpr bool kUseAbs = true;  // fixed-box tiles index in absolute coordinates (sample2)
#else
constexpr bool kUseAbs = false;  // A/B knob
#endif

// float(y) for output rows y < kYTab, in constant memory: the full-column walk
// reads each row pair's (y, y + 1) as a uniform-register pair (LDCU.64; y is
// CTA-uniform), so the coordinate FFMA2 p = fma(A_k1, Y, inner) (R4) reads two
// per-thread registers instead of three and no FADD2 steps Y.  Bit-identical:
// the same y values enter the same FMA.
constexpr int kYTab = 4096;
struct YTable {
  float v[kYTab];
  constexpr YTable() : v() {
    for (int i = 0; i < kYTab; ++i) v[i] = static_cast<float>(i);
  }
};
static __constant__ YTable c_ytab = YTable();

// one copy per instantiation unit (cube_inst_*.cu); warp3d_cube.cu sums them
static __device__ unsigned long long g_cube_tiles[4];  // [staged, gathered, TMA, parts] (warp3d_tile_stats)

// dynamic shared memory, rounded up to 128 B (TMA destinations); the launch
// reserves the slack
__device__ __forceinline__ uint32_t smem_base() {
  return (static_cast<uint32_t>(__cvta_generic_to_shared(cube_smem)) + 127u) & ~127u;
}

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 add2_rm(float2 a, float2 b) {
  float2 r;
  asm("add.rm.ftz.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ float fset_ge_half(float t) {  // 1.0f if t >= 0.5 else 0.0f
  float r;
  asm("set.ge.f32.f32 %0, %1, 0f3F000000;" : "=f"(r) : "f"(t));
  return r;
}
// lerp(a, b, t) = a + t (b - a): one rounding for the difference, one FMA (R5)
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t) {
  return __ffma2_rn(t, sub2(b, a), a);
}
__device__ __forceinline__ float lerp1(float a, float b, float t) {
  return __fmaf_rn(t, __fsub_rn(b, a), a);
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ const float* gaddr_f32(const float* base, uint32_t off) {
  const float* p;
  asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(p) : "r"(off), "l"(base));
  return p;
}
__device__ __forceinline__ const uint8_t* gaddr_u8(const uint8_t* base, uint32_t off) {
  const uint8_t* p;
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(p) : "r"(off), "l"(base));
  return p;
}

// Input image element types: float32 (the headline) and int16 HU (NEXT-4: the
// 12-bit CT range; converted to float exactly at the gather).
// kChunk = elements per 16 B chunk (cp.async granularity, TMA row alignment).
template <class T> struct InT;
template <> struct InT<float> {
  static constexpr int kBytes = 4, kChunk = 4;
  __device__ static float load(const float* p) { return __ldg(p); }
};
template <> struct InT<int16_t> {
  static constexpr int kBytes = 2, kChunk = 8;
  __device__ static float load(const int16_t* p) {  // I2FP.F32.S32 (ALU), not I2F.S16 (XU)
    float v;
    // volatile: a predicated corner load must not be speculated (out-of-volume address)
    asm volatile("{\n\t.reg .s32 h;\n\tld.global.nc.s16 h, [%1];\n\tcvt.rn.f32.s32 %0, h;\n\t}"
        : "=f"(v)
        : "l"(p));
    return v;
  }
};
// per-volume input addresses (uniform batches or per-volume allocations, NEXT-4)
template <class T> __device__ __forceinline__ const T* vol_in(const VolDev& P) {
  return reinterpret_cast<const T*>(P.in_addr);
}
__device__ __forceinline__ const uint8_t* vol_lbl(const VolDev& P) {
  return reinterpret_cast<const uint8_t*>(P.lbl_addr);
}

// Pull-back coordinate (R4): p_k = fma(A_k1, y, fma(A_k0, x, fma(A_k2, z, b_k))).
__device__ __forceinline__ float coord(const float* A, int k, float X, float Y, float Z) {
  return __fmaf_rn(A[4 * k + 1], Y, __fmaf_rn(A[4 * k + 0], X, __fmaf_rn(A[4 * k + 2], Z,
                                                                         A[4 * k + 3])));
}

// ---------------------------------------------------------------------------
// Footprint box of output rows [y0, y1] of the tile (every lane returns the
// same box).  Unclamped when it fits (then no clamp in the inner loop: the box
// holds every corner, its out-of-volume part staged as fill); else from p
// clamped to [-1, n] (the clamped coordinate reads only fill or gets weight 0
// on in-volume voxels, which reproduces R6 / R8 exactly).
// ---------------------------------------------------------------------------
struct Box {
  int bx, by, bz;  // element 0 = input voxel (bx, by, bz); cp.async boxes: bx % 4 == 0
  int W, H, D, P;  // row pitch (W % 4 == 0), rows, planes, plane pitch (elements)
  int Wl, Pl;      // label row / plane pitch (= W, P for cp.async boxes)
  int bxl;         // label box origin x (TMA: bx rounded down to 16; cp.async: = bx)
  bool clamp;
};

template <class T>
__device__ __forceinline__ void make_box(const float* mn, const float* mx, int cap, Box& b) {
  constexpr int kC = InT<T>::kChunk;
  const int lx = __float2int_rd(mn[0]), hx = __float2int_rd(mx[0]) + 1;
  const int ly = __float2int_rd(mn[1]), hy = __float2int_rd(mx[1]) + 1;
  const int lz = __float2int_rd(mn[2]), hz = __float2int_rd(mx[2]) + 1;
  b.bx = lx & ~(kC - 1);
  b.by = ly;
  b.bz = lz;
  b.W = (hx - b.bx + 1 + kC - 1) & ~(kC - 1);
  b.H = hy - ly + 1;
  b.D = hz - lz + 1;
  const int wh = b.W * b.H;
  // bank-spreading plane pitch (a whole number of 16 B chunks), if it fits
  constexpr int kRes = kC == 4 ? kPlaneRes : 16;
  b.P = wh + ((kRes - wh) & 31);
  if (b.P * b.D > cap) b.P = wh;
  b.Wl = b.W;
  b.Pl = b.P;
  b.bxl = b.bx;
}

template <class T>
__device__ __forceinline__ bool tile_box(const WarpArgs& a, const float* A, int ox, int y0,
                                         int y1, int oz, int cap, Box& b) {
  const int c = threadIdx.x & 7;
  const float X = static_cast<float>((c & 1) ? min(ox + TX, a.mx) - 1 : ox);
  const float Y = static_cast<float>((c & 2) ? y1 : y0);
  const float Z = static_cast<float>((c & 4) ? min(oz + TZ, a.mz) - 1 : oz);
  float mn[3], mx[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mn[k] = mx[k] = coord(A, k, X, Y, Z);
#pragma unroll
  for (int off = 1; off < 8; off <<= 1)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mn[k] = fminf(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
      mx[k] = fmaxf(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
    }
  bool sane = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) sane &= (mn[k] > -kSane) & (mx[k] < kSane);
  if (sane) {
    make_box<T>(mn, mx, cap, b);
    if (b.P * b.D <= cap && b.W <= 4 * THREADS) {
      b.clamp = false;
      return true;
    }
  }
  const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                      static_cast<float>(a.nz)};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    mn[k] = fminf(fmaxf(mn[k], -1.0f), n[k]);
    mx[k] = fminf(fmaxf(mx[k], -1.0f), n[k]);
  }
  make_box<T>(mn, mx, cap, b);
  b.clamp = true;
  return b.P * b.D <= cap && b.W <= 4 * THREADS;
}

// ---------------------------------------------------------------------------
// Staging: thread t owns chunk column c = t % CW (4 voxels) of plane row
// r = t / CW (+ 256 k when a plane has more than 256 chunks) and copies it in
// every plane; in-volume chunks by cp.async (16 B image + 4 B label),
// out-of-volume chunks set to fill / label_fill.  nx % 4 == 0 and bx % 4 == 0,
// so a chunk is entirely inside or outside in x.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
}
template <int kBytes>
__device__ __forceinline__ const void* gaddr(const void* base, uint32_t off) {
  const void* p;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(off), "n"(kBytes), "l"(base));
  return p;
}
// the image fill as a 32-bit smem word: float bits, or two int16 copies
template <class T> __device__ __forceinline__ uint32_t fill_word(const WarpArgs& a);
template <> __device__ __forceinline__ uint32_t fill_word<float>(const WarpArgs& a) {
  return __float_as_uint(a.fill);
}
template <> __device__ __forceinline__ uint32_t fill_word<int16_t>(const WarpArgs& a) {
  return a.fill16_pair;
}

template <class T, bool kLabels, bool kInside, bool kImg = true>
__device__ __forceinline__ void stage_impl(const WarpArgs& a, const T* __restrict__ vin,
                                           const uint8_t* __restrict__ lin, const Box& b,
                                           uint32_t simg, uint32_t slbl) {
  constexpr int kC = InT<T>::kChunk, kB = InT<T>::kBytes;
  const int CW = b.W / kC;
  const int slots = CW * b.H;
  const uint32_t plane = static_cast<uint32_t>(a.nx) * static_cast<uint32_t>(a.ny);
  const uint32_t fw = fill_word<T>(a);
  const uint32_t lf4 = a.label_fill * 0x01010101u;
  // r = s / CW in fp32: (s + 1/2) / CW is >= 1/(2 CW) away from an integer and
  // s < 2^16, CW <= 256, so the product's error (< 2^-7) cannot cross one
  const float inv_cw = __frcp_rn(static_cast<float>(CW));
  for (int s = threadIdx.x; s < slots; s += THREADS) {
    const int r = __float2int_rz(__fmul_rn(static_cast<float>(s) + 0.5f, inv_cw));
    const int c = s - r * CW;
    const int gx = b.bx + kC * c, gy = b.by + r;
    const uint32_t e = static_cast<uint32_t>(r * b.W + kC * c);
    uint32_t si = simg + kB * e, sl = slbl + e;
    uint32_t goff = static_cast<uint32_t>(b.bz) * plane + static_cast<uint32_t>(gy * a.nx + gx);
    const uint32_t sstep = static_cast<uint32_t>(b.P);
    auto copy = [&]() {
      if (kImg) cp_async16(si, gaddr<kB>(vin, goff));
      if (kLabels) {
        if (kC == 4)
          cp_async4(sl, gaddr<1>(lin, goff));
        else
          cp_async8(sl, gaddr<1>(lin, goff));
      }
    };
    if (kInside) {
#pragma unroll 4
      for (int z = 0; z < b.D; ++z) {
        copy();
        si += kB * sstep;
        sl += sstep;
        goff += plane;
      }
    } else {
      const bool row_in = (static_cast<unsigned>(gx) < static_cast<unsigned>(a.nx)) &
                          (static_cast<unsigned>(gy) < static_cast<unsigned>(a.ny));
      for (int z = 0; z < b.D; ++z) {
        const int gz = b.bz + z;
        if (row_in & (static_cast<unsigned>(gz) < static_cast<unsigned>(a.nz))) {
          copy();
        } else {
          if (kImg)
            asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(si), "r"(fw) : "memory");
          if (kLabels) {
            if (kC == 4)
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(sl), "r"(lf4) : "memory");
            else
              asm volatile("st.shared.v2.b32 [%0], {%1, %1};" ::"r"(sl), "r"(lf4) : "memory");
          }
        }
        si += kB * sstep;
        sl += sstep;
        goff += plane;
      }
    }
  }
}

template <class T, bool kLabels>
__device__ __forceinline__ void stage(const WarpArgs& a, const T* vin, const uint8_t* lin,
                                      const Box& b, uint32_t simg, uint32_t slbl) {
  const bool inside = b.bx >= 0 && b.by >= 0 && b.bz >= 0 && b.bx + b.W <= a.nx &&
                      b.by + b.H <= a.ny && b.bz + b.D <= a.nz;
  if (inside)
    stage_impl<T, kLabels, true>(a, vin, lin, b, simg, slbl);
  else
    stage_impl<T, kLabels, false>(a, vin, lin, b, simg, slbl);
}
// the label box alone (the image box comes by TMA)
template <class T>
__device__ __forceinline__ void stage_lbl(const WarpArgs& a, const uint8_t* lin, const Box& b,
                                          uint32_t slbl) {
  const bool inside = b.bx >= 0 && b.by >= 0 && b.bz >= 0 && b.bx + b.W <= a.nx &&
                      b.by + b.H <= a.ny && b.bz + b.D <= a.nz;
  if (inside)
    stage_impl<T, true, true, false>(a, nullptr, lin, b, 0u, slbl);
  else
    stage_impl<T, true, false, false>(a, nullptr, lin, b, 0u, slbl);
}

// ---------------------------------------------------------------------------
// Per-thread constants of one staged part
// ---------------------------------------------------------------------------
// Values pinned in registers: ptxas would otherwise re-load loop invariants
// from the (dynamically indexed) parameter bank inside the hot loop, one LDC
// issue slot each.
__device__ __forceinline__ float pin(float x) {
  float y;
  asm volatile("mov.b32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pin(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
template <class T>
__device__ __forceinline__ T* pin_ptr(T* p) {
  unsigned long long y;
  asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(reinterpret_cast<unsigned long long>(p)));
  return reinterpret_cast<T*>(y);
}
// A warp-uniform value ptxas cannot see through (a shuffle from lane 0), so it
// does not split constant parts off address bases into extra adds.  Every
// lane of the warp must execute it.
__device__ __forceinline__ uint32_t opaque(uint32_t x) { return __shfl_sync(0xffffffffu, x, 0); }

struct View {
  float Wf, Pf;           // pitches as floats
  float Wlf, Plf;         // label pitches as floats
  float Mby, Mbz;         // kM + by, kM + bz
  uint32_t W4, P4;        // byte pitches of the image buffer
  uint32_t PW4;           // P4 + W4: the (y+1, z+1) corner row as one [R + UR] offset
  uint32_t cimg, clbl;    // image / label byte address = bits(L) * (4 | 1) + c
  float nx, ny, nz;       // clamp bounds
#ifdef W3D_CHECK_BOX
  uint32_t img_lo, img_hi, lbl_lo, lbl_hi;  // staged boxes [lo, hi) (byte addresses)
#endif
};

// W3D_CHECK_BOX (debug build, tools/sanitize.sh): every staged shared-memory
// access must fall inside its box -- a margin too small in cube_cp_box / make_box
// would otherwise read a neighbouring row of the box silently.  Traps (a launch
// error) on the first violation.
#ifdef W3D_CHECK_BOX
#define W3D_IN_BOX(addr, bytes, lo, hi) \
  do {                                   \
    if (!((addr) >= (lo) && (addr) + (bytes) <= (hi))) __trap(); \
  } while (0)
#else
#define W3D_IN_BOX(addr, bytes, lo, hi) \
  do {                                   \
  } while (0)
#endif

template <class T>
__device__ __forceinline__ View make_view(const WarpArgs& a, const Box& b, uint32_t simg,
                                          uint32_t slbl) {
  constexpr uint32_t kB = InT<T>::kBytes;
  View v;
  v.Wf = pin(static_cast<float>(b.W));
  v.Pf = pin(static_cast<float>(b.P));
  v.Wlf = pin(static_cast<float>(b.Wl));
  v.Plf = pin(static_cast<float>(b.Pl));
  v.Mby = pin(kM + static_cast<float>(b.by));
  v.Mbz = pin(kM + static_cast<float>(b.bz));
  v.W4 = pin(kB * static_cast<uint32_t>(b.W));
  v.P4 = pin(kB * static_cast<uint32_t>(b.P));
  v.PW4 = pin(v.P4 + v.W4);
  // bits(L) - kMbits = fx + W ry + P rz; element index = that - bx
  v.cimg = opaque(simg - kB * static_cast<uint32_t>(b.bx) - kB * static_cast<uint32_t>(kMbits));
  v.clbl = opaque(slbl - static_cast<uint32_t>(b.bxl) - static_cast<uint32_t>(kMbits));
  v.nx = static_cast<float>(a.nx);
  v.ny = static_cast<float>(a.ny);
  v.nz = static_cast<float>(a.nz);
#ifdef W3D_CHECK_BOX
  v.img_lo = simg;
  v.img_hi = simg + kB * static_cast<uint32_t>(b.P * b.D);
  v.lbl_lo = slbl;
  v.lbl_hi = slbl + static_cast<uint32_t>(b.Pl * b.D);
#endif
  return v;
}

// Per-volume constants held by every thread.
struct Vol {
  float A1[3];            // y column of A
  float sigma, ws, wo, lo, hi, gamma;
  uint32_t flags;
};

enum { kPhGeneric = 0, kPhFull = 1 };

// Photometric tail for a y-pair (PAPER.md:440-467 + gamma, R9-R14).
// kPhFull: noise + window + clamp + gamma all on (host-checked), straight line.
template <int kPh>
__device__ __forceinline__ float2 photometric2(float2 img, float2 n, const Vol& V) {
  const float2 v = __ffma2_rn(f2(V.sigma), n, img);  // I + sigma n (sigma = 0 without noise)
  float2 w;
  if (kPh == kPhFull) {
    w.x = __saturatef(__fmaf_rn(v.x, V.ws, V.wo));    // min(max((I - a)/(b - a), 0), 1)
    w.y = __saturatef(__fmaf_rn(v.y, V.ws, V.wo));
    const float2 l = __fmul2_rn(make_float2(lg2_approx(w.x), lg2_approx(w.y)), f2(V.gamma));
    return make_float2(ex2_approx(l.x), ex2_approx(l.y));
  }
  w = __ffma2_rn(v, f2(V.ws), f2(V.wo));
  w.x = fminf(fmaxf(w.x, V.lo), V.hi);
  w.y = fminf(fmaxf(w.y, V.lo), V.hi);
  if (V.flags & kGamma) {
    const float2 l = __fmul2_rn(make_float2(lg2_approx(w.x), lg2_approx(w.y)), f2(V.gamma));
    w = make_float2(ex2_approx(l.x), ex2_approx(l.y));
  }
  return w;
}

// byte address bits * 4 + c  /  bits + c  (one IMAD / IADD, no re-association)
__device__ __forceinline__ uint32_t addr4(float L, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(r) : "r"(__float_as_uint(L)), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t addr1(float L, uint32_t c) {
  uint32_t r;
  asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(__float_as_uint(L)), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t addr2(float L, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(r) : "r"(__float_as_uint(L)), "r"(c));
  return r;
}
template <class T> __device__ __forceinline__ uint32_t addrT(float L, uint32_t c) {
  return InT<T>::kBytes == 4 ? addr4(L, c) : addr2(L, c);
}
// the two x-neighbours at addr and addr + element size, as floats
template <class T> __device__ __forceinline__ void lds_pair(uint32_t a, float& v0, float& v1);
template <> __device__ __forceinline__ void lds_pair<float>(uint32_t a, float& v0, float& v1) {
  asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];"
               : "=f"(v0), "=f"(v1)
               : "r"(a));
}
// int16: the load sign-extends into a 32-bit register and the exact
// conversion is cvt.rn.f32.s32 (I2FP on the ALU pipe); cvt.rn.f32.s16 from a
// 16-bit register compiles to I2F.S16 on the quarter-rate XU pipe, which the
// Box-Muller / gamma MUFUs already load
template <> __device__ __forceinline__ void lds_pair<int16_t>(uint32_t a, float& v0, float& v1) {
  asm volatile(
      "{\n\t.reg .s32 h0, h1;\n\tld.shared.s16 h0, [%2];\n\tld.shared.s16 h1, [%2+2];\n\t"
      "cvt.rn.f32.s32 %0, h0;\n\tcvt.rn.f32.s32 %1, h1;\n\t}"
      : "=f"(v0), "=f"(v1)
      : "r"(a));
}
template <class T> __device__ __forceinline__ float lds_one(uint32_t a) {
  float v0, v1;
  if (InT<T>::kBytes == 4) return lds_f32(a);
  asm volatile("{\n\t.reg .s32 h0;\n\tld.shared.s16 h0, [%1];\n\tcvt.rn.f32.s32 %0, h0;\n\t}"
               : "=f"(v0)
               : "r"(a));
  (void)v1;
  return v0;
}

struct GView {
  uint32_t nx, ny, nz;  // input dims
  uint32_t sy, sz;      // element strides nx, nx ny
  uint32_t C;           // -kMbits (1 + sy + sz) mod 2^32: o = bits(sx) + sy bits(sy) + sz bits(sz) + C
  float fnx, fny, fnz;
};
__device__ __forceinline__ GView make_gview(const WarpArgs& a) {
  GView g;
  g.nx = static_cast<uint32_t>(a.nx);
  g.ny = static_cast<uint32_t>(a.ny);
  g.nz = static_cast<uint32_t>(a.nz);
  g.sy = g.nx;
  g.sz = g.nx * g.ny;
  g.C = 0u - static_cast<uint32_t>(kMbits) * (1u + g.sy + g.sz);
  g.fnx = static_cast<float>(a.nx);
  g.fny = static_cast<float>(a.ny);
  g.fnz = static_cast<float>(a.nz);
  return g;
}
// Labels gathered from global memory (the 8-row tiles of large footprints: no
// label box, so the TMA moves half the rows -- the box wait, not dispatch, bounds
// those tiles).  The nearest voxel (R7) in volume coordinates straight from the
// magic-number floats kM + n_k, its offset mod 2^32 as gather2's; kChecked (tiles
// that can sample outside): label_fill for a nearest voxel outside the volume (R8).
template <bool kChecked>
__device__ __forceinline__ void label_gather2(const uint8_t* __restrict__ lin, const GView& g,
                                              uint32_t lfill, float2 sx, float2 sy, float2 sz,
                                              float2 hx, float2 hy, float2 hz, uint32_t& l0,
                                              uint32_t& l1) {
  const float2 nx = __fadd2_rn(sx, hx), ny = __fadd2_rn(sy, hy), nz = __fadd2_rn(sz, hz);
  auto one = [&](float fx, float fy, float fz) -> uint32_t {
    const uint32_t bx = __float_as_uint(fx), by = __float_as_uint(fy), bz = __float_as_uint(fz);
    const uint32_t o = bx + g.sy * by + g.sz * bz + g.C;
    if (kChecked) {
      const uint32_t ix = bx - static_cast<uint32_t>(kMbits), iy = by - static_cast<uint32_t>(kMbits),
                     iz = bz - static_cast<uint32_t>(kMbits);
      if (!((ix < g.nx) & (iy < g.ny) & (iz < g.nz))) return lfill;
    }
    return __ldg(lin + static_cast<size_t>(o));
  };
  l0 = one(nx.x, ny.x, nz.x);
  l1 = one(nx.y, ny.y, nz.y);
}

// Staged sampling of a y-pair: image (trilinear or nearest) and label.
// kSameLbl: the label box has the image box's pitches (cp.async boxes).
// kAbs: the index in absolute volume coordinates, kM + fx + W fy + P fz (fy, fz
// = floor(p) already formed for the fractions), the box origin folded into the
// view's address constants -- two FADD2 fewer per pair than the box-relative
// kM + fx + W (fy - by) + P (fz - bz).  Exact while |fx + W fy + P fz| < 2^22:
// the host enables it per volume (VolDev::cp_abs) from the volume's dims, box
// pitches and the range of p over the whole output volume.
template <class T, bool kLabels, bool kNearest, bool kClamp, bool kSameLbl, bool kAbs = false,
          int kLG = 0>
__device__ __forceinline__ void sample2(const View& v, float2 px, float2 py, float2 pz,
                                        float2& img, uint32_t& l0, uint32_t& l1,
                                        const uint8_t* lin = nullptr, const GView* gv = nullptr,
                                        uint32_t lfill = 0u) {
  if (kClamp) {
    px = make_float2(fminf(fmaxf(px.x, -1.0f), v.nx), fminf(fmaxf(px.y, -1.0f), v.nx));
    py = make_float2(fminf(fmaxf(py.x, -1.0f), v.ny), fminf(fmaxf(py.y, -1.0f), v.ny));
    pz = make_float2(fminf(fmaxf(pz.x, -1.0f), v.nz), fminf(fmaxf(pz.y, -1.0f), v.nz));
  }
  // floor on the FMA pipe: rm(p + kM) = kM + floor(p) exactly (|p| < 2^22)
  const float2 sx = add2_rm(px, f2(kM)), sy = add2_rm(py, f2(kM)), sz = add2_rm(pz, f2(kM));
  const float2 fy = sub2(sy, f2(kM)), fz = sub2(sz, f2(kM));  // floor(p), exact
  const float2 tx = sub2(px, sub2(sx, f2(kM)));
  const float2 ty = sub2(py, fy);
  const float2 tz = sub2(pz, fz);
  const float2 ry = kAbs ? fy : sub2(sy, f2(v.Mby)), rz = kAbs ? fz : sub2(sz, f2(v.Mbz));
  // kM + fx + W ry + P rz: exact integers below 2^24
  const float2 L = __ffma2_rn(rz, f2(v.Pf), __ffma2_rn(ry, f2(v.Wf), sx));
  float2 Ln = L;
  if (kLabels || kNearest) {  // nearest voxel (R7): + (t >= 0.5) per axis
    const float2 hx = make_float2(fset_ge_half(tx.x), fset_ge_half(tx.y));
    const float2 hy = make_float2(fset_ge_half(ty.x), fset_ge_half(ty.y));
    const float2 hz = make_float2(fset_ge_half(tz.x), fset_ge_half(tz.y));
    if (kNearest) Ln = __ffma2_rn(hz, f2(v.Pf), __ffma2_rn(hy, f2(v.Wf), __fadd2_rn(L, hx)));
    if (kLabels && kLG != 0) {  // no label box: gathered (8-row tiles)
      label_gather2<kLG == 2>(lin, *gv, lfill, sx, sy, sz, hx, hy, hz, l0, l1);
    } else if (kLabels) {  // label buffer: own pitches (kM + fx + hx - bx + Wl (ry + hy) + Pl (rz + hz))
      const float2 Ll =
          kSameLbl ? (kNearest ? Ln
                               : __ffma2_rn(hz, f2(v.Pf), __ffma2_rn(hy, f2(v.Wf), __fadd2_rn(L, hx))))
                   : __ffma2_rn(__fadd2_rn(rz, hz), f2(v.Plf),
                                __ffma2_rn(__fadd2_rn(ry, hy), f2(v.Wlf), __fadd2_rn(sx, hx)));
      W3D_IN_BOX(addr1(Ll.x, v.clbl), 1u, v.lbl_lo, v.lbl_hi);
      W3D_IN_BOX(addr1(Ll.y, v.clbl), 1u, v.lbl_lo, v.lbl_hi);
      l0 = lds_u8(addr1(Ll.x, v.clbl));
      l1 = lds_u8(addr1(Ll.y, v.clbl));
    }
  }
  if (kNearest) {
    W3D_IN_BOX(addrT<T>(Ln.x, v.cimg), InT<T>::kBytes, v.img_lo, v.img_hi);
    W3D_IN_BOX(addrT<T>(Ln.y, v.cimg), InT<T>::kBytes, v.img_lo, v.img_hi);
    img = make_float2(lds_one<T>(addrT<T>(Ln.x, v.cimg)), lds_one<T>(addrT<T>(Ln.y, v.cimg)));
    return;
  }
  const uint32_t a0 = addrT<T>(L.x, v.cimg), b0 = addrT<T>(L.y, v.cimg);
  const uint32_t a1 = a0 + v.W4, b1 = b0 + v.W4, a2 = a0 + v.P4, b2 = b0 + v.P4;
  const uint32_t a3 = a0 + v.PW4, b3 = b0 + v.PW4;
  // the 8 corners span [a0, a3 + 2 elements) (pitches > 0)
  W3D_IN_BOX(a0, 2u * InT<T>::kBytes, v.img_lo, v.img_hi);
  W3D_IN_BOX(a3, 2u * InT<T>::kBytes, v.img_lo, v.img_hi);
  W3D_IN_BOX(b0, 2u * InT<T>::kBytes, v.img_lo, v.img_hi);
  W3D_IN_BOX(b3, 2u * InT<T>::kBytes, v.img_lo, v.img_hi);
  float2 c000, c100, c010, c110, c001, c101, c011, c111;
  lds_pair<T>(a0, c000.x, c100.x);
  lds_pair<T>(b0, c000.y, c100.y);
  lds_pair<T>(a1, c010.x, c110.x);
  lds_pair<T>(b1, c010.y, c110.y);
  lds_pair<T>(a2, c001.x, c101.x);
  lds_pair<T>(b2, c001.y, c101.y);
  lds_pair<T>(a3, c011.x, c111.x);
  lds_pair<T>(b3, c011.y, c111.y);
#ifdef W3D_LERP_CP
  // A/B knob: corner pairs of ONE voxel in the packed lanes ((z0, z1) corners at
  // x0 / x1), the fraction as a broadcast scalar; same lerps in the same order
  // (R5), so the same bits
  auto vox = [](float a000, float a100, float a010, float a110, float a001, float a101,
                float a011, float a111, float fx, float fy, float fz) {
    const float2 lo = lerp2(make_float2(a000, a001), make_float2(a100, a101), f2(fx));  // (c00, c01)
    const float2 hi = lerp2(make_float2(a010, a011), make_float2(a110, a111), f2(fx));  // (c10, c11)
    const float2 cz = lerp2(lo, hi, f2(fy));                                             // (c0, c1)
    return lerp1(cz.x, cz.y, fz);
  };
  img = make_float2(vox(c000.x, c100.x, c010.x, c110.x, c001.x, c101.x, c011.x, c111.x, tx.x,
                        ty.x, tz.x),
                    vox(c000.y, c100.y, c010.y, c110.y, c001.y, c101.y, c011.y, c111.y, tx.y,
                        ty.y, tz.y));
#else
  const float2 c00 = lerp2(c000, c100, tx), c10 = lerp2(c010, c110, tx);
  const float2 c01 = lerp2(c001, c101, tx), c11 = lerp2(c011, c111, tx);
  img = lerp2(lerp2(c00, c10, ty), lerp2(c01, c11, ty), tz);
#endif
}

// The label of a y-pair alone (an occluded column, R15: the image is 0 and its
// fetch skipped): the index arithmetic of sample2's label
// path, op for op, so the labels are the same bits.
template <bool kClamp, bool kSameLbl, bool kAbs = false, int kLG = 0>
__device__ __forceinline__ void label2(const View& v, float2 px, float2 py, float2 pz,
                                       uint32_t& l0, uint32_t& l1, const uint8_t* lin = nullptr,
                                       const GView* gv = nullptr, uint32_t lfill = 0u) {
  if (kClamp) {
    px = make_float2(fminf(fmaxf(px.x, -1.0f), v.nx), fminf(fmaxf(px.y, -1.0f), v.nx));
    py = make_float2(fminf(fmaxf(py.x, -1.0f), v.ny), fminf(fmaxf(py.y, -1.0f), v.ny));
    pz = make_float2(fminf(fmaxf(pz.x, -1.0f), v.nz), fminf(fmaxf(pz.y, -1.0f), v.nz));
  }
  const float2 sx = add2_rm(px, f2(kM)), sy = add2_rm(py, f2(kM)), sz = add2_rm(pz, f2(kM));
  const float2 fy = sub2(sy, f2(kM)), fz = sub2(sz, f2(kM));
  const float2 tx = sub2(px, sub2(sx, f2(kM)));
  const float2 ty = sub2(py, fy);
  const float2 tz = sub2(pz, fz);
  const float2 ry = kAbs ? fy : sub2(sy, f2(v.Mby)), rz = kAbs ? fz : sub2(sz, f2(v.Mbz));
  const float2 hx = make_float2(fset_ge_half(tx.x), fset_ge_half(tx.y));
  const float2 hy = make_float2(fset_ge_half(ty.x), fset_ge_half(ty.y));
  const float2 hz = make_float2(fset_ge_half(tz.x), fset_ge_half(tz.y));
  if (kLG != 0) {
    label_gather2<kLG == 2>(lin, *gv, lfill, sx, sy, sz, hx, hy, hz, l0, l1);
    return;
  }
  float2 Ll;
  if (kSameLbl) {
    const float2 L = __ffma2_rn(rz, f2(v.Pf), __ffma2_rn(ry, f2(v.Wf), sx));
    Ll = __ffma2_rn(hz, f2(v.Pf), __ffma2_rn(hy, f2(v.Wf), __fadd2_rn(L, hx)));
  } else {
    Ll = __ffma2_rn(__fadd2_rn(rz, hz), f2(v.Plf),
                    __ffma2_rn(__fadd2_rn(ry, hy), f2(v.Wlf), __fadd2_rn(sx, hx)));
  }
  W3D_IN_BOX(addr1(Ll.x, v.clbl), 1u, v.lbl_lo, v.lbl_hi);
  W3D_IN_BOX(addr1(Ll.y, v.clbl), 1u, v.lbl_lo, v.lbl_hi);
  l0 = lds_u8(addr1(Ll.x, v.clbl));
  l1 = lds_u8(addr1(Ll.y, v.clbl));
}

// ---------------------------------------------------------------------------
// Gather sampling of one voxel through L1/L2 with per-corner bounds (R6-R8,
// NaN-safe float compares first).  Used for parts whose box does not fit.
// ---------------------------------------------------------------------------
template <class T, bool kLabels, bool kNearest>
__device__ __forceinline__ void sample_gather(const WarpArgs& a, const T* __restrict__ vin,
                                              const uint8_t* __restrict__ lin, float px,
                                              float py, float pz, float& img, uint32_t& lbl) {
  img = a.fill;
  lbl = a.label_fill;
  const float fnx = static_cast<float>(a.nx), fny = static_cast<float>(a.ny),
              fnz = static_cast<float>(a.nz);
  const bool near_in = (px >= -0.5f) & (px < fnx - 0.5f) & (py >= -0.5f) & (py < fny - 0.5f) &
                       (pz >= -0.5f) & (pz < fnz - 0.5f);
  const bool any_in = (px > -1.0f) & (px < fnx) & (py > -1.0f) & (py < fny) & (pz > -1.0f) &
                      (pz < fnz);
  if (!any_in) return;  // then also !near_in
  const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
  const float tx = __fsub_rn(px, fx), ty = __fsub_rn(py, fy), tz = __fsub_rn(pz, fz);
  const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
  const int64_t sy = a.nx, sz = static_cast<int64_t>(a.nx) * a.ny;
  if (near_in && (kLabels || kNearest)) {
    const int64_t r = (iz + (tz >= 0.5f)) * sz + (iy + (ty >= 0.5f)) * sy + (ix + (tx >= 0.5f));
    if (kLabels) lbl = __ldg(lin + r);
    if (kNearest) img = InT<T>::load(vin + r);
  }
  if (kNearest) return;
  const bool x0 = ix >= 0, x1 = ix + 1 < a.nx, y0 = iy >= 0, y1 = iy + 1 < a.ny;
  const bool z0 = iz >= 0, z1 = iz + 1 < a.nz;
  const T* b = vin + (iz * sz + iy * sy + ix);
  const float f = a.fill;
  const float c000 = (x0 & y0 & z0) ? InT<T>::load(b) : f;
  const float c100 = (x1 & y0 & z0) ? InT<T>::load(b + 1) : f;
  const float c010 = (x0 & y1 & z0) ? InT<T>::load(b + sy) : f;
  const float c110 = (x1 & y1 & z0) ? InT<T>::load(b + sy + 1) : f;
  const float c001 = (x0 & y0 & z1) ? InT<T>::load(b + sz) : f;
  const float c101 = (x1 & y0 & z1) ? InT<T>::load(b + sz + 1) : f;
  const float c011 = (x0 & y1 & z1) ? InT<T>::load(b + sz + sy) : f;
  const float c111 = (x1 & y1 & z1) ? InT<T>::load(b + sz + sy + 1) : f;
  const float c00 = lerp1(c000, c100, tx), c10 = lerp1(c010, c110, tx);
  const float c01 = lerp1(c001, c101, tx), c11 = lerp1(c011, c111, tx);
  img = lerp1(lerp1(c00, c10, ty), lerp1(c01, c11, ty), tz);
}

// Gather sampling of a y-pair through L1/L2 (the GATHER kernel; tiles whose
// footprint does not fit the buffer), same arithmetic as sample2: floor / frac
// by the magic-number add, 32-bit cell offsets read back from the float bits
// (o = fx + nx fy + nx ny fz, mod 2^32; the volume has < 2^31 voxels), the
// same lerp nesting (R5) and nearest rule (R7).  The tile's class (host box
// offsets, tile_inside / tile_outside) picks the mode:
//   kGIn:  every trilinear corner and nearest voxel of the tile is inside --
//          no clamps, no predicates;
//   kGOut: every sample is outside (p_k < -1 or p_k > n_k for some axis k on
//          the whole tile) -- fill / label_fill, no loads;
//   kGEdge: p clamped to [-1, n] (a clamped coordinate reads only outside
//          cells or gets weight 0 on an inside one: R6 / R8 exactly, as the
//          clamped staging boxes) and every corner load predicated on its cell
//          being inside, fill otherwise.
//   kGWide: a dim >= 2^21 (the magic-number floor needs |p| < 2^22): the
//          per-voxel sample_gather with float floors and 64-bit offsets.
enum { kGEdge = 0, kGIn = 1, kGOut = 2, kGWide = 3 };
template <class T, bool kLabels, int kGMode>
__device__ __forceinline__ void gather2(const WarpArgs& a, const T* __restrict__ vin,
                                        const uint8_t* __restrict__ lin, const GView& g, float2 px,
                                        float2 py, float2 pz, float2& img, uint32_t& l0,
                                        uint32_t& l1) {
  if (kGMode == kGOut) {
    img = f2(a.fill);
    l0 = l1 = a.label_fill;
    return;
  }
  if (kGMode == kGEdge) {
    px = make_float2(fminf(fmaxf(px.x, -1.0f), g.fnx), fminf(fmaxf(px.y, -1.0f), g.fnx));
    py = make_float2(fminf(fmaxf(py.x, -1.0f), g.fny), fminf(fmaxf(py.y, -1.0f), g.fny));
    pz = make_float2(fminf(fmaxf(pz.x, -1.0f), g.fnz), fminf(fmaxf(pz.y, -1.0f), g.fnz));
  }
  const float2 sx = add2_rm(px, f2(kM)), sy = add2_rm(py, f2(kM)), sz = add2_rm(pz, f2(kM));
  const float2 tx = sub2(px, sub2(sx, f2(kM)));
  const float2 ty = sub2(py, sub2(sy, f2(kM)));
  const float2 tz = sub2(pz, sub2(sz, f2(kM)));
  const float2 sxy[3] = {sx, sy, sz}, txy[3] = {tx, ty, tz};
  float c[2][8];
  uint32_t lab[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // the two voxels of the pair
    const uint32_t bx = __float_as_uint(h ? sxy[0].y : sxy[0].x);
    const uint32_t by = __float_as_uint(h ? sxy[1].y : sxy[1].x);
    const uint32_t bz = __float_as_uint(h ? sxy[2].y : sxy[2].x);
    const int32_t o = static_cast<int32_t>(bx + g.sy * by + g.sz * bz + g.C);
    const T* b = vin + o;
    const T* bY = b + g.sy;
    const T* bZ = b + g.sz;
    const T* bYZ = bZ + g.sy;
    if (kGMode == kGIn) {
#ifdef W3D_CHECK_BOX  // an inside tile's corners are all in the volume (tile_inside)
      if (o < 0 || int64_t(o) + g.sz + g.sy + 1 >= int64_t(g.sz) * g.nz) __trap();
#endif
      c[h][0] = InT<T>::load(b);
      c[h][1] = InT<T>::load(b + 1);
      c[h][2] = InT<T>::load(bY);
      c[h][3] = InT<T>::load(bY + 1);
      c[h][4] = InT<T>::load(bZ);
      c[h][5] = InT<T>::load(bZ + 1);
      c[h][6] = InT<T>::load(bYZ);
      c[h][7] = InT<T>::load(bYZ + 1);
    } else {
      // cell coordinates in [-1, n]: corner k inside iff (unsigned) index < n
      const uint32_t fx = bx - static_cast<uint32_t>(kMbits);
      const uint32_t fy = by - static_cast<uint32_t>(kMbits);
      const uint32_t fz = bz - static_cast<uint32_t>(kMbits);
      const bool x0 = fx < g.nx, x1 = fx + 1u < g.nx, y0 = fy < g.ny, y1 = fy + 1u < g.ny;
      const bool z0 = fz < g.nz, z1 = fz + 1u < g.nz;
      const float f = a.fill;
      c[h][0] = (x0 & y0 & z0) ? InT<T>::load(b) : f;
      c[h][1] = (x1 & y0 & z0) ? InT<T>::load(b + 1) : f;
      c[h][2] = (x0 & y1 & z0) ? InT<T>::load(bY) : f;
      c[h][3] = (x1 & y1 & z0) ? InT<T>::load(bY + 1) : f;
      c[h][4] = (x0 & y0 & z1) ? InT<T>::load(bZ) : f;
      c[h][5] = (x1 & y0 & z1) ? InT<T>::load(bZ + 1) : f;
      c[h][6] = (x0 & y1 & z1) ? InT<T>::load(bYZ) : f;
      c[h][7] = (x1 & y1 & z1) ? InT<T>::load(bYZ + 1) : f;
    }
    if (kLabels) {  // nearest voxel (R7): + (t >= 0.5) per axis
      const uint32_t hx = (h ? txy[0].y : txy[0].x) >= 0.5f;
      const uint32_t hy = (h ? txy[1].y : txy[1].x) >= 0.5f;
      const uint32_t hz = (h ? txy[2].y : txy[2].x) >= 0.5f;
      const uint8_t* q = lin + (o + static_cast<int32_t>(hx + g.sy * hy + g.sz * hz));
      if (kGMode == kGIn) {
        lab[h] = __ldg(q);
      } else {
        const uint32_t nx_ = bx - static_cast<uint32_t>(kMbits) + hx;
        const uint32_t ny_ = by - static_cast<uint32_t>(kMbits) + hy;
        const uint32_t nz_ = bz - static_cast<uint32_t>(kMbits) + hz;
        lab[h] = (nx_ < g.nx && ny_ < g.ny && nz_ < g.nz) ? static_cast<uint32_t>(__ldg(q))
                                                          : a.label_fill;
      }
    }
  }
  const float2 c000 = make_float2(c[0][0], c[1][0]), c100 = make_float2(c[0][1], c[1][1]);
  const float2 c010 = make_float2(c[0][2], c[1][2]), c110 = make_float2(c[0][3], c[1][3]);
  const float2 c001 = make_float2(c[0][4], c[1][4]), c101 = make_float2(c[0][5], c[1][5]);
  const float2 c011 = make_float2(c[0][6], c[1][6]), c111 = make_float2(c[0][7], c[1][7]);
  const float2 c00 = lerp2(c000, c100, tx), c10 = lerp2(c010, c110, tx);
  const float2 c01 = lerp2(c001, c101, tx), c11 = lerp2(c011, c111, tx);
  img = lerp2(lerp2(c00, c10, ty), lerp2(c01, c11, ty), tz);
  if (kLabels) {
    l0 = lab[0];
    l1 = lab[1];
  }
}

#ifndef W3D_DBG_NOSTORE
__device__ __forceinline__ void st_f32(float* p, float v) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
#else  // diagnostic: a store only for values no real voxel produces (kept alive, ~never taken)
__device__ __forceinline__ void st_f32(float* p, float v) {
  if (v == 1234.5f) asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_u8(uint8_t* p, uint32_t v) {
  if (v == 251u) asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
#endif
// p + bytes (a 64-bit byte step, kept as an add: ptxas would turn p + 4 * mx
// into IMAD.WIDE.U32, ~4 dispatch cycles against 2 for the add pair)
template <class P>
__device__ __forceinline__ P* step(P* p, int64_t bytes) {
  P* r;
  asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(bytes));
  return r;
}
// base + element offset in one IMAD.WIDE.U32
__device__ __forceinline__ float* at(float* base, uint32_t off) {
  float* r;
  asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(r) : "r"(off), "l"(base));
  return r;
}
__device__ __forceinline__ uint8_t* at(uint8_t* base, uint32_t off) {
  uint8_t* r;
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(r) : "r"(off), "l"(base));
  return r;
}

// ---------------------------------------------------------------------------
// Rows [y0, y0 + 4 ng) of the thread's output column (X, Z), 4-row groups.
// kStaged: sample from the staged view v, else gather.  `n` holds the first
// group's normals (computed while the staging copies were in flight); the next
// group's Philox block is computed inside each iteration (independent chain).
// ---------------------------------------------------------------------------
// kPre: the first kPre (1, 2 or 4) groups' normals arrive precomputed (n, n1,
// n2, n3; computed while the staging copies are in flight) and the loop
// computes group g + kPre's block.
template <class T, bool kLabels, bool kNearest, int kPh, bool kStaged, bool kClamp,
          bool kSameLbl, bool kFull, int kPre, int kGMode, bool kOccOnly, bool kAbs, int kLG>
__device__ __forceinline__ void column_rows_impl(const WarpArgs& a, const VolDev& P, const Vol& V0,
                                            const View& v, int vi, int X, int Z, int y0, int ng,
                                            float4 n, float4 n1 = make_float4(0.f, 0.f, 0.f, 0.f),
                                            float4 n2 = make_float4(0.f, 0.f, 0.f, 0.f),
                                            float4 n3 = make_float4(0.f, 0.f, 0.f, 0.f)) {
  const T* __restrict__ vin = vol_in<T>(P);
  const uint8_t* __restrict__ lin = kLabels ? vol_lbl(P) : nullptr;
  Vol V = V0;
#pragma unroll
  for (int k = 0; k < 3; ++k)  // per-thread registers (opaque): the FFMA2's one uniform
    V.A1[k] = __int_as_float(static_cast<int>(  // operand slot goes to the row pair Y
        opaque(static_cast<uint32_t>(__float_as_int(V0.A1[k])))));
  V.sigma = pin(V0.sigma);
  V.ws = pin(V0.ws);
  V.wo = pin(V0.wo);
  V.gamma = pin(V0.gamma);
  const float fX = static_cast<float>(X), fZ = static_cast<float>(Z);
  // x/z part of the coordinate, hoisted (R4 nesting)
  const float t0 = __fmaf_rn(P.A[0], fX, __fmaf_rn(P.A[2], fZ, P.A[3]));
  const float t1 = __fmaf_rn(P.A[4], fX, __fmaf_rn(P.A[6], fZ, P.A[7]));
  const float t2 = __fmaf_rn(P.A[8], fX, __fmaf_rn(P.A[10], fZ, P.A[11]));
  const int mx = a.mx, my = a.my;
  const uint32_t mxu = pin(static_cast<uint32_t>(mx));
  const uint32_t row1 = pin(mxu);
  const uint32_t gyn = static_cast<uint32_t>((my + 3) >> 2);
#ifdef W3D_DBG_NONOISE
  const bool noise = false;
#else
  const bool noise = kPh == kPhFull || (V.flags & kNoise);
#endif
  const PhiloxPrefix pp{pin(P.ph_K0), pin(P.ph_K1), pin(P.ph_K2), pin(P.ph_U3)};
  uint32_t rk0[10], rk1[10];
#pragma unroll
  for (int r = 2; r < 10; ++r) {  // kPhFull: launch-wide keys at fixed parameter offsets
    rk0[r] = kPh == kPhFull ? a.rk0[r] : pin(P.rk0[r]);
    rk1[r] = kPh == kPhFull ? a.rk1[r] : pin(P.rk1[r]);
  }
  // output element offset of row y within the volume (< 2^31)
  // output row pointers, pinned (else re-derived from the parameters every row)
  const size_t o = static_cast<size_t>((Z * my + y0) * mx + X);
  float* po = pin_ptr(a.out + P.out_slot * a.out_stride + o);
  uint8_t* pl = kLabels ? pin_ptr(a.out_lbl + P.out_slot * a.out_stride + o) : nullptr;
  uint32_t q = static_cast<uint32_t>(X) +
               mxu * (gyn * static_cast<uint32_t>(Z) + static_cast<uint32_t>(y0 >> 2));
  float2 Y2 = make_float2(static_cast<float>(y0), static_cast<float>(y0 + 1));
  const GView gv = make_gview(a);
  // one y-pair (rows ya, ya + 1) with its two normals; kOcc (an occluded column,
  // R15): the image is 0 and every step after the occlusion test is skipped,
  // the texture fetch included -- only the labels are warped
  auto pair = [&](int ya, float2 nsp, auto occ_tag) {
    constexpr bool kOcc = decltype(occ_tag)::value;
    const float2 px = __ffma2_rn(f2(V.A1[0]), Y2, f2(t0));
    const float2 py = __ffma2_rn(f2(V.A1[1]), Y2, f2(t1));
    const float2 pz = __ffma2_rn(f2(V.A1[2]), Y2, f2(t2));
    Y2 = __fadd2_rn(Y2, make_float2(2.0f, 2.0f));
    float2 img;
    uint32_t l0 = 0, l1 = 0;
    if (kOcc && kStaged) {
      if (kLabels) label2<kClamp, kSameLbl, kAbs, kLG>(v, px, py, pz, l0, l1, lin, &gv, a.label_fill);
    } else if (kOcc && !kLabels) {
    } else if (kStaged) {
      sample2<T, kLabels, kNearest, kClamp, kSameLbl, kAbs, kLG>(v, px, py, pz, img, l0, l1, lin,
                                                                &gv, a.label_fill);
    } else if (!kNearest && kGMode != kGWide) {
      gather2<T, kLabels, kGMode>(a, vin, lin, gv, px, py, pz, img, l0, l1);
    } else {
      sample_gather<T, kLabels, kNearest>(a, vin, lin, px.x, py.x, pz.x, img.x, l0);
      sample_gather<T, kLabels, kNearest>(a, vin, lin, px.y, py.y, pz.y, img.y, l1);
    }
    const float2 out = kOcc ? make_float2(0.0f, 0.0f) : photometric2<kPh>(img, nsp, V);
    const bool second = kFull || ya + 1 < my;
#ifndef W3D_PTR_WIDE
    // next row: 64-bit adds of the parameter pitch (IADD3 + IADD3.X on the ALU pipe)
    float* po1 = step(po, a.out_row_bytes);
    st_f32(po, out.x);
    if (second) st_f32(po1, out.y);
    po = step(po1, a.out_row_bytes);
    if (kLabels) {
      uint8_t* pl1 = step(pl, a.out_lrow_bytes);
      st_u8(pl, l0);
      if (second) st_u8(pl1, l1);
      pl = step(pl1, a.out_lrow_bytes);
    }
#else  // A/B: the element offset scaled by IMAD.WIDE.U32
    float* po1 = po + row1;
    st_f32(po, out.x);
    if (second) st_f32(po1, out.y);
    po = po1 + row1;
    if (kLabels) {
      uint8_t* pl1 = pl + row1;
      st_u8(pl, l0);
      if (second) st_u8(pl1, l1);
      pl = pl1 + row1;
    }
#endif
  };
  if constexpr (kOccOnly) {  // R15: labels only (no Philox block, no image fetch)
#pragma unroll 1
    for (int ya = y0; ya < y0 + 4 * ng && ya < my; ya += 2)
      pair(ya, make_float2(0.f, 0.f), std::true_type());
    return;
  }
  if constexpr (kFull && kPre == 2) {
    if (ng == 2) {  // a whole 8-row column (8-row tiles), normals precomputed
      const std::false_type live_col;
      pair(y0, make_float2(n.x, n.y), live_col);
      pair(y0 + 2, make_float2(n.z, n.w), live_col);
      pair(y0 + 4, make_float2(n1.x, n1.y), live_col);
      pair(y0 + 6, make_float2(n1.z, n1.w), live_col);
      return;
    }
  }
  if constexpr (kFull && kPre == 4) {
    if (ng == 4) {  // a whole 16-row column, normals precomputed: straight line, no rotation
      const std::false_type live_col;
#ifndef W3D_NO_YTAB
      // the tile's first row from the block index itself, so ptxas sees it uniform:
      // without bricks the tile's y0 IS blockIdx.y * kTY (testing y0 == yb instead
      // lets the compiler substitute y0's per-thread register for yb, and the table
      // reads become per-thread LDC)
      const int yb = static_cast<int>(blockIdx.y) * kTY;
      if (a.brick == 0 && yb + 16 <= kYTab) {  // row pairs from the uniform table
        auto yt = [&](int j) {
          return make_float2(c_ytab.v[yb + 2 * j], c_ytab.v[yb + 2 * j + 1]);
        };
        Y2 = yt(0); pair(y0, make_float2(n.x, n.y), live_col);
        Y2 = yt(1); pair(y0 + 2, make_float2(n.z, n.w), live_col);
        Y2 = yt(2); pair(y0 + 4, make_float2(n1.x, n1.y), live_col);
        Y2 = yt(3); pair(y0 + 6, make_float2(n1.z, n1.w), live_col);
        Y2 = yt(4); pair(y0 + 8, make_float2(n2.x, n2.y), live_col);
        Y2 = yt(5); pair(y0 + 10, make_float2(n2.z, n2.w), live_col);
        Y2 = yt(6); pair(y0 + 12, make_float2(n3.x, n3.y), live_col);
        Y2 = yt(7); pair(y0 + 14, make_float2(n3.z, n3.w), live_col);
        return;
      }
#endif
      pair(y0, make_float2(n.x, n.y), live_col);
      pair(y0 + 2, make_float2(n.z, n.w), live_col);
      pair(y0 + 4, make_float2(n1.x, n1.y), live_col);
      pair(y0 + 6, make_float2(n1.z, n1.w), live_col);
      pair(y0 + 8, make_float2(n2.x, n2.y), live_col);
      pair(y0 + 10, make_float2(n2.z, n2.w), live_col);
      pair(y0 + 12, make_float2(n3.x, n3.y), live_col);
      pair(y0 + 14, make_float2(n3.z, n3.w), live_col);
      return;
    }
  }
#pragma unroll 1
  for (int g = 0; g < ng; ++g) {
    const int y = y0 + 4 * g;
    if (!kFull && y >= my) break;
    float4 nn = make_float4(0.f, 0.f, 0.f, 0.f);
    if (noise && g + kPre < ng)
      nn = box_muller4(philox_block(q + static_cast<uint32_t>(kPre) * mxu, pp, rk0, rk1));
    pair(y, make_float2(n.x, n.y), std::false_type());
    if (kFull || y + 2 < my) pair(y + 2, make_float2(n.z, n.w), std::false_type());
    if (kPre == 1) {
      n = nn;
    } else if (kPre == 2) {
      n = n1;
      n1 = nn;
    } else {
      n = n1;
      n1 = n2;
      n2 = n3;
      n3 = nn;
    }
    q += mxu;
  }
}

// The rows of one column: an occluded column (R15: output z in
// the volume's prism) takes the label-only instance, every other column the full
// chain.  The column is one thread, so the test is per thread.
template <class T, bool kLabels, bool kNearest, int kPh, bool kStaged, bool kClamp,
          bool kSameLbl = false, bool kFull = false, int kPre = 1, int kGMode = kGEdge,
          bool kAbs = false, int kLG = 0>
__device__ __forceinline__ void column_rows(const WarpArgs& a, const VolDev& P, const Vol& V,
                                            const View& v, int vi, int X, int Z, int y0, int ng,
                                            float4 n, float4 n1 = make_float4(0.f, 0.f, 0.f, 0.f),
                                            float4 n2 = make_float4(0.f, 0.f, 0.f, 0.f),
                                            float4 n3 = make_float4(0.f, 0.f, 0.f, 0.f)) {
  if ((V.flags & kOcclude) && Z >= P.occ_lo && Z <= P.occ_hi)
    column_rows_impl<T, kLabels, kNearest, kPh, kStaged, kClamp, kSameLbl, kFull, kPre, kGMode,
                     true, kAbs, kLG>(a, P, V, v, vi, X, Z, y0, ng, n, n1, n2, n3);
  else
    column_rows_impl<T, kLabels, kNearest, kPh, kStaged, kClamp, kSameLbl, kFull, kPre, kGMode,
                     false, kAbs, kLG>(a, P, V, v, vi, X, Z, y0, ng, n, n1, n2, n3);
}

__device__ __forceinline__ Vol load_vol(const VolDev& P) {
  Vol V;
  V.A1[0] = P.A[1];
  V.A1[1] = P.A[5];
  V.A1[2] = P.A[9];
  V.sigma = P.sigma;
  V.ws = P.win_s;
  V.wo = P.win_off;
  V.lo = P.clamp_lo;
  V.hi = P.clamp_hi;
  V.gamma = P.gamma;
  V.flags = P.flags;
  return V;
}

template <int kPh>
__device__ __forceinline__ float4 first_normals(const WarpArgs& a, const VolDev& P, const Vol& V,
                                                int X, int Z, int y0) {
#ifdef W3D_DBG_NONOISE
  return make_float4(0.f, 0.f, 0.f, 0.f);
#endif
  if (!(kPh == kPhFull || (V.flags & kNoise))) return make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t gyn = static_cast<uint32_t>((a.my + 3) >> 2);
  const uint32_t q = static_cast<uint32_t>(X) +
                     static_cast<uint32_t>(a.mx) * (gyn * static_cast<uint32_t>(Z) +
                                                    static_cast<uint32_t>(y0 >> 2));
  const PhiloxPrefix pp{P.ph_K0, P.ph_K1, P.ph_K2, P.ph_U3};
  return box_muller4(philox_block(q, pp, kPh == kPhFull ? a.rk0 : P.rk0,
                                  kPh == kPhFull ? a.rk1 : P.rk1));
}

// Every trilinear corner / nearest voxel of the tile inside the volume, from
// the tile's origin coordinate p0 and the per-volume offsets of the box (host,
// cube_cp_box: the box margin bounds the fp32 rounding of every p of the
// tile): lower corner floor(p0 + box_mlo) >= 0, upper corner p0 + box_mhi <
// n - 1, the adds rounded outwards.
__device__ __forceinline__ bool tile_inside(const WarpArgs& a, const VolDev& P, const float p0[3]) {
  const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                      static_cast<float>(a.nz)};
  bool in = true;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    in &= (__fadd_rd(p0[k], P.box_mlo[k]) >= 0.0f) &
          (__fadd_ru(p0[k], P.box_mhi[k]) < n[k] - 1.0f);
  return in;
}

// Every sample of the tile outside the volume on some axis k: all p_k < -1
// (every corner index <= -1, the nearest voxel too) or all p_k > n_k (every
// index >= n_k), from the same per-volume offsets, adds rounded outwards.
__device__ __forceinline__ bool tile_outside(const WarpArgs& a, const VolDev& P, const float p0[3]) {
  const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                      static_cast<float>(a.nz)};
  bool out = false;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    out |= (__fadd_ru(p0[k], P.box_mhi[k]) < -1.0f) | (__fadd_rd(p0[k], P.box_mlo[k]) > n[k]);
  return out;
}

// The tile's coordinates stay below 2^21 (magic-number floor, float indices):
// its origin voxel's p below 2^20 and the footprint extent below 200 (host).
// p0 = p(tile origin voxel), computed once per tile.
__device__ __forceinline__ bool cp_sane(const VolDev& P, int ox, int oy, int oz, float p0[3]) {
  const float X = static_cast<float>(ox), Y = static_cast<float>(oy), Z = static_cast<float>(oz);
  bool sane = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    p0[k] = coord(P.A, k, X, Y, Z);
    sane &= fabsf(p0[k]) < 1048576.0f;
  }
  return sane;
}

#ifdef W3D_CHECK_BOX
// Debug build: after staging (TMA + fix-up, or cp.async) and the barrier that
// publishes it, every cell of the tile's boxes must hold the volume's value
// (in-volume cells) or fill / label_fill (out-of-volume cells, when the box was
// fixed up; a skipped fix-up leaves TMA's zeros, which no sample reads).  This
// checks the async-proxy -> generic-proxy ordering (mbarrier wait, barrier) and
// the fix-up's chunk coverage from inside the kernel (compute-sanitizer is not
// available on this pool).  Traps on the first mismatch.
template <class T>
__device__ __noinline__ void check_box_content(const WarpArgs& a, const VolDev& P, const Box& b,
                                               uint32_t simg, uint32_t slbl, bool labels,
                                               bool img_fixed, bool lbl_fixed) {
  const T* vin = vol_in<T>(P);
  const uint8_t* lin = vol_lbl(P);
  const int64_t sy = a.nx, sz = int64_t(a.nx) * a.ny;
  const uint32_t fw = fill_word<T>(a);
  const int cells = b.W * b.H * b.D;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) {
    const int x = c % b.W, y = (c / b.W) % b.H, z = c / (b.W * b.H);
    const int gx = b.bx + x, gy = b.by + y, gz = b.bz + z;
    const bool in = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny && gz >= 0 && gz < a.nz;
    const uint32_t s = simg + InT<T>::kBytes * static_cast<uint32_t>(z * b.P + y * b.W + x);
    uint32_t got;
    if (InT<T>::kBytes == 4) {
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(got) : "r"(s));
      if (in && got != __float_as_uint(__ldg(reinterpret_cast<const float*>(vin) +
                                             (gz * sz + gy * sy + gx))))
        __trap();
      if (!in && img_fixed && got != fw) __trap();
    } else {
      asm volatile("ld.shared.u16 %0, [%1];" : "=r"(got) : "r"(s));
      const uint16_t want = in ? static_cast<uint16_t>(__ldg(reinterpret_cast<const short*>(vin) +
                                                             (gz * sz + gy * sy + gx)))
                               : static_cast<uint16_t>(fw);
      if ((in || img_fixed) && got != want) __trap();
    }
  }
  if (!labels) return;
  const int hl = b.Pl / b.Wl;  // label rows per plane
  const int lcells = b.Wl * hl * b.D;
  for (int c = threadIdx.x; c < lcells; c += blockDim.x) {
    const int x = c % b.Wl, y = (c / b.Wl) % hl, z = c / (b.Wl * hl);
    if (y >= b.H) continue;  // padding rows of a cp.async box
    const int gx = b.bxl + x, gy = b.by + y, gz = b.bz + z;
    const bool in = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny && gz >= 0 && gz < a.nz;
    uint32_t got;
    asm volatile("ld.shared.u8 %0, [%1];"
                 : "=r"(got)
                 : "r"(slbl + static_cast<uint32_t>(z * b.Pl + y * b.Wl + x)));
    if (in && got != __ldg(lin + (gz * sz + gy * sy + gx))) __trap();
    if (!in && lbl_fixed && got != a.label_fill) __trap();
  }
}
#define W3D_CHECK_CONTENT(T, ...) check_box_content<T>(__VA_ARGS__)
#else
#define W3D_CHECK_CONTENT(T, ...) \
  do {                            \
  } while (0)
#endif

// Rare path (out of line): the tile in y-parts of TY/2, TY/4, ... rows, each
// staged on its own, or gathered when even a 4-row part does not fit (or
// always, for the W3D_KERNEL_GATHER variant).
template <class T, int TY, bool kLabels, bool kNearest, int kPh>
__device__ __forceinline__ void tile_parts(const WarpArgs& a, int cap, bool gather_only, int vi,
                                           int ox, int oy, int oz) {
  const uint32_t simg = smem_base();
  const VolDev& P = a.vol[vi];
  const Vol V = load_vol(P);
  const T* vin = vol_in<T>(P);
  const uint8_t* lin = kLabels ? vol_lbl(P) : nullptr;
  const int lane = threadIdx.x & 31;
  const int X = ox + (lane & 15), Z = oz + 2 * static_cast<int>(threadIdx.x >> 5) + (lane >> 4);
  const bool live = X < a.mx && Z < a.mz;
  const int ylast = min(oy + TY, a.my) - 1;
  int rows = gather_only ? 0 : TY / 2;
  Box b;
  // largest part size whose every part fits
  for (; rows >= 4; rows >>= 1) {
    bool all = true;
    for (int y = oy; y <= ylast; y += rows)
      all &= tile_box<T>(a, P.A, ox, y, min(y + rows - 1, ylast), oz, cap, b);
    if (all) break;
  }
  if (rows < 4) {  // gathers
    if (threadIdx.x == 0) atomicAdd(&g_cube_tiles[1], 1ull);
    if (!live) return;
    View v;
    const float4 n = first_normals<kPh>(a, P, V, X, Z, oy);
    // tile class from the tile's origin coordinate and the per-volume box
    // offsets (uniform): inside / outside / edge (gather2)
    float p0[3];
    const bool sane = cp_sane(P, ox, oy, oz, p0);
    if (a.nx >= (1 << 21) || a.ny >= (1 << 21) || a.nz >= (1 << 21))
      column_rows<T, kLabels, kNearest, kPh, false, false, false, false, 1, kGWide>(
          a, P, V, v, vi, X, Z, oy, TY / 4, n);
    else if (sane && tile_inside(a, P, p0))
      column_rows<T, kLabels, kNearest, kPh, false, false, false, false, 1, kGIn>(
          a, P, V, v, vi, X, Z, oy, TY / 4, n);
    else if (sane && tile_outside(a, P, p0))
      column_rows<T, kLabels, kNearest, kPh, false, false, false, false, 1, kGOut>(
          a, P, V, v, vi, X, Z, oy, TY / 4, n);
    else
      column_rows<T, kLabels, kNearest, kPh, false, false, false, false, 1, kGEdge>(
          a, P, V, v, vi, X, Z, oy, TY / 4, n);
    return;
  }
  if (threadIdx.x == 0) {
    atomicAdd(&g_cube_tiles[0], 1ull);
    atomicAdd(&g_cube_tiles[3], 1ull);
  }
  for (int y = oy; y <= ylast; y += rows) {
    tile_box<T>(a, P.A, ox, y, min(y + rows - 1, ylast), oz, cap, b);
    const uint32_t slbl = simg + InT<T>::kBytes * static_cast<uint32_t>(b.P * b.D);
    __syncthreads();  // previous part's buffer no longer read
    stage<T, kLabels>(a, vin, lin, b, simg, slbl);
    const float4 n = live ? first_normals<kPh>(a, P, V, X, Z, y) : make_float4(0, 0, 0, 0);
    const View v = make_view<T>(a, b, simg, slbl);
    cp_async_wait_all();
    __syncthreads();
    W3D_CHECK_CONTENT(T, a, P, b, simg, slbl, kLabels, true, true);
    if (!live) continue;
    if (b.clamp)
      column_rows<T, kLabels, kNearest, kPh, true, true, true>(a, P, V, v, vi, X, Z, y, rows / 4, n);
    else
      column_rows<T, kLabels, kNearest, kPh, true, false, true>(a, P, V, v, vi, X, Z, y, rows / 4, n);
  }
}

// ---------------------------------------------------------------------------
// TMA image staging: the tile's image footprint box is ONE 3D tensor box of the
// volume (dims fixed per volume, cube_cp_box), loaded by one thread with
// cp.async.bulk.tensor, completion on an mbarrier; out-of-volume elements
// arrive as 0 and boxes that leave the volume get fill written over them before
// the compute (R6).  The label box (1 B elements) goes by cp.async with the
// same pitches: a TMA box row must start 16 B aligned (measured: an unaligned
// inner origin faults), which for labels would cost a 16-element x slack.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}
// Bounded wait: a TMA that never completes traps (a launch error) instead of
// hanging the device.
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  for (uint32_t tries = 0;; ++tries) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred P1;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(mbar), "r"(phase)
        : "memory");
    if (done) return;
    if (tries > (1u << 22)) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            int z, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(mbar)
      : "memory");
}

// Out-of-volume 16 B chunks of a TMA box (TMA wrote 0) set to `word`: a box of
// D planes x Hb rows x CW chunks (rows contiguous: row pitch CW chunks, plane
// pitch Pb bytes) whose origin is (bx, by, bz) in elements of kC per chunk (bx
// and nx multiples of kC, so a chunk is wholly in or out).  Thread t owns one
// (chunk column, row) slot s = t / nsplit and the t % nsplit-th of nsplit
// plane ranges (nsplit = THREADS / slots when the slots are fewer than the
// threads, so small label boxes still spread over every thread): a slot
// outside in x or y is written in every plane of its range, an inside one in
// the planes outside [zlo, zhi) only.  q / d for small q, d by one fp32
// multiply ((q + 1/2) / d is >= 1/(2 d) from an integer; q < 2^16, d <= 2^8:
// error < 2^-8).
__device__ __forceinline__ int small_div(int q, float inv_d) {
  return __float2int_rz(__fmul_rn(static_cast<float>(q) + 0.5f, inv_d));
}
__device__ __forceinline__ void fix_chunks(uint32_t base, int CW, int Hb, uint32_t Pb, int D,
                                           int bx, int by, int bz, int kC, int nx, int ny, int nz,
                                           uint32_t word) {
  const int hc = min(CW, max(0, -bx / kC)), tc = max(hc, min(CW, (nx - bx) / kC));
  const int ylo = min(Hb, max(0, -by)), yhi = max(ylo, min(Hb, ny - by));
  const int zlo = min(D, max(0, -bz)), zhi = max(zlo, min(D, nz - bz));
  const int slots = CW * Hb;
  // plane ranges per slot: 4, 2 or 1 threads share a slot (a power of two: no divisions)
  const int lg = 4 * slots <= THREADS ? 2 : (2 * slots <= THREADS ? 1 : 0);
  const int t = static_cast<int>(threadIdx.x);
  const float inv_cw = __frcp_rn(static_cast<float>(CW));
  const uint4 w4 = make_uint4(word, word, word, word);
  auto st = [&](uint32_t addr) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w4.x), "r"(w4.y),
                 "r"(w4.z), "r"(w4.w)
                 : "memory");
  };
  // the out-of-volume planes of slot s in [zs, ze): all of them when the slot's
  // (chunk column, row) is outside, else those below zlo and from zhi on
  auto slot = [&](int s, int zs, int ze) {
    const int r = small_div(s, inv_cw), c = s - r * CW;
    const bool out = (c < hc) | (c >= tc) | (r < ylo) | (r >= yhi);
    const uint32_t a0 = base + 16u * static_cast<uint32_t>(s);
    if (out) {
      for (int z = zs; z < ze; ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
    } else {
      for (int z = zs; z < min(ze, zlo); ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
      for (int z = max(zs, zhi); z < ze; ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
    }
  };
  if (lg > 0) {
    const int s = t >> lg, part = t & ((1 << lg) - 1);
    if (s < slots) slot(s, (D * part) >> lg, (D * (part + 1)) >> lg);
    return;
  }
  for (int s = t; s < slots; s += THREADS) slot(s, 0, D);
}

#ifdef W3D_OLD_FIXUP  // A/B knob: the round-1 slot scheduling (integer divisions)
__device__ __forceinline__ void fix_chunks_div(uint32_t base, int CW, int Hb, uint32_t Pb, int D,
                                           int bx, int by, int bz, int kC, int nx, int ny, int nz,
                                           uint32_t word) {
  const int hc = min(CW, max(0, -bx / kC)), tc = max(hc, min(CW, (nx - bx) / kC));
  const int ylo = min(Hb, max(0, -by)), yhi = max(ylo, min(Hb, ny - by));
  const int zlo = min(D, max(0, -bz)), zhi = max(zlo, min(D, nz - bz));
  const int slots = CW * Hb;
  const int nsplit = max(1, THREADS / slots);
  const int t = static_cast<int>(threadIdx.x);
  const float inv_cw = __frcp_rn(static_cast<float>(CW));
  auto st = [&](uint32_t addr) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(word) : "memory");
  };
  if (nsplit > 1) {
    const int s = small_div(t, __frcp_rn(static_cast<float>(nsplit)));
    if (s >= slots) return;
    const int part = t - s * nsplit;
    const int zs = (D * part) / nsplit, ze = (D * (part + 1)) / nsplit;
    const int r = small_div(s, inv_cw), c = s - r * CW;
    const bool out = (c < hc) | (c >= tc) | (r < ylo) | (r >= yhi);
    const uint32_t a0 = base + 16u * static_cast<uint32_t>(s);
    for (int z = zs; z < ze; ++z)
      if (out | (z < zlo) | (z >= zhi)) st(a0 + static_cast<uint32_t>(z) * Pb);
    return;
  }
  for (int s = t; s < slots; s += THREADS) {
    const int r = small_div(s, inv_cw), c = s - r * CW;
    const bool out = (c < hc) | (c >= tc) | (r < ylo) | (r >= yhi);
    const uint32_t a0 = base + 16u * static_cast<uint32_t>(s);
    if (out) {
      for (int z = 0; z < D; ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
    } else {
      for (int z = 0; z < zlo; ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
      for (int z = zhi; z < D; ++z) st(a0 + static_cast<uint32_t>(z) * Pb);
    }
  }
}
#define fix_chunks fix_chunks_div
#endif

// fill over the out-of-volume elements of a TMA image box (TMA wrote 0).
template <class T>
__device__ __forceinline__ void tma_fixup(const WarpArgs& a, const Box& b, uint32_t simg) {
  constexpr int kC = InT<T>::kChunk;
  fix_chunks(simg, b.W / kC, b.H, InT<T>::kBytes * static_cast<uint32_t>(b.P), b.D, b.bx, b.by,
             b.bz, kC, a.nx, a.ny, a.nz, fill_word<T>(a));
}

// label_fill over the out-of-volume elements of a TMA label box (rows of Wl
// bytes from bxl, a multiple of 16, as nx is; plane pitch Pl).
__device__ __forceinline__ void tma_fixup_lbl(const WarpArgs& a, const Box& b, uint32_t slbl) {
  fix_chunks(slbl, b.Wl / 16, b.Pl / b.Wl, static_cast<uint32_t>(b.Pl), b.D, b.bxl, b.by, b.bz,
             16, a.nx, a.ny, a.nz, a.label_fill * 0x01010101u);
}



__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void decode_brick(int32_t brick, int& tx, int& ty, int& tz);

// The next volume of the launch into L2, one disjoint slice per tile: tile t of
// volume vi prefetches slice t of volume vi + 1's image and labels (contiguous bytes,
// cp.async.bulk.prefetch.L2), so when that volume's tiles start -- about one volume's
// worth of CTAs later -- their TMA boxes hit in L2 instead of waiting for DRAM.  The
// slices add up to the volume exactly once (no extra DRAM traffic).
template <class T>
__device__ __forceinline__ void prefetch_next_volume(const WarpArgs& a, int vi, int oz, int oy,
                                                     int ox, int TY) {
  const VolDev& N = a.vol[vi + 1];
  const int64_t tiles_x = (a.mx + TX - 1) / TX, tiles_y = (a.my + TY - 1) / TY;
  const int64_t tiles = tiles_x * tiles_y * ((a.mz + TZ - 1) / TZ);
  const int64_t t = ox / TX + tiles_x * (oy / TY + tiles_y * (oz / TZ));
  const int64_t nvox = a.in_stride;
  const int64_t chunk = ((nvox + tiles - 1) / tiles + 15) & ~int64_t(15);  // elements
  const int64_t lo = t * chunk;
  if (lo >= nvox) return;
  const int64_t n = min(chunk, nvox - lo) & ~int64_t(15);
  if (n <= 0) return;
  const uint64_t img = N.in_addr + static_cast<uint64_t>(lo) * InT<T>::kBytes;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(img),
               "r"(static_cast<uint32_t>(n * InT<T>::kBytes))
               : "memory");
  if (N.lbl_addr != 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(N.lbl_addr +
                                                                   static_cast<uint64_t>(lo)),
                 "r"(static_cast<uint32_t>(n))
                 : "memory");
}

// L2 prefetch of the boxes of the tile a.prefetch_ahead CTAs later in launch order
// (same volume only): by the time that CTA issues its TMA the box is in L2 (C4,
// where the box wait -- not dispatch -- bounds the kernel).
template <class T, int TY, bool kTmaLbl>
__device__ __noinline__ void prefetch_ahead(const WarpArgs& a, const VolDev& P, int vi) {
  constexpr int kC = InT<T>::kChunk;
  const uint32_t gx = gridDim.x, gy = gridDim.y;
  const uint32_t tiles_z = static_cast<uint32_t>((a.mz + TZ - 1) / TZ);
  const uint32_t z0 = blockIdx.z - static_cast<uint32_t>(vi) * tiles_z;
  const uint32_t L = blockIdx.x + gx * (blockIdx.y + gy * z0) + static_cast<uint32_t>(a.prefetch_ahead);
  if (L >= gx * gy * tiles_z) return;
  int tx = static_cast<int>(L % gx), ty = static_cast<int>((L / gx) % gy);
  int tz = static_cast<int>(L / (gx * gy));
  if (a.brick) decode_brick(a.brick, tx, ty, tz);
  float p0[3];
  const float X = static_cast<float>(tx * TX), Y = static_cast<float>(ty * TY),
              Z = static_cast<float>(tz * TZ);
  for (int k = 0; k < 3; ++k) p0[k] = coord(P.A, k, X, Y, Z);
  if (!(fabsf(p0[0]) < 1048576.0f && fabsf(p0[1]) < 1048576.0f && fabsf(p0[2]) < 1048576.0f)) return;
  const int bx = __float2int_rd(__fadd_rd(p0[0], P.box_mlo[0])) & ~(kC - 1);
  const int by = __float2int_rd(__fadd_rd(p0[1], P.box_mlo[1]));
  const int bz = __float2int_rd(__fadd_rd(p0[2], P.box_mlo[2]));
  tma_prefetch_3d(&a.tm[2 * vi], bx, by, bz);
  if (kTmaLbl) tma_prefetch_3d(&a.tm[2 * vi + 1], bx & ~15, by, bz);
}

// The common path: the whole tile staged as ONE box of the volume's fixed dims
// (cp_w, cp_h, cp_d; host-computed by cube_cp_box to hold any tile's
// footprint) whose origin follows from the tile's origin voxel alone -- every
// value here is CTA-uniform (no per-tile corner reduction; the view's pitches
// sit in uniform registers, folded into the shared-memory addresses).  The
// image box comes by TMA when the volume has a tensor map (tma), else by
// cp.async; the labels by cp.async.
// kTmaLbl: the label box comes by TMA too (its own tensor map; rows of box_wl
// bytes from a 16 B aligned x origin, box_h rows per plane) and the tile waits
// on the mbarrier alone.
template <class T, int TY, bool kLabels, bool kNearest, int kPh, bool kTmaLbl = false>
__device__ __forceinline__ void cp_tile(const WarpArgs& a, const VolDev& P, int vi, int ox, int oy,
                                        int oz, bool tma, uint32_t mbar, const float p0[3],
                                        uint32_t phase = 0u, bool init = true) {
  constexpr int kC = InT<T>::kChunk;
  constexpr uint32_t kB = InT<T>::kBytes;
  // A/B knob W3D_LBL_GATHER: 8-row tiles gather their labels from global memory
  // instead of staging a label box (half the TMA rows) -- measured slower on C4
  // (164 vs 190 GVoxel/s: the rotated gathers stall the rows more than the box wait
  // they save), so off
#if defined(W3D_LBL_GATHER_ALL)  // A/B knob: every fixed-box tile
  constexpr bool kLblG = kLabels && !kNearest;
#elif defined(W3D_LBL_GATHER)
  constexpr bool kLblG = kLabels && !kNearest && TY < kTY;
#else
  constexpr bool kLblG = false;
#endif
  constexpr bool kTmaL = kTmaLbl && !kLblG;  // a label box by TMA
  const uint32_t simg = smem_base();
#ifdef W3D_DBG_TIMING  // diagnostic: per-tile phase times of a few CTAs (printf)
  const long long dbg_t0 = clock64();
  long long dbg_t[5] = {0, 0, 0, 0, 0};
#define W3D_T(i) dbg_t[i] = clock64() - dbg_t0
#else
#define W3D_T(i) \
  do {           \
  } while (0)
#endif
  Box b;
  b.W = P.cp_w;
  b.H = P.cp_h;
  b.D = P.cp_d;
  b.P = P.cp_p;
  b.Wl = b.W;
  b.Pl = b.P;
  b.clamp = false;
  b.bx = __float2int_rd(__fadd_rd(p0[0], P.box_mlo[0])) & ~(kC - 1);
  b.by = __float2int_rd(__fadd_rd(p0[1], P.box_mlo[1]));
  b.bz = __float2int_rd(__fadd_rd(p0[2], P.box_mlo[2]));
  b.bxl = kTmaLbl ? (b.bx & ~15) : b.bx;
  if (kTmaLbl) {
    b.Wl = P.box_wl;
    b.Pl = b.Wl * P.box_h;
  }
  const uint32_t slbl = simg + ((kB * static_cast<uint32_t>(b.P * b.D) + 127u) & ~127u);
  const Vol V = load_vol(P);
  const T* vin = vol_in<T>(P);
  const uint8_t* lin = kLabels ? vol_lbl(P) : nullptr;
  const int lane = threadIdx.x & 31;
  const int X = ox + (lane & 15), Z = oz + 2 * static_cast<int>(threadIdx.x >> 5) + (lane >> 4);
  const bool live = X < a.mx && Z < a.mz;
  if (tma) {
    if (threadIdx.x == 0) {
      if (init) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      mbar_expect_tx(mbar, kB * static_cast<uint32_t>(b.P * b.D) +
                               (kTmaL ? static_cast<uint32_t>(b.Pl * b.D) : 0u));
      tma_load_3d(simg, &a.tm[2 * vi], b.bx, b.by, b.bz, mbar);
      if (kTmaL) tma_load_3d(slbl, &a.tm[2 * vi + 1], b.bxl, b.by, b.bz, mbar);
    }
    if (a.prefetch_ahead > 0 && threadIdx.x == 32)  // another warp than the issuer
      prefetch_ahead<T, TY, kTmaLbl>(a, P, vi);
#ifdef W3D_VOLPF  // A/B knob, off: no gain measured (274.0 vs 275.0) and +5 % DRAM reads
    if (threadIdx.x == 64 && vi + 1 < a.nvol) prefetch_next_volume<T>(a, vi, oz, oy, ox, TY);
#endif
    if (kLabels && !kTmaLbl && !kLblG) stage_lbl<T>(a, lin, b, slbl);
  } else {
    stage<T, kLabels && !kLblG>(a, vin, lin, b, simg, slbl);
  }
#ifdef W3D_EARLY_BAR
  // A/B knob: with image and labels both by TMA the barrier only publishes the
  // mbarrier init and could come before the Philox prologue -- measured slower
  // (266.7 vs 272.5 GVoxel/s, profiles/round2/HISTORY.md r3k): the barrier after
  // the prologue re-aligns the CTA's warps before the straight-line rows
  constexpr bool kEarlyBar = kTmaLbl;
#else
  constexpr bool kEarlyBar = false;
#endif
  W3D_T(0);  // TMA issued
  if (kEarlyBar) __syncthreads();
  // an occluded column (R15) needs no noise: its Philox blocks are skipped
#ifndef W3D_DBG_NONOISE
  const bool need_noise = live && !((P.flags & kOcclude) && Z >= P.occ_lo && Z <= P.occ_hi);
#else
  const bool need_noise = false;  // diagnostic knock-out: no Philox / Box-Muller at all
#endif
  // the training chain (kPhFull, launch-wide keys) computes kPre Philox blocks
  // here, under the staging latency (at most the tile's TY / 4); the generic
  // chain one (register budget)
  constexpr int kPre = kPh == kPhFull ? (W3D_PRE < TY / 4 ? W3D_PRE : TY / 4) : 1;
  float4 n = (need_noise && kPre != 4 && !(kPre == 2 && kPh == kPhFull))
                  ? first_normals<kPh>(a, P, V, X, Z, oy)
                  : make_float4(0, 0, 0, 0);
  const float4 z4 = make_float4(0, 0, 0, 0);
  float4 n1 = z4, n2 = z4, n3 = z4;
  if (kPre == 4 && need_noise) {  // the column's four blocks in lockstep
    const uint32_t gyn = static_cast<uint32_t>((a.my + 3) >> 2), mxu = static_cast<uint32_t>(a.mx);
    const uint32_t q0 = static_cast<uint32_t>(X) +
                        mxu * (gyn * static_cast<uint32_t>(Z) + static_cast<uint32_t>(oy >> 2));
    const uint32_t qs[4] = {q0, q0 + mxu, q0 + 2u * mxu, q0 + 3u * mxu};
    uint4 r[4];
    philox_block4<4>(qs, PhiloxPrefix{P.ph_K0, P.ph_K1, P.ph_K2, P.ph_U3}, a.rk0, a.rk1, r);
    n = box_muller4(r[0]);
    n1 = box_muller4(r[1]);
    n2 = box_muller4(r[2]);
    n3 = box_muller4(r[3]);
  } else if (kPre == 2 && kPh == kPhFull && need_noise) {  // 8-row tiles: two in lockstep
    const uint32_t gyn = static_cast<uint32_t>((a.my + 3) >> 2), mxu = static_cast<uint32_t>(a.mx);
    const uint32_t q0 = static_cast<uint32_t>(X) +
                        mxu * (gyn * static_cast<uint32_t>(Z) + static_cast<uint32_t>(oy >> 2));
    const uint32_t qs[2] = {q0, q0 + mxu};
    uint4 r[2];
    philox_block4<2>(qs, PhiloxPrefix{P.ph_K0, P.ph_K1, P.ph_K2, P.ph_U3}, a.rk0, a.rk1, r);
    n = box_muller4(r[0]);
    n1 = box_muller4(r[1]);
  } else if (kPre == 2 && need_noise) {
    n1 = first_normals<kPh>(a, P, V, X, Z, oy + 4);
  }
  View v = make_view<T>(a, b, simg, slbl);
  v.W4 = P.cp_w_bytes;  // straight from the parameters: uniform registers, folded
  v.P4 = P.cp_p_bytes;  // into the shared-memory addresses ([R + UR])
  v.PW4 = static_cast<uint32_t>(P.cp_w_bytes) + static_cast<uint32_t>(P.cp_p_bytes);
  // absolute index (sample2 kAbs, host-checked P.cp_abs): the box origin in y and z
  // moves from the float index into the address constants
  if (kUseAbs) {
    v.cimg = opaque(v.cimg - kB * static_cast<uint32_t>(b.W * b.by + b.P * b.bz));
    v.clbl = opaque(v.clbl - static_cast<uint32_t>(b.Wl * b.by + b.Pl * b.bz));
  }
  // which boxes need a fix-up: decided before the barrier and the box wait (under
  // the staging latency), not after them on the tile's critical path
  const bool inside = b.bx >= 0 && b.by >= 0 && b.bz >= 0 && b.bx + b.W <= a.nx &&
                      b.by + b.H <= a.ny && b.bz + b.D <= a.nz;
  const bool insidel = !kTmaL || (b.bxl >= 0 && b.bxl + b.Wl <= a.nx &&
                                  b.by + b.Pl / b.Wl <= a.ny && inside);
  bool fi = tma && !inside && a.fill != 0.0f, fl = tma && kTmaL && !insidel && a.label_fill != 0u;
  // boxes carry margins: skip the fix-up when no sample of the tile can read
  // an out-of-volume cell (every trilinear corner and nearest voxel inside)
  if ((fi || fl) && tile_inside(a, P, p0)) fi = fl = false;
  if (!kTmaL) cp_async_wait_all();
  W3D_T(1);  // Philox prologue done
  if (!kEarlyBar) __syncthreads();  // label copies (and the mbarrier init) visible to all
  W3D_T(2);  // barrier passed
  if (tma) {
#ifndef W3D_DBG_LATEWAIT
    mbar_wait(mbar, phase);
#endif
    W3D_T(3);  // box landed
    if (fi || fl) {  // uniform
      if (fi) tma_fixup<T>(a, b, simg);
      if (fl) tma_fixup_lbl(a, b, slbl);
      __syncthreads();
    }
    // zero fill / label_fill equal TMA's out-of-volume zeros: fixed without a fix-up
    W3D_CHECK_CONTENT(T, a, P, b, simg, slbl, kLabels && !kLblG,
                      fi || (inside || a.fill == 0.0f), !kTmaL || fl || (insidel || a.label_fill == 0u));
  } else {
    W3D_CHECK_CONTENT(T, a, P, b, simg, slbl, kLabels && !kLblG, true, true);
  }
#ifdef W3D_DBG_LATEWAIT  // diagnostic: compute as if the box had arrived (garbage outputs)
  const bool late_wait = true;
#endif
  if (live) {
    if constexpr (kLblG) {  // gathered labels: unchecked when no sample can leave the volume
      const bool edge = !tile_inside(a, P, p0);
      if (oy + TY <= a.my && !edge)
        column_rows<T, kLabels, kNearest, kPh, true, false, !kTmaLbl, true, kPre, kGEdge, kUseAbs,
                    1>(a, P, V, v, vi, X, Z, oy, TY / 4, n, n1, n2, n3);
      else if (oy + TY <= a.my)
        column_rows<T, kLabels, kNearest, kPh, true, false, !kTmaLbl, true, kPre, kGEdge, kUseAbs,
                    2>(a, P, V, v, vi, X, Z, oy, TY / 4, n, n1, n2, n3);
      else
        column_rows<T, kLabels, kNearest, kPh, true, false, !kTmaLbl, false, kPre, kGEdge, kUseAbs,
                    2>(a, P, V, v, vi, X, Z, oy, TY / 4, n, n1, n2, n3);
    } else {
      if (oy + TY <= a.my)  // every row of the tile is an output row
        column_rows<T, kLabels, kNearest, kPh, true, false, !kTmaLbl, true, kPre, kGEdge, kUseAbs>(
            a, P, V, v, vi, X, Z, oy, TY / 4, n, n1, n2, n3);
      else
        column_rows<T, kLabels, kNearest, kPh, true, false, !kTmaLbl, false, kPre, kGEdge, kUseAbs>(
            a, P, V, v, vi, X, Z, oy, TY / 4, n, n1, n2, n3);
    }
  }
#ifdef W3D_DBG_LATEWAIT
  if (tma && late_wait) mbar_wait(mbar, phase);
#endif
  W3D_T(4);  // rows done
#ifdef W3D_DBG_TIMING
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 3 && blockIdx.y == 3 && blockIdx.z % 37 == 0)
    printf("W3DT z %d warp %d: issue %lld philox %lld bar %lld box %lld rows %lld\n",
           blockIdx.z, threadIdx.x >> 5, dbg_t[0], dbg_t[1], dbg_t[2], dbg_t[3], dbg_t[4]);
#endif
#undef W3D_T
}

// One output tile (volume vi, origin ox, oy, oz).  mbar / phase: the CTA's
// TMA mbarrier and the parity of its next phase (init: initialise it here, the
// one-tile-per-CTA grid).  Returns true when the tile used the mbarrier.
template <class T, int TY, bool kLabels, bool kNearest, int kPh, bool kGather>
__device__ __forceinline__ bool cube_tile(const WarpArgs& a, int cap, int vi, int ox, int oy,
                                          int oz, uint32_t mbar, uint32_t phase, bool init) {
  const uint32_t simg = smem_base();
  const VolDev& P = a.vol[vi];
  const int ylast = min(oy + TY, a.my) - 1;
  float p0[3];
  if (!kGather && P.cp_rows == TY && cp_sane(P, ox, oy, oz, p0)) {
    const bool tma = a.use_tma && vi < kTmaVolPerLaunch && P.box_w != 0;
    if (threadIdx.x == 0) atomicAdd(&g_cube_tiles[tma ? 2 : 0], 1ull);
    if (kLabels && tma && P.box_wl != 0)
      cp_tile<T, TY, kLabels, kNearest, kPh, true>(a, P, vi, ox, oy, oz, true, mbar, p0, phase,
                                                   init);
    else
      cp_tile<T, TY, kLabels, kNearest, kPh>(a, P, vi, ox, oy, oz, tma, mbar, p0, phase, init);
    return tma;
  }
  // per-tile exact boxes (volumes whose worst-case box does not fit)
  Box b;
  if (kGather || !tile_box<T>(a, P.A, ox, oy, ylast, oz, cap, b)) {
    tile_parts<T, TY, kLabels, kNearest, kPh>(a, cap, kGather, vi, ox, oy, oz);
    return false;
  }
  if (threadIdx.x == 0) atomicAdd(&g_cube_tiles[0], 1ull);
  const uint32_t slbl = simg + InT<T>::kBytes * static_cast<uint32_t>(b.P * b.D);
#ifndef W3D_DBG_NOSTAGE
  stage<T, kLabels>(a, vol_in<T>(P), kLabels ? vol_lbl(P) : nullptr, b, simg, slbl);
#endif
  const Vol V = load_vol(P);
  const int lane = threadIdx.x & 31;
  const int X = ox + (lane & 15), Z = oz + 2 * static_cast<int>(threadIdx.x >> 5) + (lane >> 4);
  const bool live = X < a.mx && Z < a.mz;
  // the first Philox block overlaps the copies in flight
  const float4 n = live ? first_normals<kPh>(a, P, V, X, Z, oy) : make_float4(0, 0, 0, 0);
  const View v = make_view<T>(a, b, simg, slbl);
  cp_async_wait_all();
  __syncthreads();
  W3D_CHECK_CONTENT(T, a, P, b, simg, slbl, kLabels, true, true);
  if (!live) return false;
#ifdef W3D_DBG_NOCOMPUTE
  if (n.x == 12345.0f) a.out[X] = n.y;  // keep the first Philox block alive
  return false;
#endif
  if (b.clamp)
    column_rows<T, kLabels, kNearest, kPh, true, true, true>(a, P, V, v, vi, X, Z, oy, TY / 4, n);
  else
    column_rows<T, kLabels, kNearest, kPh, true, false, true>(a, P, V, v, vi, X, Z, oy, TY / 4, n);
  return false;
}

// Launch order (x, y, z fastest to slowest, within one volume) -> bricks of
// 2^sx x 2^sy x 2^sz tiles (WarpArgs::brick; shifts and masks only).
__device__ __forceinline__ void decode_brick(int32_t brick, int& tx, int& ty, int& tz) {
  const uint32_t f = static_cast<uint32_t>(brick);
  const int sx = f & 15, sy = (f >> 4) & 15, sz = (f >> 8) & 15, lbx = (f >> 12) & 15,
            lby = (f >> 16) & 15;
  const uint32_t L = static_cast<uint32_t>(tx) +
                     gridDim.x * (static_cast<uint32_t>(ty) + gridDim.y * static_cast<uint32_t>(tz));
  const uint32_t w = L & ((1u << (sx + sy + sz)) - 1u), bi = L >> (sx + sy + sz);
  tx = static_cast<int>(((bi & ((1u << lbx) - 1u)) << sx) | (w & ((1u << sx) - 1u)));
  ty = static_cast<int>((((bi >> lbx) & ((1u << lby) - 1u)) << sy) | ((w >> sx) & ((1u << sy) - 1u)));
  tz = static_cast<int>(((bi >> (lbx + lby)) << sz) | (w >> (sx + sy)));
}

// grid = (tiles_x, tiles_y, tiles_z * volumes): one tile per CTA, tiles
// x-fastest, then y, then z.  (A persistent grid of 3 CTAs per SM walking the
// tiles with the mbarrier phase carried across tiles measured 207 vs 272
// GVoxel/s on C3: each CTA's staging latency is exposed between its tiles.)
template <class T, int TY, int MINB, bool kLabels, bool kNearest, int kPh, bool kGather, int NV>
__global__ void __launch_bounds__(THREADS, MINB)
    warp3d_cube_kernel(const __grid_constant__ WarpArgsT<NV> an, const int tiles_z, const int cap,
                       const uint32_t tz_magic) {
  // the WarpArgs prefix of the parameter block (vol[vi] read for vi < nvol <= NV only)
  const WarpArgs& a = reinterpret_cast<const WarpArgs&>(an);
  __shared__ __align__(8) unsigned long long s_mbar;
  // let a programmatic dependent launch (the next chunk of the same call,
  // WarpArgs::pdl) start as this grid's last CTAs run; a no-op otherwise
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
  // vi = blockIdx.z / tiles_z by multiply-high with tz_magic = ceil(2^32 /
  // tiles_z) (exact for operands < 2^16)
  const int vi = tiles_z == 1 ? static_cast<int>(blockIdx.z)
                              : static_cast<int>(__umulhi(blockIdx.z, tz_magic));
  int tx = static_cast<int>(blockIdx.x), ty = static_cast<int>(blockIdx.y);
  int tz = static_cast<int>(blockIdx.z) - vi * tiles_z;
  if (a.brick) decode_brick(a.brick, tx, ty, tz);
  const int ox = tx * TX, oy = ty * TY, oz = tz * TZ;
  cube_tile<T, TY, kLabels, kNearest, kPh, kGather>(a, cap, vi, ox, oy, oz, mbar, 0u, true);
  // A programmatic dependent (a later chunk of the same call) never reads its
  // primary's output, but the grid must not COMPLETE before its primary: work
  // ordered after the call on the stream (events, copies, the next kernel)
  // waits for the last chunk only.  Waiting here, after the tile's stores,
  // keeps the overlap of the whole tile with the primary's last wave (PTX:
  // griddepcontrol.wait; a no-op when the launch has no primary).
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Launch
// ---------------------------------------------------------------------------

template <class T, bool kLabels, bool kNearest, int kPh, bool kGather, int NV, int TY = kTY>
static cudaError_t launch_n(const WarpArgsT<NV>& a, cudaStream_t s) {
  const int tiles_x = (a.mx + TX - 1) / TX, tiles_y = (a.my + TY - 1) / TY;
  const int tiles_z = (a.mz + TZ - 1) / TZ;
  if (tiles_y > 65535 || int64_t(tiles_z) * a.nvol > 65535) return cudaErrorInvalidConfiguration;
  const size_t smem = kGather ? 0 : static_cast<size_t>(kCapVox) * 5 + 256;
  const int cap = kCapVox * 5 / (InT<T>::kBytes + 1);  // staged voxels (image + label bytes)
  // the dynamic shared-memory opt-in is a per-device function attribute: one
  // bit per device ordinal (a process may drive several GPUs)
  static std::atomic<uint64_t> configured{0};
  if (!kGather) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
      const cudaError_t e = cudaFuncSetAttribute(
          warp3d_cube_kernel<T, TY, kGather ? kGMinB : kMinB, kLabels, kNearest, kPh, kGather, NV>,
          cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      configured.fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  const dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y),
                  static_cast<unsigned>(tiles_z * a.nvol));
  const uint32_t tz_magic =
      tiles_z > 1 ? static_cast<uint32_t>(((uint64_t(1) << 32) + tiles_z - 1) / tiles_z) : 0u;
  if (!a.pdl) {
    warp3d_cube_kernel<T, TY, kGather ? kGMinB : kMinB, kLabels, kNearest, kPh, kGather, NV>
        <<<grid, THREADS, smem, s>>>(a, tiles_z, cap, tz_magic);
    return cudaGetLastError();
  }
  // a later chunk of the same call: its CTAs may start while the previous
  // chunk's last wave drains (every CTA triggers its dependents on entry, so
  // the dependent launches only once every CTA of the primary is resident; the
  // chunks share no data, so a CTA computes and stores its whole tile first and
  // waits for the primary's completion only before it exits -- the grids
  // complete in stream order)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(
      &cfg, warp3d_cube_kernel<T, TY, kGather ? kGMinB : kMinB, kLabels, kNearest, kPh, kGather, NV>,
      a, tiles_z, cap, tz_magic);
}

// The full photometric chain on every volume of the launch (the training
// configuration): noise, window + clamp to [0, 1], gamma != 1, with or without
// occlusion (R15: per-column test in column_rows).
// ... and one seed for every volume (the round keys are launch constants, a.rk*).
template <int NV>
static bool all_full(const WarpArgsT<NV>& a) {
  for (int i = 0; i < a.nvol; ++i) {
    const VolDev& P = a.vol[i];
    if ((P.flags & ~kOcclude) != (kNoise | kGamma) || P.clamp_lo != 0.0f || P.clamp_hi != 1.0f)
      return false;
    if (P.rk0[0] != a.vol[0].rk0[0] || P.rk1[0] != a.vol[0].rk1[0]) return false;
  }
  return true;
}

// Every kernel instance of one (image type, parameter block) pair; explicitly
// instantiated once per pair in cube_inst_*.cu (parallel compilation units).
template <class T, int NV>
cudaError_t launch_typed_nv(const WarpArgsT<NV>& a, bool gather_only, cudaStream_t s) {
  const bool labels = a.in_lbl != nullptr;
  const bool nearest = a.interp == W3D_INTERP_NEAREST;
  if (gather_only) {
    if (nearest)
      return labels ? launch_n<T, true, true, kPhGeneric, true>(a, s)
                    : launch_n<T, false, true, kPhGeneric, true>(a, s);
    return labels ? launch_n<T, true, false, kPhGeneric, true>(a, s)
                  : launch_n<T, false, false, kPhGeneric, true>(a, s);
  }
  if (a.tile_rows == kTY / 2 && !nearest) {  // AUTO's 8-row tiles (large footprints)
    if (all_full(a))
      return labels ? launch_n<T, true, false, kPhFull, false, NV, kTY / 2>(a, s)
                    : launch_n<T, false, false, kPhFull, false, NV, kTY / 2>(a, s);
    return labels ? launch_n<T, true, false, kPhGeneric, false, NV, kTY / 2>(a, s)
                  : launch_n<T, false, false, kPhGeneric, false, NV, kTY / 2>(a, s);
  }
  if (a.tile_rows != kTY) return cudaErrorInvalidValue;
  if (nearest)
    return labels ? launch_n<T, true, true, kPhGeneric, false>(a, s)
                  : launch_n<T, false, true, kPhGeneric, false>(a, s);
  if (all_full(a))
    return labels ? launch_n<T, true, false, kPhFull, false>(a, s)
                  : launch_n<T, false, false, kPhFull, false>(a, s);
  return labels ? launch_n<T, true, false, kPhGeneric, false>(a, s)
                : launch_n<T, false, false, kPhGeneric, false>(a, s);
}

// this unit's tile counters (warp3d_tile_stats)
template <class T, int NV>
cudaError_t read_stats_nv(unsigned long long out[4]) {
  return cudaMemcpyFromSymbol(out, g_cube_tiles, 4 * sizeof(unsigned long long));
}

}  // namespace cube
}  // namespace w3d
