// warp3d_kernels.cu -- sm_100a kernels of the Sec. IV augmentation path
// (Rister et al., arXiv 1811.11226).
//
// One pass per output voxel, in the paper's order:
//   occlusion test -> p = A x + b -> image/label sample -> noise -> window -> gamma
// The arithmetic contract is DESIGN.md readings R1-R21.  Compiled without
// fast-math and with -fmad=false: every FMA below is an explicit __fmaf_rn.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "philox.cuh"
#include "warp3d_internal.cuh"

namespace w3d {

// ----------------------------------------------------------------------------
// Shared per-voxel pieces
// ----------------------------------------------------------------------------
extern __shared__ __align__(16) unsigned char g_smem[];

// Diagnostics (warp3d_tile_stats): tiles computed from a staged box / by gathers.
__device__ unsigned long long g_tiles_staged = 0, g_tiles_gather = 0;
__device__ __forceinline__ void count_tile(bool staged) {
  if (threadIdx.x == 0) atomicAdd(staged ? &g_tiles_staged : &g_tiles_gather, 1ull);
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
// packed fp32x2 (sm_100 FADD2/FFMA2): per-lane IEEE rounding identical to scalar
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// lerp(a, b, t) = a + t (b - a): one rounding for the difference, one FMA (R5).
__device__ __forceinline__ float lerp(float a, float b, float t) {
  return __fmaf_rn(t, __fsub_rn(b, a), a);
}
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t) {
  return __ffma2_rn(t, sub2(b, a), a);
}

// Per-volume parameters held in registers for the whole CTA (uniform).
struct Params {
  float A[12];
  float sigma, win_s, win_off, lo, hi, gamma;
  uint32_t flags, vid0, vid1;
  int occ_lo, occ_hi;
  uint32_t rk0[10], rk1[10];
};

__device__ __forceinline__ Params load_params(const VolDev& P) {
  Params p;
#pragma unroll
  for (int k = 0; k < 12; ++k) p.A[k] = P.A[k];
  p.sigma = P.sigma; p.win_s = P.win_s; p.win_off = P.win_off;
  p.lo = P.clamp_lo; p.hi = P.clamp_hi; p.gamma = P.gamma;
  p.flags = P.flags; p.vid0 = P.vid0; p.vid1 = P.vid1;
  p.occ_lo = P.occ_lo; p.occ_hi = P.occ_hi;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    p.rk0[r] = P.rk0[r];
    p.rk1[r] = P.rk1[r];
  }
  return p;
}

// Photometric tail for two voxels (PAPER.md:440-467 + gamma, R9-R14), branch
// free: disabled steps carry neutral parameters (VolDev).
__device__ __forceinline__ float2 photometric2(float2 v, float2 n, const Params& p) {
  v = __ffma2_rn(f2(p.sigma), n, v);                      // I + sigma n
  float2 w = __ffma2_rn(v, f2(p.win_s), f2(p.win_off));   // (I - a) / (b - a)
  w.x = fminf(fmaxf(w.x, p.lo), p.hi);                    // clamp to [0, 1]
  w.y = fminf(fmaxf(w.y, p.lo), p.hi);
  if (p.flags & kGamma) {                                 // w^gamma
    const float2 l = __fmul2_rn(make_float2(lg2_approx(w.x), lg2_approx(w.y)), f2(p.gamma));
    w = make_float2(ex2_approx(l.x), ex2_approx(l.y));
  }
  return w;
}

// Normals of the 4 voxels (rows y = 4g .. 4g+3) of Philox block q (R10).
__device__ __forceinline__ void normals4(uint32_t q, const Params& P, float n[4]) {
  const uint4 r = philox4x32_10_rk(make_uint4(q, 0u, P.vid0, P.vid1), P.rk0, P.rk1);
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
// Staged sampling of two voxels: the CTA's source footprint box is in shared
// memory (g_smem) with `fill` / `label_fill` in its out-of-volume part, so no
// per-corner predicate is needed.  Tiles whose transformed corners leave
// [-1, n] clamp p to [-1, n] first: a clamped coordinate reads only pad voxels
// or gets weight 0 on in-volume ones, which reproduces the border-fill rule
// (R6) and the label rule (R8) exactly.
// ----------------------------------------------------------------------------
struct Stage {
  int W, HW;            // image row / plane pitch (elements)
  int WL, HWL;          // label row / plane pitch (kSepLbl layouts; else = W, HW)
  int img_off, lbl_off; // byte offsets of this buffer's image / label regions in g_smem
  float bx, by, bz;     // box origin (input voxel coords of element 0)
  float Wf, HWf, WLf, HWLf;
  float nx, ny, nz;     // clamp bounds
};

template <bool kLabels, bool kNearest, bool kClamp, bool kSepLbl>
__device__ __forceinline__ void sample_staged2(const Stage& v, float2 px, float2 py, float2 pz,
                                               bool want_img, float2& img, uint32_t& l0,
                                               uint32_t& l1) {
  const float* simg = reinterpret_cast<const float*>(g_smem + v.img_off);
  const uint8_t* slbl = g_smem + v.lbl_off;
  if (kClamp) {
    px = make_float2(fminf(fmaxf(px.x, -1.0f), v.nx), fminf(fmaxf(px.y, -1.0f), v.nx));
    py = make_float2(fminf(fmaxf(py.x, -1.0f), v.ny), fminf(fmaxf(py.y, -1.0f), v.ny));
    pz = make_float2(fminf(fmaxf(pz.x, -1.0f), v.nz), fminf(fmaxf(pz.y, -1.0f), v.nz));
  }
  const float2 fx = make_float2(floorf(px.x), floorf(px.y));
  const float2 fy = make_float2(floorf(py.x), floorf(py.y));
  const float2 fz = make_float2(floorf(pz.x), floorf(pz.y));
  const float2 tx = sub2(px, fx), ty = sub2(py, fy), tz = sub2(pz, fz);
  // local element index: all terms are small integers, exact in fp32
  const float2 rx = sub2(fx, f2(v.bx)), ry = sub2(fy, f2(v.by)), rz = sub2(fz, f2(v.bz));
  const float2 lf = __ffma2_rn(rz, f2(v.HWf), __ffma2_rn(ry, f2(v.Wf), rx));
  const int li0 = __float2int_rz(lf.x), li1 = __float2int_rz(lf.y);
  int ln0 = 0, ln1 = 0;
  if (kNearest || (kLabels && !kSepLbl)) {
    ln0 = li0 + (tx.x >= 0.5f ? 1 : 0) + (ty.x >= 0.5f ? v.W : 0) + (tz.x >= 0.5f ? v.HW : 0);
    ln1 = li1 + (tx.y >= 0.5f ? 1 : 0) + (ty.y >= 0.5f ? v.W : 0) + (tz.y >= 0.5f ? v.HW : 0);
  }
  if (kLabels) {
    if (kSepLbl) {  // label box with its own pitches (TMA layout)
      const float2 lfl = __ffma2_rn(rz, f2(v.HWLf), __ffma2_rn(ry, f2(v.WLf), rx));
      const int m0 = __float2int_rz(lfl.x), m1 = __float2int_rz(lfl.y);
      l0 = slbl[m0 + (tx.x >= 0.5f ? 1 : 0) + (ty.x >= 0.5f ? v.WL : 0) +
                (tz.x >= 0.5f ? v.HWL : 0)];
      l1 = slbl[m1 + (tx.y >= 0.5f ? 1 : 0) + (ty.y >= 0.5f ? v.WL : 0) +
                (tz.y >= 0.5f ? v.HWL : 0)];
    } else {
      l0 = slbl[ln0];
      l1 = slbl[ln1];
    }
  }
  if (!want_img) return;
  if (kNearest) {
    img = make_float2(simg[ln0], simg[ln1]);
    return;
  }
  const float* b0 = simg + li0;
  const float* b1 = simg + li1;
  const int W = v.W, HW = v.HW;
  const float2 c000 = make_float2(b0[0], b1[0]), c100 = make_float2(b0[1], b1[1]);
  const float2 c010 = make_float2(b0[W], b1[W]), c110 = make_float2(b0[W + 1], b1[W + 1]);
  const float2 c001 = make_float2(b0[HW], b1[HW]), c101 = make_float2(b0[HW + 1], b1[HW + 1]);
  const float2 c011 = make_float2(b0[HW + W], b1[HW + W]);
  const float2 c111 = make_float2(b0[HW + W + 1], b1[HW + W + 1]);
  const float2 c00 = lerp2(c000, c100, tx), c10 = lerp2(c010, c110, tx);
  const float2 c01 = lerp2(c001, c101, tx), c11 = lerp2(c011, c111, tx);
  img = lerp2(lerp2(c00, c10, ty), lerp2(c01, c11, ty), tz);
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ----------------------------------------------------------------------------
// Tile shapes.  Lane = output x (a warp covers 32 consecutive x of one row, so
// stores are 128 B + 32 B and shared-memory gathers stay bank-friendly); warp
// w covers z = w % TZ and the y-rows [yh * RPT, (yh + 1) * RPT), yh = w / TZ.
// ----------------------------------------------------------------------------
template <int TX_, int TY_, int TZ_, int THREADS_>
struct Shape {
  static constexpr int TX = TX_, TY = TY_, TZ = TZ_, THREADS = THREADS_;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int RPT = TY * TZ / WARPS;  // rows per thread
  static_assert(TX == 32 && WARPS % TZ == 0 && RPT % 4 == 0 && TY % RPT == 0, "shape");
};
// One-tile-per-CTA configurations: shape, CTAs per SM (register bound) and the
// staging capacity in voxels (shared memory: CTAS * (CAP * 5 B + 1 KB) <= 228 KB).
template <class S_, int MINB_, int CAP_>
struct TileCfg {
  using S = S_;
  static constexpr int MINB = MINB_, CAP = CAP_;
};
using CfgA = TileCfg<Shape<32, 16, 8, 256>, 2, 16384>;  // 16 rows / thread
using CfgB = TileCfg<Shape<32, 8, 8, 256>, 4, 11008>;   //  8 rows / thread, 32 warps / SM
using CfgC = TileCfg<Shape<32, 16, 8, 256>, 3, 14592>;  // 16 rows / thread, 24 warps / SM
using CfgD = TileCfg<Shape<32, 8, 16, 512>, 2, 16384>;  //  8 rows / thread, 32 warps / SM
using CfgE = TileCfg<Shape<32, 16, 8, 512>, 2, 16384>;  //  8 rows / thread, 32 warps / SM
using PersShape = Shape<32, 8, 8, 256>;              // persistent, double-buffered, 2 CTAs/SM

// 64-bit address base + 32-bit element offset in one IMAD.WIDE.U32
__device__ __forceinline__ float* addr_f32(float* base, uint32_t off) {
  float* p;
  asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(p) : "r"(off), "l"(base));
  return p;
}
__device__ __forceinline__ uint8_t* addr_u8(uint8_t* base, uint32_t off) {
  uint8_t* p;
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(p) : "r"(off), "l"(base));
  return p;
}
__device__ __forceinline__ void st_f32(float* p, float v) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Rows ybeg .. of one output column, as y-pairs (NR / 2 of them).  kFull: every
// pair has both rows (no per-pair bounds).
template <int NR, bool kStagedPath, bool kLabels, bool kNearest, bool kClamp, bool kSepLbl,
          bool kFull>
__device__ __forceinline__ void column_pairs(const WarpArgs& a, const Params& P,
                                             const float* __restrict__ vin,
                                             const uint8_t* __restrict__ lin,
                                             float* __restrict__ vout,
                                             uint8_t* __restrict__ lout, const Stage& sv,
                                             int X, int Z, int ybeg, int yend, const float* n) {
  const int mx = a.mx;
  const float fX = static_cast<float>(X), fZ = static_cast<float>(Z);
  const float2 cz0 = f2(__fmaf_rn(P.A[2], fZ, P.A[3]));
  const float2 cz1 = f2(__fmaf_rn(P.A[6], fZ, P.A[7]));
  const float2 cz2 = f2(__fmaf_rn(P.A[10], fZ, P.A[11]));
  // output offsets are 32-bit within a volume (< 2^31 voxels)
  const uint32_t o0 = static_cast<uint32_t>((Z * a.my + ybeg) * mx + X);
#pragma unroll
  for (int j = 0; j < NR / 2; ++j) {
    const int Ya = ybeg + 2 * j;
    bool second = true;
    if (!kFull) {
      if (Ya >= yend) break;
      second = Ya + 1 < yend;
    }
    const float2 fY = make_float2(static_cast<float>(Ya), static_cast<float>(second ? Ya + 1 : Ya));
    const float2 px = __ffma2_rn(f2(P.A[0]), f2(fX), __ffma2_rn(f2(P.A[1]), fY, cz0));
    const float2 py = __ffma2_rn(f2(P.A[4]), f2(fX), __ffma2_rn(f2(P.A[5]), fY, cz1));
    const float2 pz = __ffma2_rn(f2(P.A[8]), f2(fX), __ffma2_rn(f2(P.A[9]), fY, cz2));
    float2 img = make_float2(0.0f, 0.0f);
    uint32_t l0 = 0, l1 = 0;
    if (kStagedPath) {
      sample_staged2<kLabels, kNearest, kClamp, kSepLbl>(sv, px, py, pz, true, img, l0, l1);
    } else {
      const Sample s0 = sample_gather(a, vin, lin, px.x, py.x, pz.x, true);
      const Sample s1 = sample_gather(a, vin, lin, px.y, py.y, pz.y, true);
      img = make_float2(s0.img, s1.img);
      l0 = s0.lbl;
      l1 = s1.lbl;
    }
    const float2 out = photometric2(img, make_float2(n[2 * j], n[2 * j + 1]), P);
    const uint32_t o = o0 + static_cast<uint32_t>(2 * j * mx);
    st_f32(addr_f32(vout, o), out.x);
    if (kLabels) st_u8(addr_u8(lout, o), l0);
    if (second) {
      st_f32(addr_f32(vout, o + mx), out.y);
      if (kLabels) st_u8(addr_u8(lout, o + mx), l1);
    }
  }
}

// Occluded output z (R15): image 0, every later step skipped;
// labels are still warped.  Rare: kept out of line (instruction-cache
// footprint of the hot loop); P and the stage view are passed by value.
template <bool kStagedPath, bool kLabels, bool kClamp, bool kSepLbl>
__device__ __noinline__ void column_occluded(const WarpArgs& a, const Params P,
                                             const uint8_t* __restrict__ lin, float* vout,
                                             uint8_t* lout, const Stage sv, int X, int Z,
                                             int ybeg, int yend) {
  const float fX = static_cast<float>(X), fZ = static_cast<float>(Z);
  const float cz0 = __fmaf_rn(P.A[2], fZ, P.A[3]), cz1 = __fmaf_rn(P.A[6], fZ, P.A[7]);
  const float cz2 = __fmaf_rn(P.A[10], fZ, P.A[11]);
  for (int Y = ybeg; Y < yend; ++Y) {
    const float fY = static_cast<float>(Y);
    const float px = __fmaf_rn(P.A[0], fX, __fmaf_rn(P.A[1], fY, cz0));
    const float py = __fmaf_rn(P.A[4], fX, __fmaf_rn(P.A[5], fY, cz1));
    const float pz = __fmaf_rn(P.A[8], fX, __fmaf_rn(P.A[9], fY, cz2));
    uint32_t l = 0;
    if (kLabels) {
      if (kStagedPath) {
        float2 img;
        uint32_t l1;
        sample_staged2<true, false, kClamp, kSepLbl>(sv, make_float2(px, px), make_float2(py, py),
                                                    make_float2(pz, pz), false, img, l, l1);
      } else {
        l = sample_gather(a, nullptr, lin, px, py, pz, false).lbl;
      }
    }
    const uint32_t o = static_cast<uint32_t>((Z * a.my + Y) * a.mx + X);
    st_f32(addr_f32(vout, o), 0.0f);
    if (kLabels) st_u8(addr_u8(lout, o), l);
  }
}

// ----------------------------------------------------------------------------
// Output column work.  A thread owns output column x at one z and NR rows
// [ybeg, ybeg + NR), ybeg % 4 == 0, i.e. NR/4 Philox blocks (R10: block =
// (x, y/4, z), lane = y mod 4) computed first as independent chains, then
// y-pairs with FFMA2/FADD2.  The coordinate keeps the R4 nesting
// p = fma(A_k0, x, fma(A_k1, y, fma(A_k2, z, b))).
// ----------------------------------------------------------------------------
// Standard normals of NR rows (NR/4 Philox blocks, independent chains).
template <int NR>
__device__ __forceinline__ void column_noise(const WarpArgs& a, const Params& P, int X, int Z,
                                             int ybeg, float* n) {
#pragma unroll
  for (int i = 0; i < NR; ++i) n[i] = 0.0f;
  if (!(P.flags & kNoise)) return;
  const int Gy = (a.my + 3) >> 2;
  const uint32_t q0 = static_cast<uint32_t>(X) +
                      static_cast<uint32_t>(a.mx) * static_cast<uint32_t>(Gy * Z + (ybeg >> 2));
  uint4 r[NR / 4];
#pragma unroll
  for (int g = 0; g < NR / 4; ++g)
    r[g] = philox4x32_10_rk(make_uint4(q0 + static_cast<uint32_t>(g * a.mx), 0u, P.vid0, P.vid1),
                            P.rk0, P.rk1);
#pragma unroll
  for (int g = 0; g < NR / 4; ++g) {
    const float2 u = box_muller(r[g].x, r[g].y), v = box_muller(r[g].z, r[g].w);
    n[4 * g] = u.x; n[4 * g + 1] = u.y; n[4 * g + 2] = v.x; n[4 * g + 3] = v.y;
  }
}

__device__ __forceinline__ bool column_occluded_z(const Params& P, int Z) {
  return (P.flags & kOcclude) && Z >= P.occ_lo && Z <= P.occ_hi;  // warp-uniform
}

// NR rows of one column whose noise n[] is already computed.
template <int NR, bool kStagedPath, bool kLabels, bool kNearest, bool kClamp, bool kSepLbl>
__device__ __forceinline__ void column_rows_n(const WarpArgs& a, const Params& P,
                                              const float* __restrict__ vin,
                                              const uint8_t* __restrict__ lin,
                                              float* __restrict__ vout,
                                              uint8_t* __restrict__ lout, const Stage& sv, int X,
                                              int Z, int ybeg, const float* n) {
  const int my = a.my;
  if (X >= a.mx || Z >= a.mz || ybeg >= my) return;
  const int yend = min(ybeg + NR, my);
  if (column_occluded_z(P, Z)) {
    column_occluded<kStagedPath, kLabels, kClamp, kSepLbl>(a, P, lin, vout, lout, sv, X, Z, ybeg,
                                                           yend);
    return;
  }
  if (yend - ybeg == NR)
    column_pairs<NR, kStagedPath, kLabels, kNearest, kClamp, kSepLbl, true>(
        a, P, vin, lin, vout, lout, sv, X, Z, ybeg, yend, n);
  else
    column_pairs<NR, kStagedPath, kLabels, kNearest, kClamp, kSepLbl, false>(
        a, P, vin, lin, vout, lout, sv, X, Z, ybeg, yend, n);
}

// NR rows [ybeg, ybeg + NR) of one output column, in groups of 8 rows (two
// interleaved Philox chains per group; the group loop is not unrolled to keep
// the hot code inside the instruction cache).
template <int NR, bool kStagedPath, bool kLabels, bool kNearest, bool kClamp, bool kSepLbl>
__device__ __forceinline__ void column_rows(const WarpArgs& a, const Params& P,
                                            const float* __restrict__ vin,
                                            const uint8_t* __restrict__ lin,
                                            float* __restrict__ vout, uint8_t* __restrict__ lout,
                                            const Stage& sv, int X, int Z, int ybeg) {
  constexpr int G = NR < 8 ? NR : 8;
  const bool occl = column_occluded_z(P, Z);
#pragma unroll 1
  for (int y = ybeg; y < ybeg + NR; y += G) {
    float n[G];
    if (!occl && X < a.mx && Z < a.mz && y < a.my)
      column_noise<G>(a, P, X, Z, y, n);
    column_rows_n<G, kStagedPath, kLabels, kNearest, kClamp, kSepLbl>(a, P, vin, lin, vout, lout,
                                                                      sv, X, Z, y, n);
  }
}

template <class S, bool kStagedPath, bool kLabels, bool kNearest, bool kClamp>
__device__ __forceinline__ void tile_compute(const WarpArgs& a, const Params& P,
                                             const float* __restrict__ vin,
                                             const uint8_t* __restrict__ lin,
                                             float* __restrict__ vout,
                                             uint8_t* __restrict__ lout, const Stage& sv,
                                             int ox, int oy, int oz) {
  const int w = static_cast<int>(threadIdx.x >> 5);
  column_rows<S::RPT, kStagedPath, kLabels, kNearest, kClamp, false>(
      a, P, vin, lin, vout, lout, sv, ox + static_cast<int>(threadIdx.x & 31), oz + w % S::TZ,
      oy + (w / S::TZ) * S::RPT);
}

// Box of one tile (warp 0): the bounding box of the 8 transformed tile corners
// -- exact, because p is monotone in each output coordinate -- clamped to
// [-1, n+1], x origin rounded down to a multiple of 4 and width up.
// box = {x0, y0, z0, W, H, D, staged, clamp}.
template <class S>
__device__ __forceinline__ void tile_box(const WarpArgs& a, const Params& P, int ox, int oy,
                                         int oz, int cap_vox, int* box) {
  const int c = threadIdx.x & 7;
  const float X = static_cast<float>((c & 1) ? min(ox + S::TX, a.mx) - 1 : ox);
  const float Y = static_cast<float>((c & 2) ? min(oy + S::TY, a.my) - 1 : oy);
  const float Z = static_cast<float>((c & 4) ? min(oz + S::TZ, a.mz) - 1 : oz);
  float mn[3], mxv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float p = __fmaf_rn(P.A[4 * k], X, __fmaf_rn(P.A[4 * k + 1], Y,
                                                       __fmaf_rn(P.A[4 * k + 2], Z, P.A[4 * k + 3])));
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
  if ((threadIdx.x & 31) == 0) {
    const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                        static_cast<float>(a.nz)};
    int lo[3], hi[3];
    bool inside = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = static_cast<int>(floorf(fminf(fmaxf(mn[k], -1.0f), n[k])));
      hi[k] = static_cast<int>(floorf(fminf(fmaxf(mxv[k], -1.0f), n[k]))) + 1;
      inside &= (mn[k] >= -1.0f) & (mxv[k] <= n[k]);
    }
    const int x0 = lo[0] >= 0 ? (lo[0] & ~3) : -4;
    const int W = (hi[0] + 1 - x0 + 3) & ~3;
    const int H = hi[1] - lo[1] + 1, D = hi[2] - lo[2] + 1;
    box[0] = x0; box[1] = lo[1]; box[2] = lo[2];
    box[3] = W; box[4] = H; box[5] = D;
    box[6] = (static_cast<int64_t>(W) * H * D <= cap_vox && W <= 4 * S::THREADS) ? 1 : 0;
    box[7] = inside ? 0 : 1;  // clamp needed
  }
}

// Issue the staging of one box {x0, y0, z0, W, H, D} into the buffer at byte
// offsets (img_off, lbl_off) of g_smem: 16 B chunks (4 voxels); in-volume
// chunks by cp.async (image 16 B + label 4 B), out-of-volume chunks set to fill
// / label_fill.  nx % 4 == 0 and x0 % 4 == 0, so a chunk is entirely inside or
// outside in x.  Thread t owns chunk column c = t % CW of rows r = t / CW +
// k (THREADS / CW); rows advance in (y, z) without division; sources are one
// mad.wide off hoisted 64-bit column bases.  Completion: cp.async.wait_*.
// q = floor(i / d) for 0 <= i < 2^20, 1 <= d < 2^12: the rounded reciprocal
// quotient is within 2^-21 relative of (i + 0.5) / d, whose distance to an
// integer is >= 0.5 / d, so truncation is exact.
__device__ __forceinline__ int div_small(int i, float inv_d) {
  return __float2int_rz((static_cast<float>(i) + 0.5f) * inv_d);
}

template <class S, bool kLabels, bool kInside>
__device__ __forceinline__ void stage_box_impl(const WarpArgs& a, const float* __restrict__ vin,
                                               const uint8_t* __restrict__ lin, const int* box,
                                               uint32_t img_off, uint32_t lbl_off) {
  const int bx = box[0], by = box[1], bz = box[2], W = box[3], H = box[4], D = box[5];
  const int CW = W >> 2;
  const int rows_per_pass = S::THREADS / CW;
  const int tid = static_cast<int>(threadIdx.x);
  int r = div_small(tid, __frcp_rn(static_cast<float>(CW)));
  const int c = tid - r * CW;
  if (r >= rows_per_pass) return;
  const int rows = H * D;
  const int nx = a.nx, ny = a.ny, nz = a.nz, plane = nx * ny;
  const float inv_h = __frcp_rn(static_cast<float>(H));
  int rz = div_small(r, inv_h), ry = r - rz * H;
  int gy = by + ry, gz = bz + rz;
  const int gx = bx + 4 * c;
  const bool x_in = static_cast<unsigned>(gx) < static_cast<unsigned>(nx);
  float* gcol = const_cast<float*>(vin) + gx;
  uint8_t* lcol = kLabels ? const_cast<uint8_t*>(lin) + gx : nullptr;
  uint32_t goff = static_cast<uint32_t>(gz * plane + gy * nx);
  const int step_z = div_small(rows_per_pass, inv_h), step_y = rows_per_pass - step_z * H;
  const uint32_t goff_step = static_cast<uint32_t>(step_z * plane + step_y * nx);
  const uint32_t goff_wrap = static_cast<uint32_t>(plane - H * nx);
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(g_smem));
  uint32_t si = sbase + img_off + 4u * static_cast<uint32_t>(r * W + 4 * c);
  uint32_t sl = sbase + lbl_off + static_cast<uint32_t>(r * W + 4 * c);
  const uint32_t sstep = static_cast<uint32_t>(rows_per_pass * W);
  const float f = a.fill;
  const uint32_t lf4 = a.label_fill * 0x01010101u;
#pragma unroll 2
  for (; r < rows; r += rows_per_pass) {
    if (kInside) {
      cp_async16(si, addr_f32(gcol, goff));
      if (kLabels) cp_async4(sl, addr_u8(lcol, goff));
    } else {
      const bool in = x_in & (static_cast<unsigned>(gy) < static_cast<unsigned>(ny)) &
                      (static_cast<unsigned>(gz) < static_cast<unsigned>(nz));
      if (in) {
        cp_async16(si, addr_f32(gcol, goff));
        if (kLabels) cp_async4(sl, addr_u8(lcol, goff));
      } else {
        asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};\n" ::"r"(si), "f"(f) : "memory");
        if (kLabels) asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(sl), "r"(lf4) : "memory");
      }
      gy += step_y;
      gz += step_z;
    }
    si += 4u * sstep;
    sl += sstep;
    ry += step_y;
    goff += goff_step;
    if (ry >= H) {
      ry -= H;
      goff += goff_wrap;
      if (!kInside) {
        gy -= H;
        ++gz;
      }
    }
  }
}

// Issue the staging of one box {x0, y0, z0, W, H, D} into the buffer at byte
// offsets (img_off, lbl_off) of g_smem: 16 B chunks (4 voxels); in-volume
// chunks by cp.async (image 16 B + label 4 B), out-of-volume chunks set to fill
// / label_fill.  nx % 4 == 0 and x0 % 4 == 0, so a chunk is entirely inside or
// outside in x.  Thread t owns chunk column c = t % CW of rows r = t / CW +
// k (THREADS / CW); rows advance in (y, z) without division; sources are one
// mad.wide off hoisted 64-bit column bases.  Boxes inside the volume skip the
// per-chunk bounds test.  Completion: cp.async.wait_*.
template <class S, bool kLabels>
__device__ __forceinline__ void stage_box(const WarpArgs& a, const float* __restrict__ vin,
                                          const uint8_t* __restrict__ lin, const int* box,
                                          uint32_t img_off, uint32_t lbl_off) {
  const bool inside = box[0] >= 0 && box[1] >= 0 && box[2] >= 0 && box[0] + box[3] <= a.nx &&
                      box[1] + box[4] <= a.ny && box[2] + box[5] <= a.nz;
  if (inside)
    stage_box_impl<S, kLabels, true>(a, vin, lin, box, img_off, lbl_off);
  else
    stage_box_impl<S, kLabels, false>(a, vin, lin, box, img_off, lbl_off);
}

__device__ __forceinline__ Stage make_stage(const WarpArgs& a, const int* box, int img_off,
                                            int lbl_off) {
  Stage sv;
  sv.W = box[3];
  sv.HW = box[3] * box[4];
  sv.img_off = img_off;
  sv.lbl_off = lbl_off;
  sv.bx = static_cast<float>(box[0]);
  sv.by = static_cast<float>(box[1]);
  sv.bz = static_cast<float>(box[2]);
  sv.Wf = static_cast<float>(sv.W);
  sv.HWf = static_cast<float>(sv.HW);
  sv.WL = sv.W;
  sv.HWL = sv.HW;
  sv.WLf = sv.Wf;
  sv.HWLf = sv.HWf;
  sv.nx = static_cast<float>(a.nx);
  sv.ny = static_cast<float>(a.ny);
  sv.nz = static_cast<float>(a.nz);
  return sv;
}

template <class S, bool kLabels, bool kNearest>
__device__ __forceinline__ void compute_staged(const WarpArgs& a, const Params& P,
                                               const float* vin, const uint8_t* lin, float* vout,
                                               uint8_t* lout, const int* box, int img_off,
                                               int lbl_off, int ox, int oy, int oz) {
  const Stage sv = make_stage(a, box, img_off, lbl_off);
  if (box[7])
    tile_compute<S, true, kLabels, kNearest, true>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
  else
    tile_compute<S, true, kLabels, kNearest, false>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
}

// ----------------------------------------------------------------------------
// Kernel A (one tile per CTA): grid = (tiles_x, tiles_y, tiles_z * volumes).
// kStage: stage the tile's footprint box; tiles whose box exceeds cap_vox (or
// kStage = false: the W3D_KERNEL_GATHER variant) gather through L1/L2.
// ----------------------------------------------------------------------------
// Box record: image origin x (multiple of 4: TMA needs 16 B aligned inner
// coordinates), label origin x (multiple of 16), y, z, image / label widths
// from those origins, H, D, classes, flags, byte sizes, first output row.
enum { kBx, kBxl, kBy, kBz, kBW, kBWl, kBH, kBD, kBCi, kBCl, kBClamp, kBFix, kBImgBytes,
       kBLblBytes, kBPart, kBPI, kBRI, kBPL, kBRL, kBNF };  // pitches / rows per plane

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes)
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
    if (tries > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            int z, int v, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(v), "r"(mbar)
      : "memory");
}

// Every warp computes the whole tile's cp.async box itself (identical in all
// lanes: lanes 8g..8g+7 evaluate the 8 corners, reduced within 8-lane groups),
// so the common case needs no barrier before staging.  Returns whether the box
// fits cap_vox; b receives the kPlanCp record for nsub = 1.
template <class S>
__device__ __forceinline__ bool warp_box_cp(const WarpArgs& a, const float* __restrict__ A, int ox,
                                            int oy, int oz, int cap_vox, int* b) {
  const int c = threadIdx.x & 7;
  const float X = static_cast<float>((c & 1) ? min(ox + S::TX, a.mx) - 1 : ox);
  const float Y = static_cast<float>((c & 2) ? min(oy + S::TY, a.my) - 1 : oy);
  const float Z = static_cast<float>((c & 4) ? min(oz + S::TZ, a.mz) - 1 : oz);
  float mn[3], mxv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float p = __fmaf_rn(A[4 * k], X, __fmaf_rn(A[4 * k + 1], Y,
                                                     __fmaf_rn(A[4 * k + 2], Z, A[4 * k + 3])));
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
  const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                      static_cast<float>(a.nz)};
  int lo[3], hi[3];
  bool inside = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = static_cast<int>(floorf(fminf(fmaxf(mn[k], -1.0f), n[k])));
    hi[k] = static_cast<int>(floorf(fminf(fmaxf(mxv[k], -1.0f), n[k]))) + 1;
    inside &= (mn[k] >= -1.0f) & (mxv[k] <= n[k]);
  }
  const int bx = lo[0] & ~3;
  const int W = (hi[0] - bx + 1 + 3) & ~3, H = hi[1] - lo[1] + 1, D = hi[2] - lo[2] + 1;
  b[kBx] = bx; b[kBy] = lo[1]; b[kBz] = lo[2];
  b[kBPI] = W; b[kBH] = H; b[kBD] = D;
  b[kBClamp] = inside ? 0 : 1;
  b[kBImgBytes] = D * H * W * 4;
  b[kBPart] = oy;
  return static_cast<int64_t>(W) * H * D <= cap_vox;
}

// Warp 0: boxes of the tile split into nsub y-parts (nsub = 1, 2, 4: the
// first that fits).  Lanes 8g .. 8g+7 evaluate part g's 8 corners.  Layout
// modes: kPlanCp (cp.async: image and labels share origin x0 % 4 and pitch),
// kPlanBulk (1D bulk rows: label origin x0 % 16, own pitch), kPlanTensor
// (tensor boxes: width classes, 4 / 8-row groups).  Labels follow the image.
enum { kPlanCp = 0, kPlanBulk = 1, kPlanTensor = 2 };
template <class S, int kMode>
__device__ __forceinline__ void tma_plan(const WarpArgs& a, const float* __restrict__ A, int ox,
                                         int oy, int oz, int capb, bool labels,
                                         int (*box)[kBNF], int* nsub_out) {
  const int lane = threadIdx.x & 31, g = lane >> 3, c = lane & 7;
  const float n[3] = {static_cast<float>(a.nx), static_cast<float>(a.ny),
                      static_cast<float>(a.nz)};
  const bool fill_nz = a.fill != 0.0f, lfill_nz = labels && a.label_fill != 0u;
  constexpr int kMaxSub = S::TY / 4 < 4 ? S::TY / 4 : 4;  // parts keep whole Philox blocks
  for (int nsub = 1; nsub <= kMaxSub; nsub <<= 1) {
    const int rows = S::TY / nsub;
    const int y0 = oy + min(g, nsub - 1) * rows;
    const bool empty = y0 >= a.my;
    const float X = static_cast<float>((c & 1) ? min(ox + S::TX, a.mx) - 1 : ox);
    const float Y = static_cast<float>((c & 2) ? min(y0 + rows, a.my) - 1 : min(y0, a.my - 1));
    const float Z = static_cast<float>((c & 4) ? min(oz + S::TZ, a.mz) - 1 : oz);
    float mn[3], mxv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float p = __fmaf_rn(A[4 * k], X, __fmaf_rn(A[4 * k + 1], Y,
                                                       __fmaf_rn(A[4 * k + 2], Z, A[4 * k + 3])));
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
    int lo[3], hi[3];
    bool inside = true, touches = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = static_cast<int>(floorf(fminf(fmaxf(mn[k], -1.0f), n[k])));
      hi[k] = static_cast<int>(floorf(fminf(fmaxf(mxv[k], -1.0f), n[k]))) + 1;
      inside &= (mn[k] >= -1.0f) & (mxv[k] <= n[k]);
      touches |= (lo[k] < 0) | (hi[k] >= static_cast<int>(n[k]));
    }
    const int bxi = lo[0] & ~3, bxl = lo[0] & ~15;  // floor to 4 / 16 (lo >= -1)
    const int W = hi[0] - bxi + 1, Wl = hi[0] - bxl + 1;
    const int H = hi[1] - lo[1] + 1, D = hi[2] - lo[2] + 1;
    int ci = -1, cl = -1, PI, RI, PL, RL;
    if (kMode == kPlanCp) {  // cp.async chunks: one index space for image and labels
      ci = cl = 0;
      PI = (W + 3) & ~3; RI = H;
      PL = PI; RL = H;
    } else if (kMode == kPlanBulk) {  // 1D bulk row copies: 16 B granularity only
      ci = cl = 0;
      PI = (W + 3) & ~3; RI = H;
      PL = (Wl + 15) & ~15; RL = H;
    } else {      // tensor boxes: width classes, 4 / 8-row groups
#pragma unroll
      for (int q = kNumImgCls - 1; q >= 0; --q)
        if (img_cls_width(q) >= W) ci = q;
#pragma unroll
      for (int q = kNumLblCls - 1; q >= 0; --q)
        if (lbl_cls_width(q) >= Wl) cl = q;
      PI = ci < 0 ? 0 : img_cls_width(ci); RI = (H + 3) & ~3;
      PL = cl < 0 ? 0 : lbl_cls_width(cl); RL = (H + 7) & ~7;
    }
    const int64_t bimg = static_cast<int64_t>(D) * RI * PI * 4;
    const int64_t blbl = labels ? static_cast<int64_t>(D) * RL * PL : 0;
    const bool fits = empty || (ci >= 0 && (!labels || cl >= 0) && bimg + blbl <= capb);
    const bool all_fit = __all_sync(0xffffffffu, (g >= nsub) || fits);
    if (all_fit) {
      if (c == 0 && g < nsub) {
        int* b = box[g];
        b[kBx] = bxi; b[kBxl] = kMode == kPlanCp ? bxi : bxl; b[kBy] = lo[1]; b[kBz] = lo[2];
        b[kBW] = W; b[kBWl] = Wl; b[kBH] = H; b[kBD] = empty ? 0 : D;
        b[kBCi] = ci; b[kBCl] = cl;
        b[kBClamp] = inside ? 0 : 1;
        b[kBFix] = touches ? ((fill_nz ? 1 : 0) | (lfill_nz ? 2 : 0)) : 0;
        b[kBImgBytes] = static_cast<int>(bimg);
        b[kBLblBytes] = static_cast<int>(blbl);
        b[kBPart] = y0;
        b[kBPI] = PI; b[kBRI] = RI; b[kBPL] = PL; b[kBRL] = RL;
      }
      if (lane == 0) *nsub_out = nsub;
      return;
    }
  }
  if (lane == 0) *nsub_out = 0;
}

template <class Cfg, bool kStage, bool kLabels, bool kNearest>
__global__ void __launch_bounds__(Cfg::S::THREADS, Cfg::MINB)
    warp3d_tile_kernel(const __grid_constant__ WarpArgs a, const int tiles_z, const int cap_vox);

// cp.async-staged part of a tile: stage the part's box, wait, compute its rows.
template <int NR, bool kLabels, bool kNearest>
__device__ __forceinline__ void cp_part_compute(const WarpArgs& a, const Params& P, float* vout,
                                                uint8_t* lout, const int* box6, int lbl_off,
                                                bool clamp, int X, int Z, int ybeg) {
  const Stage sv = make_stage(a, box6, 0, lbl_off);
  if (clamp)
    column_rows<NR, true, kLabels, kNearest, true, false>(a, P, nullptr, nullptr, vout, lout, sv,
                                                          X, Z, ybeg);
  else
    column_rows<NR, true, kLabels, kNearest, false, false>(a, P, nullptr, nullptr, vout, lout,
                                                           sv, X, Z, ybeg);
}

// Out-of-line rare paths of the tile kernel (keep the hot loop's code small).
template <class S, bool kLabels, bool kNearest>
__device__ __noinline__ void gather_tile(const WarpArgs& a, int vi, int ox, int oy, int oz) {
  const Params P = load_params(a.vol[vi]);
  Stage sv;
  tile_compute<S, false, kLabels, kNearest, false>(
      a, P, a.in + vi * a.in_stride, kLabels ? a.in_lbl + vi * a.in_stride : nullptr,
      a.out + vi * a.out_stride, kLabels ? a.out_lbl + vi * a.out_stride : nullptr, sv, ox, oy,
      oz);
}

template <class S, bool kLabels, bool kNearest>
__device__ __noinline__ void subtile_path(const WarpArgs& a, const int* boxes, int vi, int ox,
                                          int oy, int oz, int nsub) {
  const float* vin = a.in + vi * a.in_stride;
  const uint8_t* lin = kLabels ? a.in_lbl + vi * a.in_stride : nullptr;
  float* vout = a.out + vi * a.out_stride;
  uint8_t* lout = kLabels ? a.out_lbl + vi * a.out_stride : nullptr;
  const int X = ox + static_cast<int>(threadIdx.x & 31);
  const int Z = oz + static_cast<int>(threadIdx.x >> 5);
  for (int k = 0; k < nsub; ++k) {
    int b[kBNF];
#pragma unroll
    for (int i = 0; i < kBNF; ++i) b[i] = boxes[k * kBNF + i];
    if (b[kBD] == 0) continue;  // part entirely beyond the volume's last row
    const int box6[6] = {b[kBx], b[kBy], b[kBz], b[kBPI], b[kBH], b[kBD]};
    stage_box<S, kLabels>(a, vin, lin, box6, 0u, static_cast<uint32_t>(b[kBImgBytes]));
    cp_async_wait_all();
    __syncthreads();
    const Params P = load_params(a.vol[vi]);
    if (nsub == 2) {
      if constexpr (S::TY / 2 >= 4)
        cp_part_compute<S::TY / 2, kLabels, kNearest>(a, P, vout, lout, box6, b[kBImgBytes],
                                                      b[kBClamp] != 0, X, Z, b[kBPart]);
    } else {
      if constexpr (S::TY / 4 >= 4)
        cp_part_compute<S::TY / 4, kLabels, kNearest>(a, P, vout, lout, box6, b[kBImgBytes],
                                                      b[kBClamp] != 0, X, Z, b[kBPart]);
    }
    __syncthreads();  // buffer reuse by the next part
  }
}

template <class Cfg, bool kStage, bool kLabels, bool kNearest>
__global__ void __launch_bounds__(Cfg::S::THREADS, Cfg::MINB)
    warp3d_tile_kernel(const __grid_constant__ WarpArgs a, const int tiles_z, const int cap_vox) {
  using S = typename Cfg::S;
  __shared__ int s_box[4][kBNF];
  __shared__ int s_nsub;
  const int vi = static_cast<int>(blockIdx.z) / tiles_z;
  const int ox = static_cast<int>(blockIdx.x) * S::TX;
  const int oy = static_cast<int>(blockIdx.y) * S::TY;
  const int oz = (static_cast<int>(blockIdx.z) - vi * tiles_z) * S::TZ;
  const float* __restrict__ vin = a.in + vi * a.in_stride;
  const uint8_t* __restrict__ lin = kLabels ? a.in_lbl + vi * a.in_stride : nullptr;
  float* __restrict__ vout = a.out + vi * a.out_stride;
  uint8_t* __restrict__ lout = kLabels ? a.out_lbl + vi * a.out_stride : nullptr;
  if (!kStage || S::WARPS != S::TZ) {  // gather variant
    count_tile(false);
    gather_tile<S, kLabels, kNearest>(a, vi, ox, oy, oz);
    return;
  }
  int b[kBNF];
  if (!warp_box_cp<S>(a, a.vol[vi].A, ox, oy, oz, cap_vox, b)) {
    // rare: the footprint exceeds the buffer -> y-parts (or gathers)
    if (threadIdx.x < 32)
      tma_plan<S, kPlanCp>(a, a.vol[vi].A, ox, oy, oz, cap_vox * 5, kLabels, s_box, &s_nsub);
    __syncthreads();
    const int nsub = s_nsub;
    count_tile(nsub != 0);
    if (nsub == 0)
      gather_tile<S, kLabels, kNearest>(a, vi, ox, oy, oz);
    else
      subtile_path<S, kLabels, kNearest>(a, &s_box[0][0], vi, ox, oy, oz, nsub);
    return;
  }
  count_tile(true);
  const int X = ox + static_cast<int>(threadIdx.x & 31);
  const int Z = oz + static_cast<int>(threadIdx.x >> 5);
  // whole tile: issue the staging, compute the column's noise (independent of
  // the box) while the copies are in flight, then wait and sample
  const int box6[6] = {b[kBx], b[kBy], b[kBz], b[kBPI], b[kBH], b[kBD]};
  stage_box<S, kLabels>(a, vin, lin, box6, 0u, static_cast<uint32_t>(b[kBImgBytes]));
  const Params P = load_params(a.vol[vi]);
  const bool live = X < a.mx && Z < a.mz && oy < a.my && !column_occluded_z(P, Z);
  float n[S::TY];
  if (live) column_noise<S::TY>(a, P, X, Z, oy, n);
  cp_async_wait_all();
  __syncthreads();
  const Stage sv = make_stage(a, box6, 0, b[kBImgBytes]);
  if (b[kBClamp])
    column_rows_n<S::TY, true, kLabels, kNearest, true, false>(a, P, nullptr, nullptr, vout, lout,
                                                               sv, X, Z, oy, n);
  else
    column_rows_n<S::TY, true, kLabels, kNearest, false, false>(a, P, nullptr, nullptr, vout,
                                                                lout, sv, X, Z, oy, n);
}

// ----------------------------------------------------------------------------
// Kernel B (persistent, cp.async pipeline): each CTA walks the tiles t =
// blockIdx.x + k * gridDim.x (volume-major order, so concurrently processed
// tiles share the L2-resident slab of one volume).  Two staging buffers: the
// cp.async copies of tile k+1 are issued before tile k is computed, and each
// thread computes tile k's noise while its copies are in flight.  Plans use 3
// metadata slots (k % 3) so warp 0 can publish tile k+1's plan while slower
// warps still read tile k-1's.  Tiles whose footprint exceeds a buffer are
// split into y-parts and staged serially (no prefetch); if even those do not
// fit, gathered.
// ----------------------------------------------------------------------------
template <class S>
__device__ __forceinline__ void tile_coords(int t, int tiles_x, int tiles_y, int per_vol,
                                            int& vi, int& ox, int& oy, int& oz) {
  vi = t / per_vol;
  int r = t - vi * per_vol;
  const int txy = tiles_x * tiles_y;
  const int tzi = r / txy;
  r -= tzi * txy;
  const int tyi = r / tiles_x;
  ox = (r - tyi * tiles_x) * S::TX;
  oy = tyi * S::TY;
  oz = tzi * S::TZ;
}

template <class S, bool kLabels, bool kNearest>
__global__ void __launch_bounds__(S::THREADS, 2)
    warp3d_persistent_kernel(const __grid_constant__ WarpArgs a, const int tiles_x,
                             const int tiles_y, const int tiles_z, const int total,
                             const int cap_vox) {
  static_assert(S::WARPS == S::TZ && S::RPT == S::TY && S::TY == 8, "persistent shape");
  __shared__ int s_box[3][2][kBNF];
  __shared__ int s_nsub[3];
  const int per_vol = tiles_x * tiles_y * tiles_z;
  const uint32_t buf_bytes = static_cast<uint32_t>(cap_vox) * 5u;
  int t = static_cast<int>(blockIdx.x);
  if (t >= total) return;
  const int lane_x = static_cast<int>(threadIdx.x & 31), wz = static_cast<int>(threadIdx.x >> 5);
  auto plan = [&](int tt, int slot) {
    int vi, ox, oy, oz;
    tile_coords<S>(tt, tiles_x, tiles_y, per_vol, vi, ox, oy, oz);
    tma_plan<S, kPlanCp>(a, a.vol[vi].A, ox, oy, oz, cap_vox * 5, kLabels, s_box[slot],
                         &s_nsub[slot]);
  };
  auto stage_tile = [&](int tt, int slot, uint32_t buf) {
    int vi, ox, oy, oz;
    tile_coords<S>(tt, tiles_x, tiles_y, per_vol, vi, ox, oy, oz);
    const int* b = s_box[slot][0];
    const int box6[6] = {b[kBx], b[kBy], b[kBz], b[kBPI], b[kBH], b[kBD]};
    if (box6[5] > 0)
      stage_box<S, kLabels>(a, a.in + vi * a.in_stride,
                            kLabels ? a.in_lbl + vi * a.in_stride : nullptr, box6, buf,
                            buf + static_cast<uint32_t>(b[kBImgBytes]));
  };
  if (threadIdx.x < 32) plan(t, 0);
  __syncthreads();
  if (s_nsub[0] == 1) stage_tile(t, 0, 0u);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int k = 0;; ++k) {
    const int tn = t + static_cast<int>(gridDim.x);
    const int slot = k % 3, nslot = (k + 1) % 3;
    const uint32_t buf = (k & 1) ? buf_bytes : 0u, nbuf = (k & 1) ? 0u : buf_bytes;
    if (tn < total && threadIdx.x < 32) plan(tn, nslot);
    __syncthreads();  // (1) next plan visible; every warp is done with tile k-1's buffer
    if (tn < total && s_nsub[nslot] == 1) stage_tile(tn, nslot, nbuf);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int vi, ox, oy, oz;
    tile_coords<S>(t, tiles_x, tiles_y, per_vol, vi, ox, oy, oz);
    const Params P = load_params(a.vol[vi]);
    float* vout = a.out + vi * a.out_stride;
    uint8_t* lout = kLabels ? a.out_lbl + vi * a.out_stride : nullptr;
    const int X = ox + lane_x, Z = oz + wz;
    const int nsub = s_nsub[slot];
    const bool live = X < a.mx && Z < a.mz && oy < a.my && !column_occluded_z(P, Z);
    float n[S::TY];
    if (live) column_noise<S::TY>(a, P, X, Z, oy, n);  // overlaps the copies in flight
    if (nsub == 1) {
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // tile k's group is complete
      __syncthreads();  // (2) tile k's staged box visible to all
      count_tile(true);
      const int* b = s_box[slot][0];
      const int box6[6] = {b[kBx], b[kBy], b[kBz], b[kBPI], b[kBH], b[kBD]};
      const Stage sv = make_stage(a, box6, static_cast<int>(buf),
                                  static_cast<int>(buf) + b[kBImgBytes]);
      if (b[kBClamp])
        column_rows_n<S::TY, true, kLabels, kNearest, true, false>(a, P, nullptr, nullptr, vout,
                                                                   lout, sv, X, Z, oy, n);
      else
        column_rows_n<S::TY, true, kLabels, kNearest, false, false>(a, P, nullptr, nullptr, vout,
                                                                    lout, sv, X, Z, oy, n);
    } else if (nsub == 2) {  // two y-parts staged serially into this tile's buffer
      count_tile(true);
      for (int part = 0; part < 2; ++part) {
        const int* b = s_box[slot][part];
        const int box6[6] = {b[kBx], b[kBy], b[kBz], b[kBPI], b[kBH], b[kBD]};
        if (box6[5] > 0)
          stage_box<S, kLabels>(a, a.in + vi * a.in_stride,
                                kLabels ? a.in_lbl + vi * a.in_stride : nullptr, box6, buf,
                                buf + static_cast<uint32_t>(b[kBImgBytes]));
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (box6[5] > 0) {
          const Stage sv = make_stage(a, box6, static_cast<int>(buf),
                                      static_cast<int>(buf) + b[kBImgBytes]);
          if (part == 0)
            column_rows_n<S::TY / 2, true, kLabels, kNearest, true, false>(
                a, P, nullptr, nullptr, vout, lout, sv, X, Z, b[kBPart], n);
          else
            column_rows_n<S::TY / 2, true, kLabels, kNearest, true, false>(
                a, P, nullptr, nullptr, vout, lout, sv, X, Z, b[kBPart], n + S::TY / 2);
        }
        __syncthreads();
      }
    } else {  // footprint too large even in parts: gathers
      count_tile(false);
      Stage sv;
      const float* vin = a.in + vi * a.in_stride;
      const uint8_t* lin = kLabels ? a.in_lbl + vi * a.in_stride : nullptr;
      column_rows_n<S::TY, false, kLabels, kNearest, false, false>(a, P, vin, lin, vout, lout,
                                                                    sv, X, Z, oy, n);
    }
    if (tn >= total) break;
    t = tn;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

static int g_pers_cap_vox = kPersCapVox;
static int g_num_sms = 0;

template <class Cfg, bool kStage, bool kLabels, bool kNearest>
static cudaError_t launch_variant(const WarpArgs& a, cudaStream_t s) {
  using S = typename Cfg::S;
  const int tiles_x = (a.mx + S::TX - 1) / S::TX, tiles_y = (a.my + S::TY - 1) / S::TY;
  const int tiles_z = (a.mz + S::TZ - 1) / S::TZ;
  const int64_t gz = static_cast<int64_t>(tiles_z) * a.nvol;
  if (tiles_y > 65535 || gz > 65535) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y),
                  static_cast<unsigned>(gz));
  if (kStage) {
    const int cap = Cfg::CAP;
    const size_t smem = static_cast<size_t>(cap) * 5;
    static bool configured = false;
    if (!configured) {
      const cudaError_t e = cudaFuncSetAttribute(warp3d_tile_kernel<Cfg, kStage, kLabels, kNearest>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      configured = true;
    }
    warp3d_tile_kernel<Cfg, kStage, kLabels, kNearest><<<grid, S::THREADS, smem, s>>>(a, tiles_z,
                                                                                    cap);
  } else {
    warp3d_tile_kernel<Cfg, kStage, kLabels, kNearest><<<grid, S::THREADS, 0, s>>>(a, tiles_z, 0);
  }
  return cudaGetLastError();
}

template <class Cfg>
static cudaError_t launch_cfg(const WarpArgs& a, bool staged, cudaStream_t s) {
  const bool labels = a.in_lbl != nullptr;
  const bool nearest = a.interp == W3D_INTERP_NEAREST;
  if (staged) {
    if (labels)
      return nearest ? launch_variant<Cfg, true, true, true>(a, s)
                     : launch_variant<Cfg, true, true, false>(a, s);
    return nearest ? launch_variant<Cfg, true, false, true>(a, s)
                   : launch_variant<Cfg, true, false, false>(a, s);
  }
  if (labels)
    return nearest ? launch_variant<Cfg, false, true, true>(a, s)
                   : launch_variant<Cfg, false, true, false>(a, s);
  return nearest ? launch_variant<Cfg, false, false, true>(a, s)
                 : launch_variant<Cfg, false, false, false>(a, s);
}

// Tuning knob for experiments (not part of the ABI): W3D_TILE_CFG = A..E.
static char tile_cfg() {
  static char v = 0;
  if (!v) {
    const char* e = getenv("W3D_TILE_CFG");
    v = (e && e[0] >= 'A' && e[0] <= 'E') ? e[0] : 'C';
  }
  return v;
}



template <class S, bool kLabels, bool kNearest>
static cudaError_t launch_persistent_variant(const WarpArgs& a, int cap, cudaStream_t s) {
  const int tiles_x = (a.mx + S::TX - 1) / S::TX, tiles_y = (a.my + S::TY - 1) / S::TY;
  const int tiles_z = (a.mz + S::TZ - 1) / S::TZ;
  const int64_t total = static_cast<int64_t>(tiles_x) * tiles_y * tiles_z * a.nvol;
  if (total >= (int64_t(1) << 31)) return cudaErrorInvalidConfiguration;
  const size_t smem = static_cast<size_t>(cap) * 10;  // two buffers of cap * (4 + 1) B
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(warp3d_persistent_kernel<S, kLabels, kNearest>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  const int64_t ctas = static_cast<int64_t>(g_num_sms) * 2;
  const int grid = static_cast<int>(total < ctas ? total : ctas);
  warp3d_persistent_kernel<S, kLabels, kNearest><<<grid, S::THREADS, smem, s>>>(
      a, tiles_x, tiles_y, tiles_z, static_cast<int>(total), cap);
  return cudaGetLastError();
}

template <bool kLabels, bool kNearest>
static cudaError_t launch_persistent_variant(const WarpArgs& a, cudaStream_t s) {
  return launch_persistent_variant<PersShape, kLabels, kNearest>(a, g_pers_cap_vox, s);
}

static cudaError_t launch_tiles(const WarpArgs& a, bool staged, cudaStream_t s) {
  cudaError_t e;
  switch (tile_cfg()) {
    case 'B': e = launch_cfg<CfgB>(a, staged, s); break;
    case 'C': e = launch_cfg<CfgC>(a, staged, s); break;
    case 'D': e = launch_cfg<CfgD>(a, staged, s); break;
    case 'E': e = launch_cfg<CfgE>(a, staged, s); break;
    case 'A': e = launch_cfg<CfgA>(a, staged, s); break;
    default: e = launch_cfg<CfgC>(a, staged, s); break;
  }
  note_launch();
  return e;
}

static cudaError_t launch_persistent(const WarpArgs& a, cudaStream_t s) {
  const bool labels = a.in_lbl != nullptr;
  const bool nearest = a.interp == W3D_INTERP_NEAREST;
  cudaError_t e;
  if (labels)
    e = nearest ? launch_persistent_variant<true, true>(a, s)
                : launch_persistent_variant<true, false>(a, s);
  else
    e = nearest ? launch_persistent_variant<false, true>(a, s)
                : launch_persistent_variant<false, false>(a, s);
  note_launch();
  return e;
}

// ----------------------------------------------------------------------------
// Kernel C (TMA staging, the default): one CTA per output tile (cfg C shape,
// WARPS == TZ so every thread owns all TY rows of its column).  Warp 0 plans
// the tile: the footprint box of the whole tile, or of 2 / 4 y-parts when the
// whole box exceeds the buffer (sub-tiling replaces the gather fallback).
// Each part's box is loaded by cp.async.bulk.tensor (4D tensor map per width
// class: image boxes of 4 rows, label boxes of 8 rows; out-of-tensor elements
// arrive as 0), completion tracked by one mbarrier (one phase per part).
// Boundary boxes with a nonzero fill / label_fill get their out-of-volume
// elements overwritten before compute (R6, R8).
// ----------------------------------------------------------------------------
template <bool kLabels>
__device__ __forceinline__ void tma_issue(const WarpArgs& a, const int* b, int vi, uint32_t sbase,
                                          uint32_t mbar) {
  const int lane = threadIdx.x & 31;
  const int H4 = b[kBRI], H8 = b[kBRL], D = b[kBD];
  const int WI = b[kBPI];
  const int nimg_r = H4 / kTmaRowsImg, nimg = D * nimg_r;
  const int nlbl_r = H8 / kTmaRowsLbl, nlbl = kLabels ? D * nlbl_r : 0;
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(mbar, static_cast<uint32_t>(b[kBImgBytes] + (kLabels ? b[kBLblBytes] : 0)));
  }
  __syncwarp();
  const uint32_t lbase = sbase + static_cast<uint32_t>(b[kBImgBytes]);
  const int WL = kLabels ? b[kBPL] : 0;
  for (int i = lane; i < nimg + nlbl; i += 32) {
    if (i < nimg) {
      const int d = i / nimg_r, r = i - d * nimg_r;
      const uint32_t dst = sbase + static_cast<uint32_t>(((d * H4) + kTmaRowsImg * r) * WI * 4);
      tma_load_4d(dst, &a.tm_img[b[kBCi]], b[kBx], b[kBy] + kTmaRowsImg * r, b[kBz] + d, vi, mbar);
    } else {
      const int j = i - nimg, d = j / nlbl_r, r = j - d * nlbl_r;
      const uint32_t dst = lbase + static_cast<uint32_t>(((d * H8) + kTmaRowsLbl * r) * WL);
      tma_load_4d(dst, &a.tm_lbl[b[kBCl]], b[kBxl], b[kBy] + kTmaRowsLbl * r, b[kBz] + d, vi,
                  mbar);
    }
  }
}

// Overwrite the out-of-volume elements of a boundary box (TMA wrote 0) with
// fill / label_fill.  The box is clamped to [-1, n+1]: per in-volume row only
// a few columns at either end are outside.
__device__ __forceinline__ bool col_out(int x, int nx) {
  return static_cast<unsigned>(x) >= static_cast<unsigned>(nx);
}
template <class S, bool kLabels>
__device__ __forceinline__ void tma_fixup(const WarpArgs& a, const int* b, int pad) {
  const int H = b[kBH], D = b[kBD];
  const int H4 = b[kBRI], H8 = b[kBRL];
  const int WI = b[kBPI];
  const int WL = kLabels ? b[kBPL] : 0;
  const uint32_t simg = static_cast<uint32_t>(__cvta_generic_to_shared(g_smem)) + pad;
  const uint32_t slbl = simg + static_cast<uint32_t>(b[kBImgBytes]);
  const bool fi = b[kBFix] & 1, fl = kLabels && (b[kBFix] & 2);
  const float f = a.fill;
  const uint32_t lf4 = a.label_fill * 0x01010101u;
  // columns [0, left) and [right, W) of an in-volume row are outside in x
  const int left_i = min(b[kBW], max(0, -b[kBx])), right_i = max(0, a.nx - b[kBx]);
  const int left_l = min(b[kBWl], max(0, -b[kBxl])), right_l = max(0, a.nx - b[kBxl]);
  for (int r = threadIdx.x; r < H * D; r += S::THREADS) {
    const int rz = r / H, ry = r - rz * H;
    const bool row_out = col_out(b[kBz] + rz, a.nz) || col_out(b[kBy] + ry, a.ny);
    if (fi) {
      const uint32_t row = simg + 4u * static_cast<uint32_t>((rz * H4 + ry) * WI);
      if (row_out) {
        for (int x = 0; x < WI; x += 4)
          asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(row + 4u * x), "f"(f)
                       : "memory");
      } else {
        for (int x = 0; x < left_i; ++x)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(row + 4u * x), "f"(f) : "memory");
        for (int x = right_i; x < b[kBW]; ++x)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(row + 4u * x), "f"(f) : "memory");
      }
    }
    if (fl) {
      const uint32_t row = slbl + static_cast<uint32_t>((rz * H8 + ry) * WL);
      if (row_out) {
        for (int x = 0; x < WL; x += 16)
          asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(row + x), "r"(lf4)
                       : "memory");
      } else {
        for (int x = 0; x < left_l; ++x)
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(row + x), "r"(lf4) : "memory");
        for (int x = right_l; x < b[kBWl]; ++x)
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(row + x), "r"(lf4) : "memory");
      }
    }
  }
}

// Bulk staging: every thread copies whole box rows with 1D cp.async.bulk
// (image row [max(x0,0), min(x0+PI, nx)) and label row likewise; 16 B aligned
// because x0 % 4 == 0 (labels x0 % 16 == 0) and nx % 4 (16) == 0) and writes
// fill / label_fill into the out-of-volume rest of its rows.  Each copy adds
// its bytes to the mbarrier's transaction count; every thread arrives once.
template <class S, bool kLabels>
__device__ __forceinline__ void bulk_issue(const WarpArgs& a, const int* b,
                                           const float* __restrict__ vin,
                                           const uint8_t* __restrict__ lin, uint32_t sbase,
                                           uint32_t mbar) {
  const int H = b[kBH], D = b[kBD], PI = b[kBPI], PL = b[kBPL];
  const int bx = b[kBx], bxl = b[kBxl];
  const int nx = a.nx, ny = a.ny, nz = a.nz;
  const int xs = max(bx, 0), xe = min(bx + PI, nx);
  const uint32_t bytes_i = xe > xs ? 4u * static_cast<uint32_t>(xe - xs) : 0u;
  const int xsl = max(bxl, 0), xel = min(bxl + PL, nx);
  const uint32_t bytes_l = xel > xsl ? static_cast<uint32_t>(xel - xsl) : 0u;
  const uint32_t lbase = sbase + static_cast<uint32_t>(b[kBImgBytes]);
  const float f = a.fill;
  const uint32_t lf4 = a.label_fill * 0x01010101u;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  const int rows = H * D;
  int r = threadIdx.x;
  int rz = r / H, ry = r - (r / H) * H;
  const int step_z = S::THREADS / H, step_y = S::THREADS - step_z * H;
  for (; r < rows; r += S::THREADS) {
    const int z = b[kBz] + rz, y = b[kBy] + ry;
    const bool in_row = static_cast<unsigned>(z) < static_cast<unsigned>(nz) &&
                        static_cast<unsigned>(y) < static_cast<unsigned>(ny);
    const uint32_t irow = sbase + 4u * static_cast<uint32_t>(r * PI);
    const int64_t g = (static_cast<int64_t>(z) * ny + y) * nx;
    if (in_row && bytes_i) {
      mbar_expect(mbar, bytes_i);
      bulk_g2s(irow + 4u * static_cast<uint32_t>(xs - bx), vin + g + xs, bytes_i, mbar);
      for (int x = 0; x < xs - bx; ++x)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(irow + 4u * x), "f"(f) : "memory");
      for (int x = xe - bx; x < PI; ++x)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(irow + 4u * x), "f"(f) : "memory");
    } else {
      for (int x = 0; x < PI; x += 4)
        asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(irow + 4u * x), "f"(f)
                     : "memory");
    }
    if (kLabels) {
      const uint32_t lrow = lbase + static_cast<uint32_t>(r * PL);
      if (in_row && bytes_l) {
        mbar_expect(mbar, bytes_l);
        bulk_g2s(lrow + static_cast<uint32_t>(xsl - bxl), lin + g + xsl, bytes_l, mbar);
        for (int x = 0; x < xsl - bxl; ++x)
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(lrow + x), "r"(lf4) : "memory");
        for (int x = xel - bxl; x < PL; ++x)
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(lrow + x), "r"(lf4) : "memory");
      } else {
        for (int x = 0; x < PL; x += 16)
          asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(lrow + x), "r"(lf4)
                       : "memory");
      }
    }
    rz += step_z;
    ry += step_y;
    if (ry >= H) {
      ry -= H;
      ++rz;
    }
  }
  mbar_arrive(mbar);
}

__device__ __forceinline__ Stage make_stage_tma(const WarpArgs& a, const int* b, int pad) {
  Stage sv;
  sv.W = b[kBPI];
  sv.HW = sv.W * b[kBRI];
  sv.WL = b[kBPL];
  sv.HWL = sv.WL * b[kBRL];
  sv.img_off = pad;
  // label row origin is b[kBxl] <= b[kBx]: shift the label base so that the
  // image-relative column index addresses the label buffer
  sv.lbl_off = pad + b[kBImgBytes] + (b[kBx] - b[kBxl]);
  sv.bx = static_cast<float>(b[kBx]);
  sv.by = static_cast<float>(b[kBy]);
  sv.bz = static_cast<float>(b[kBz]);
  sv.Wf = static_cast<float>(sv.W);
  sv.HWf = static_cast<float>(sv.HW);
  sv.WLf = static_cast<float>(sv.WL);
  sv.HWLf = static_cast<float>(sv.HWL);
  sv.nx = static_cast<float>(a.nx);
  sv.ny = static_cast<float>(a.ny);
  sv.nz = static_cast<float>(a.nz);
  return sv;
}

template <int NR, bool kLabels, bool kNearest>
__device__ __forceinline__ void tma_part_compute(const WarpArgs& a, const Params& P,
                                                 float* vout, uint8_t* lout, const int* b,
                                                 int X, int Z, int pad) {
  const Stage sv = make_stage_tma(a, b, pad);
  if (b[kBClamp])
    column_rows<NR, true, kLabels, kNearest, true, true>(a, P, nullptr, nullptr, vout, lout, sv,
                                                         X, Z, b[kBPart]);
  else
    column_rows<NR, true, kLabels, kNearest, false, true>(a, P, nullptr, nullptr, vout, lout, sv,
                                                          X, Z, b[kBPart]);
}

template <class Cfg, bool kBulk, bool kLabels, bool kNearest>
__global__ void __launch_bounds__(Cfg::S::THREADS, Cfg::MINB)
    warp3d_tma_kernel(const __grid_constant__ WarpArgs a, const int tiles_z) {
  using S = typename Cfg::S;
  static_assert(S::WARPS == S::TZ && S::RPT == S::TY && S::TY % 16 == 0, "TMA kernel shape");
  __shared__ int s_box[4][kBNF];
  __shared__ int s_nsub;
  __shared__ __align__(8) unsigned long long s_mbar;
  const int vi = static_cast<int>(blockIdx.z) / tiles_z;
  const Params P = load_params(a.vol[vi]);
  const int ox = static_cast<int>(blockIdx.x) * S::TX;
  const int oy = static_cast<int>(blockIdx.y) * S::TY;
  const int oz = (static_cast<int>(blockIdx.z) - vi * tiles_z) * S::TZ;
  float* __restrict__ vout = a.out + vi * a.out_stride;
  uint8_t* __restrict__ lout = kLabels ? a.out_lbl + vi * a.out_stride : nullptr;
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
  // TMA destinations must be 128 B aligned: align the dynamic region at run time
  // (the launch reserves 128 extra bytes)
  const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(g_smem));
  const int pad = static_cast<int>((128u - (sraw & 127u)) & 127u);
  const uint32_t sbase = sraw + static_cast<uint32_t>(pad);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      mbar_init(mbar, kBulk ? S::THREADS : 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tma_plan<S, kBulk ? kPlanBulk : kPlanTensor>(a, a.vol[vi].A, ox, oy, oz, Cfg::CAP * 5,
                                                 kLabels, s_box, &s_nsub);
  }
  __syncthreads();
  const int nsub = s_nsub;
  const int X = ox + static_cast<int>(threadIdx.x & 31);
  const int Z = oz + static_cast<int>(threadIdx.x >> 5);
  if (nsub == 0) {  // even a quarter of the tile does not fit: gathers
    count_tile(false);
    Stage sv;
    const float* vin = a.in + vi * a.in_stride;
    const uint8_t* lin = kLabels ? a.in_lbl + vi * a.in_stride : nullptr;
    tile_compute<S, false, kLabels, kNearest, false>(a, P, vin, lin, vout, lout, sv, ox, oy, oz);
    return;
  }
  count_tile(true);
  uint32_t phase = 0;
  for (int k = 0; k < nsub; ++k) {
    int b[kBNF];
#pragma unroll
    for (int i = 0; i < kBNF; ++i) b[i] = s_box[k][i];
    if (b[kBD] == 0) continue;  // part entirely beyond the volume's last row
    // bulk: every thread issues its rows; tensor: warp 0 issues.  Warp 0 waits
    // on the mbarrier, the other warps block on bar.sync (no issue slots).
    if (kBulk)
      bulk_issue<S, kLabels>(a, b, a.in + vi * a.in_stride,
                             kLabels ? a.in_lbl + vi * a.in_stride : nullptr, sbase, mbar);
    if (threadIdx.x < 32) {
      if (!kBulk) tma_issue<kLabels>(a, b, vi, sbase, mbar);
      mbar_wait(mbar, phase);
    }
    phase ^= 1u;
    __syncthreads();
    if (!kBulk && b[kBFix]) {
      tma_fixup<S, kLabels>(a, b, pad);
      __syncthreads();
    }
    if (nsub == 1)
      tma_part_compute<S::TY, kLabels, kNearest>(a, P, vout, lout, b, X, Z, pad);
    else if (nsub == 2)
      tma_part_compute<S::TY / 2, kLabels, kNearest>(a, P, vout, lout, b, X, Z, pad);
    else
      tma_part_compute<S::TY / 4, kLabels, kNearest>(a, P, vout, lout, b, X, Z, pad);
    if (k + 1 < nsub) __syncthreads();  // buffer reuse by the next part
  }
}

template <class Cfg, bool kBulk, bool kLabels, bool kNearest>
static cudaError_t launch_tma_variant(const WarpArgs& a, cudaStream_t s) {
  using S = typename Cfg::S;
  const int tiles_x = (a.mx + S::TX - 1) / S::TX, tiles_y = (a.my + S::TY - 1) / S::TY;
  const int tiles_z = (a.mz + S::TZ - 1) / S::TZ;
  const int64_t gz = static_cast<int64_t>(tiles_z) * a.nvol;
  if (tiles_y > 65535 || gz > 65535) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y),
                  static_cast<unsigned>(gz));
  const size_t smem = static_cast<size_t>(Cfg::CAP) * 5 + 128;  // + alignment slack
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(warp3d_tma_kernel<Cfg, kBulk, kLabels, kNearest>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  warp3d_tma_kernel<Cfg, kBulk, kLabels, kNearest><<<grid, S::THREADS, smem, s>>>(a, tiles_z);
  return cudaGetLastError();
}

template <bool kBulk>
static cudaError_t launch_tma_kind(const WarpArgs& a, cudaStream_t s) {
  const bool labels = a.in_lbl != nullptr;
  const bool nearest = a.interp == W3D_INTERP_NEAREST;
  cudaError_t e;
  if (labels)
    e = nearest ? launch_tma_variant<CfgC, kBulk, true, true>(a, s)
                : launch_tma_variant<CfgC, kBulk, true, false>(a, s);
  else
    e = nearest ? launch_tma_variant<CfgC, kBulk, false, true>(a, s)
                : launch_tma_variant<CfgC, kBulk, false, false>(a, s);
  note_launch();
  return e;
}

cudaError_t launch_tma(const WarpArgs& a, cudaStream_t s) { return launch_tma_kind<false>(a, s); }
cudaError_t launch_bulk(const WarpArgs& a, cudaStream_t s) { return launch_tma_kind<true>(a, s); }

bool tma_supported(const WarpArgs& a) {
  const bool img_ok = (a.nx % 4 == 0) && (reinterpret_cast<uintptr_t>(a.in) % 16 == 0);
  const bool lbl_ok = a.in_lbl == nullptr ||
                      ((a.nx % 16 == 0) && (reinterpret_cast<uintptr_t>(a.in_lbl) % 16 == 0));
  return img_ok && lbl_ok;
}

cudaError_t read_tile_stats(unsigned long long out[2]) {
  cudaError_t e = cudaMemcpyFromSymbol(&out[0], g_tiles_staged, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(&out[1], g_tiles_gather, sizeof(unsigned long long));
  return e;
}

bool staged_supported(const WarpArgs& a) {
  return (a.nx % 4 == 0) && (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) &&
         (a.in_stride % 4 == 0) &&
         (a.in_lbl == nullptr || reinterpret_cast<uintptr_t>(a.in_lbl) % 4 == 0);
}

cudaError_t launch_gather(const WarpArgs& a, cudaStream_t s) { return launch_tiles(a, false, s); }

cudaError_t launch_persistent_api(const WarpArgs& a, cudaStream_t s) {
  return staged_supported(a) ? launch_persistent(a, s) : launch_tiles(a, false, s);
}

cudaError_t launch_staged(const WarpArgs& a, cudaStream_t s) {
  return launch_tiles(a, staged_supported(a), s);
}

// AUTO: the cp.async-staged tile kernel (measured faster than the bulk / tensor
// TMA variants on ~200 B footprint rows), else gathers when the
// layout does not allow 16 B chunks.  W3D_PERSISTENT=1 selects the persistent
// double-buffered kernel (experiment knob).
cudaError_t launch_auto(const WarpArgs& a, cudaStream_t s) {
  const char* e = getenv("W3D_PERSISTENT");
  if (e && e[0] == '1' && staged_supported(a)) return launch_persistent(a, s);
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
