// philox.cuh -- Philox4x32-10 and the Box-Muller normal pair for sm_100a.
//
// Counter-based replacement for the paper's per-thread cuRAND generators
// ("a copy of the same RNG, starting at a different seed";
// DESIGN.md reading R10).  Stateless: a thread derives its words from
// (seed, volume_id, voxel block) alone, so the stream is independent of launch
// shape, batch split and GPU count.  Round function: Salmon et al., SC'11.
#pragma once
#include <cstdint>

namespace w3d {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

__host__ __device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                                      uint32_t& c3, uint32_t k0, uint32_t k1) {
  // one IMAD.WIDE.U32 each: (hi, lo) = M * c
  const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c0;
  const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c2;
  const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
  const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
  c0 = hi1 ^ c1 ^ k0;
  c1 = lo1;
  c2 = hi0 ^ c3 ^ k1;
  c3 = lo0;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c.x, c.y, c.z, c.w, k0, k1);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
}

// Philox4x32-10 of the counter (q, 0, vid0, vid1) -- the hot path's only
// counter shape (R10: word 1 = 0, words 2/3 = the volume id).  The parts of
// rounds 0 and 1 that depend only on (vid, key) are per-volume constants
// precomputed on the host (host code philox_prefix below), so those rounds cost
// one multiply each instead of two.  Bit-identical to philox4x32_10.
struct PhiloxPrefix {
  uint32_t K0;  // vid1 ^ rk1[0]
  uint32_t K1;  // lo(M1 vid0) ^ rk0[1]
  uint32_t K2;  // hi(M0 U0) ^ rk1[1],  U0 = hi(M1 vid0) ^ rk0[0]
  uint32_t U3;  // lo(M0 U0)
};

__host__ __forceinline__ PhiloxPrefix philox_prefix(uint32_t vid0, uint32_t vid1, uint32_t key0,
                                                    uint32_t key1) {
  const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * vid0;
  const uint32_t u0 = static_cast<uint32_t>(p1 >> 32) ^ key0;
  const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * u0;
  PhiloxPrefix P;
  P.K0 = vid1 ^ key1;
  P.K1 = static_cast<uint32_t>(p1) ^ (key0 + kPhiloxW0);
  P.K2 = static_cast<uint32_t>(p0 >> 32) ^ (key1 + kPhiloxW1);
  P.U3 = static_cast<uint32_t>(p0);
  return P;
}

// rk0/rk1: the 10 round keys (k + r W); only rounds 2..9 are read.
__device__ __forceinline__ uint4 philox_block(uint32_t q, const PhiloxPrefix& P,
                                              const uint32_t* rk0, const uint32_t* rk1) {
  // round 0: c = (q, 0, vid0, vid1)
  const uint64_t a = static_cast<uint64_t>(kPhiloxM0) * q;
  const uint32_t c2a = static_cast<uint32_t>(a >> 32) ^ P.K0;
  const uint32_t c3a = static_cast<uint32_t>(a);
  // round 1: c = (U0, lo(M1 vid0), c2a, c3a)
  const uint64_t b = static_cast<uint64_t>(kPhiloxM1) * c2a;
  uint32_t c0 = static_cast<uint32_t>(b >> 32) ^ P.K1;
  uint32_t c1 = static_cast<uint32_t>(b);
  uint32_t c2 = c3a ^ P.K2;
  uint32_t c3 = P.U3;
#pragma unroll
  for (int r = 2; r < 10; ++r) philox_round(c0, c1, c2, c3, rk0[r], rk1[r]);
  return make_uint4(c0, c1, c2, c3);
}

// NB (4, or 2 for 8-row tiles) blocks (counters q[0..NB-1]) in lockstep: each
// round key is read once for all, and the independent multiply chains overlap.
// Bit-identical to NB philox_block calls.
template <int NB = 4>
__device__ __forceinline__ void philox_block4(const uint32_t q[NB], const PhiloxPrefix& P,
                                              const uint32_t* rk0, const uint32_t* rk1,
                                              uint4 out[NB]) {
  uint32_t c0[NB], c1[NB], c2[NB], c3[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const uint64_t a = static_cast<uint64_t>(kPhiloxM0) * q[b];
    const uint32_t c2a = static_cast<uint32_t>(a >> 32) ^ P.K0;
    const uint32_t c3a = static_cast<uint32_t>(a);
    const uint64_t m = static_cast<uint64_t>(kPhiloxM1) * c2a;
    c0[b] = static_cast<uint32_t>(m >> 32) ^ P.K1;
    c1[b] = static_cast<uint32_t>(m);
    c2[b] = c3a ^ P.K2;
    c3[b] = P.U3;
  }
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    const uint32_t k0 = rk0[r], k1 = rk1[r];
#pragma unroll
    for (int b = 0; b < NB; ++b) philox_round(c0[b], c1[b], c2[b], c3[b], k0, k1);
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) out[b] = make_uint4(c0[b], c1[b], c2[b], c3[b]);
}

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller on the two word pairs of one Philox block (R10):
//   u1 = (2 (ua >> 9) + 1) 2^-24 in (0,1),   s = (ub >> 8) 2^-23 - 1 in [-1,1)
//   R  = sqrt(-2 ln u1);  n_even = R cos(pi s), n_odd = R sin(pi s)
// returns (n0, n1, n2, n3) = pair (r.x, r.y) then pair (r.z, r.w).
//
// Arithmetic (all exact up to the marked roundings):
//   f = 1 + (ua >> 9) 2^-23 built from the bits (no int->float conversion);
//   u1 = f - (1 - 2^-24) and t = 1 - u1 are exact.
//   -2 ln u1: MUFU lg2 (absolute error <= 2^-22.6) times -2 ln 2 when
//   t >= 2^-14; below, the series 2t + t^2 (truncation (2/3) t^3 < 2^-29.6
//   relative).  The MUFU branch's absolute error 2.3e-7 in R^2 = -2 ln u1 gives
//   |dR| <= 2.3e-7 / (2 sqrt(2 * 2^-14)) = 1.0e-5 at the threshold (less above).
//   R = r2 rsqrt(r2) (relative error ~2^-22.9); sin/cos by MUFU on pi s (one
//   rounding of the angle, absolute error ~2^-20.5).
// Worst case |n_gpu - n| < 1.1e-5, i.e. < 2.2e-4 HU at sigma = 20 HU (DESIGN.md
// tolerance budget).
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  return __ffma2_rn(a, b, c);
}

__device__ __forceinline__ float4 box_muller4(uint4 r) {
  const float2 f = make_float2(__uint_as_float(0x3F800000u | (r.x >> 9)),
                               __uint_as_float(0x3F800000u | (r.z >> 9)));
  const float2 u1 = fadd2(f, make_float2(-0.99999994039535522f, -0.99999994039535522f));
  const float2 t = fadd2(make_float2(1.0f, 1.0f), make_float2(-u1.x, -u1.y));
  const float2 ser = ffma2(t, t, fadd2(t, t));  // 2t + t^2
  const float2 lg = fmul2(make_float2(lg2_approx(u1.x), lg2_approx(u1.y)),
                          make_float2(-1.38629436f, -1.38629436f));  // -2 ln 2 lg2 u1
  const float2 r2 = make_float2(t.x < 0x1.0p-14f ? ser.x : lg.x, t.y < 0x1.0p-14f ? ser.y : lg.y);
  const float2 R = fmul2(r2, make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y)));
  // angle = pi s = j (pi 2^-23) - pi, one rounding
  const float2 ang = ffma2(make_float2(__uint2float_rn(r.y >> 8), __uint2float_rn(r.w >> 8)),
                           make_float2(3.14159265358979f * 0x1.0p-23f, 3.14159265358979f * 0x1.0p-23f),
                           make_float2(-3.14159274f, -3.14159274f));
  float s0, c0, s1, c1;
  __sincosf(ang.x, &s0, &c0);
  __sincosf(ang.y, &s1, &c1);
  const float2 a = fmul2(make_float2(R.x, R.x), make_float2(c0, s0));
  const float2 b = fmul2(make_float2(R.y, R.y), make_float2(c1, s1));
  return make_float4(a.x, a.y, b.x, b.y);
}

}  // namespace w3d
