// philox.cuh -- Philox4x32-10 and the Box-Muller normal pair for sm_100a.
//
// Counter-based replacement for the paper's per-thread cuRAND generators
// ("a copy of the same RNG, starting at a different seed";
// DESIGN.md reading R10).  Stateless: a thread derives its words from
// (seed, volume_id, voxel >> 2) alone, so the stream is independent of launch
// shape, batch split and GPU count.  Round function: Salmon et al., SC'11.
#pragma once
#include <cstdint>

namespace w3d {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    // one IMAD.WIDE.U32 each: (hi, lo) = M * c
    const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c.z;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
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

// Same, with the 10 round keys (k0 + r W0, k1 + r W1) precomputed per volume
// (bit-identical; saves the key-schedule adds in the hot loop).
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t rk0[10],
                                                  const uint32_t rk1[10]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c.z;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c = make_uint4(hi1 ^ c.y ^ rk0[r], lo1, hi0 ^ c.w ^ rk1[r], lo0);
  }
  return c;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller on one Philox word pair (R10):
//   u1 = (2*(ua >> 9) + 1) * 2^-24  in (0,1), exact in fp32
//   s  = (ub >> 8) * 2^-23 - 1      in [-1,1), exact in fp32
//   R  = sqrt(-2 ln u1);  n_even = R cos(pi s), n_odd = R sin(pi s)
// Error budget: -2 ln u1 uses MUFU.LG2 for
// u1 <= 15/16 (absolute error ~2^-22.6 in lg2, relative < 2e-6 there) and the
// series ln(1-t) = -t(1 + t/2 + t^2/3 + t^3/4 + t^4/5), t = 1 - u1 exact, for
// u1 > 15/16 where the MUFU's absolute error would dominate (truncation
// < 2e-7 relative).  R = x * rsqrt(x); sin/cos by MUFU on pi*s in [-pi, pi)
// (absolute error ~2^-20.5; the angle itself is rounded once).  Worst case |n_gpu - n| < 1e-5, i.e. < 2e-4 HU
// at sigma = 20 HU, inside the 1e-3 HU image tolerance.
__device__ __forceinline__ float2 box_muller(uint32_t ua, uint32_t ub) {
  // u1 = k 2^-23 + 2^-24 (exact), angle = pi s = j (pi 2^-23) - pi (one rounding)
  const float u1 = __fmaf_rn(__uint2float_rn(ua >> 9), 0x1.0p-23f, 0x1.0p-24f);
  const float angle = __fmaf_rn(__uint2float_rn(ub >> 8), 3.14159265358979f * 0x1.0p-23f,
                                -3.14159274f);
  const float t = 1.0f - u1;  // exact wherever the series is used (u1 > 1/2)
  float ser = __fmaf_rn(t, 0.2f, 0.25f);
  ser = __fmaf_rn(t, ser, 0.333333343f);
  ser = __fmaf_rn(t, ser, 0.5f);
  ser = __fmaf_rn(t, ser, 1.0f);
  const float m2ln_series = 2.0f * t * ser;                       // -2 ln(1 - t)
  const float m2ln_mufu = lg2_approx(u1) * -1.38629436f;         // -2 ln 2 * lg2(u1)
  const float r2 = (t < 0.0625f) ? m2ln_series : m2ln_mufu;      // > 0
  const float R = r2 * rsqrt_approx(r2);  // r2 >= 1.1e-7: no denormal input
  float sn, cs;
  __sincosf(angle, &sn, &cs);
  return __fmul2_rn(make_float2(R, R), make_float2(cs, sn));
}

}  // namespace w3d
