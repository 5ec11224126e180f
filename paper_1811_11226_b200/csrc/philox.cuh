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

// Box-Muller on one Philox word pair (R10):
//   u1 = (2*(ua >> 9) + 1) * 2^-24  in (0,1), exact in fp32
//   s  = (ub >> 8) * 2^-23 - 1      in [-1,1), exact in fp32
//   R  = sqrt(-2 ln u1);  n_even = R cos(pi s), n_odd = R sin(pi s)
// logf is the accurate libdevice version (the fast __logf's absolute error
// near u1 -> 1 breaks the 1e-3 HU tolerance, SURVEY.md key finding 5).
__device__ __forceinline__ float2 box_muller(uint32_t ua, uint32_t ub) {
  const float u1 = __int2float_rn(static_cast<int>(((ua >> 9) << 1) | 1u)) * 0x1.0p-24f;
  const float s = __fmaf_rn(__int2float_rn(static_cast<int>(ub >> 8)), 0x1.0p-23f, -1.0f);
  const float R = sqrtf(-2.0f * logf(u1));
  float sn, cs;
  sincospif(s, &sn, &cs);
  return make_float2(R * cs, R * sn);
}

}  // namespace w3d
