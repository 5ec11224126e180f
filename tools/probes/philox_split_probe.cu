#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
template <int V, uint32_t M>
__device__ __forceinline__ void mulhilo(uint32_t a, uint32_t& hi, uint32_t& lo) {
  if (V == 0) { uint64_t p = (uint64_t)M * a; hi = p >> 32; lo = (uint32_t)p; }
  if (V == 1) { asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "n"(M)); asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(a), "n"(M)); }
  if (V == 2) { asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "n"(M)); asm("mad.lo.u32 %0, %1, %2, %1;" : "=r"(lo) : "r"(a), "n"(M - 1)); }
  if (V == 3) { uint32_t Mr; asm volatile("mov.b32 %0, %1;" : "=r"(Mr) : "n"(M)); asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "n"(M)); lo = a * Mr; }
  if (V == 4) { uint32_t Mr; asm volatile("mov.b32 %0, %1;" : "=r"(Mr) : "n"(M)); hi = __umulhi(a, Mr); lo = a * Mr; }
}
template <int V>
__global__ void philox(uint32_t* out, int iters, const uint32_t* __restrict__ keys) {
  uint32_t c0[4], c1[4], c2[4], c3[4];
  for (int b = 0; b < 4; ++b) { c0[b] = threadIdx.x + b; c1[b] = blockIdx.x; c2[b] = b * 77; c3[b] = 5; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t k0 = keys[2 * r], k1 = keys[2 * r + 1];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t h0, l0, h1, l1;
        mulhilo<V, M0>(c0[b], h0, l0);
        mulhilo<V, M1>(c2[b], h1, l1);
        c0[b] = h1 ^ c1[b] ^ k0; c1[b] = l1; c2[b] = h0 ^ c3[b] ^ k1; c3[b] = l0;
      }
    }
  }
  uint32_t s = 0;
  for (int b = 0; b < 4; ++b) s ^= c0[b] + c1[b] * 3 + c2[b] * 5 + c3[b] * 7;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int V>
void run(const char* name, uint32_t* out, const uint32_t* keys) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 384, N = 256;
  philox<V><<<blocks, threads>>>(out, 4, keys);
  cudaEventRecord(a);
  philox<V><<<blocks, threads>>>(out, N, keys);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double warp_rounds_per_smsp = (double)blocks * threads / 32 * N * 10 * 4 / 148 / 4;
  printf("V%d %-34s %.3f cycles per block-round per SMSP (%.3f ms)\n", V, name, cycles / warp_rounds_per_smsp, ms);
}
int main() {
  uint32_t *out, *keys; cudaMalloc(&out, 148 * 4 * 384 * 4); cudaMalloc(&keys, 80);
  cudaMemset(keys, 3, 80);
  run<0>("IMAD.WIDE", out, keys);
  run<1>("asm mul.hi + mul.lo", out, keys);
  run<2>("mul.hi + mad.lo (M-1)+a", out, keys);
  run<3>("mul.hi imm + mul.lo reg", out, keys);
  run<4>("umulhi reg + mul reg", out, keys);
  run<0>("IMAD.WIDE (again)", out, keys);
  return 0;
}
