// Micro-benchmark: dispatch cost of the Philox multiply forms on sm_100a (8 independent
// chains, 16 warps per SMSP).  Finding: ptxas fuses umulhi + mul.lo of the same operands
// into one IMAD.WIDE.U32 (immediate or parameter multiplier alike), ~4 cycles each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 4096
template <int K>
__global__ void probe(float* out, int n, uint32_t M) {
  uint32_t u[8], v[8];
  float2 a[8], b[8], t[8];
  for (int i = 0; i < 8; ++i) {
    u[i] = threadIdx.x * 7 + i; v[i] = threadIdx.x ^ (i * 13);
    a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); b[i] = make_float2(i * 0.25f, 1.0f);
    t[i] = make_float2(0.5f + i * 1e-3f, 0.25f);
  }
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) { uint64_t p = (uint64_t)u[i] * M; u[i] = (uint32_t)(p >> 32); v[i] ^= (uint32_t)p; }  // IMAD.WIDE
      if (K == 1) { u[i] = __umulhi(u[i], M) ^ v[i]; }                                             // IMAD.HI
      if (K == 2) { uint32_t h = __umulhi(u[i], M); uint32_t l = u[i] * M; u[i] = h; v[i] ^= l; }  // HI + LO
      if (K == 3) { u[i] = u[i] * M + v[i]; }                                                      // IMAD lo
      if (K == 4) { a[i] = __ffma2_rn(t[i], __fadd2_rn(b[i], a[i]), a[i]); }                       // lerp pair form
      if (K == 5) { a[i] = __fadd2_rn(b[i], a[i]); }                                               // FADD2 2 pairs
      if (K == 6) { a[i] = __ffma2_rn(t[i], b[i], a[i]); }                                         // FFMA2 3 pairs
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + b[i].x + t[i].y + (float)(u[i] ^ v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(const char* name, float* out, double ops_per_iter) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512;
  probe<K><<<blocks, threads>>>(out, 16, 0xD2511F53u);
  cudaEventRecord(a);
  probe<K><<<blocks, threads>>>(out, N, 0xD2511F53u);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double per_smsp = (double)blocks * threads / 32 * N * ops_per_iter / 148 / 4;
  printf("%-28s %.2f cycles per op per SMSP\n", name, cycles / per_smsp);
}

int main() {
  float* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  run<0>("IMAD.WIDE (+LOP3)", out, 8);
  run<1>("IMAD.HI (+LOP3)", out, 8);
  run<2>("IMAD.HI + IMAD (+LOP3)", out, 8);
  run<3>("IMAD lo (3 regs)", out, 8);
  run<4>("lerp FADD2+FFMA2 (per lerp)", out, 8);
  run<5>("FADD2 2 pairs", out, 8);
  run<6>("FFMA2 3 pairs", out, 8);
  return 0;
}
