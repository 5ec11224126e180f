// Micro-benchmark: issue throughput of the instruction classes of the warp kernel
// on sm_100a (cycles per warp-instruction per SM sub-partition, 8 independent chains,
// 4 warps per SMSP).  Prints thread-instructions per cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 4096
template <int K>
__global__ void probe(float* out, int n) {
  float2 a[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); u[i] = threadIdx.x + i; }
  const float2 m = make_float2(1.0001f, 0.9999f), c = make_float2(1e-7f, 2e-7f);
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) a[i] = __ffma2_rn(a[i], m, c);                 // FFMA2
      if (K == 1) a[i] = __fadd2_rn(a[i], c);                    // FADD2
      if (K == 2) a[i].x = __fmaf_rn(a[i].x, m.x, c.x);          // FFMA
      if (K == 3) u[i] = u[i] * 0x9E3779B9u + 7u;               // IMAD
      if (K == 4) { uint64_t p = (uint64_t)u[i] * 0xD2511F53u; u[i] = (uint32_t)(p >> 32) ^ (uint32_t)p; }  // IMAD.WIDE + LOP3
      if (K == 5) u[i] = (u[i] ^ 0x5bd1e995u) + (u[i] >> 3);    // LOP3/IADD/SHF
      if (K == 6) { a[i].x = __fmaf_rn(a[i].x, m.x, c.x); a[i].y = __fadd_rn(a[i].y, c.y); }  // FFMA + FADD
      if (K == 7) { a[i] = __ffma2_rn(a[i], m, c); u[i] = (u[i] ^ 0x5bd1e995u) + 3u; }  // FFMA2 + LOP3/IADD
      if (K == 8) { float r; asm volatile("set.ge.f32.f32 %0, %1, 0f3F000000;" : "=f"(r) : "f"(a[i].x)); a[i].x = __int_as_float(__float_as_int(r) ^ u[i]); }  // FSET + LOP3
      if (K == 9) { u[i] = __float_as_uint(__uint2float_rn(u[i])) ^ 0x1234u; }  // I2FP + LOP3
      if (K == 10) { uint64_t p = (uint64_t)u[i] * 0xD2511F53u; u[i] = (uint32_t)(p >> 32) + (uint32_t)p; a[i] = __fadd2_rn(a[i], c); }  // IMAD.WIDE + IADD + FADD2
      if (K == 11) { a[i] = __fadd2_rn(a[i], c); u[i] = u[i] * 0x9E3779B9u + 7u; }  // FADD2 + IMAD
      if (K == 12) { a[i].x = __fadd_rn(a[i].x, c.x); a[i].y = __fadd_rn(a[i].y, c.y); }  // 2 FADD
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(const char* name, float* out, double ops_per_iter) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512;  // 64 warps / SM
  probe<K><<<blocks, threads>>>(out, 16);
  cudaEventRecord(a);
  probe<K><<<blocks, threads>>>(out, N);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double warp_instr_per_sm = (double)blocks * threads / 32 * N * ops_per_iter / 148;
  printf("%-22s %.3f warp-instr/cycle/SM  (%.2f cycles per warp-instr per SMSP)\n", name,
         warp_instr_per_sm / cycles, 4 * cycles / warp_instr_per_sm);
}

int main() {
  float* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  run<0>("FFMA2", out, 8);
  run<1>("FADD2", out, 8);
  run<2>("FFMA", out, 8);
  run<3>("IMAD", out, 8);
  run<4>("IMAD.WIDE+LOP3", out, 16);
  run<5>("LOP3+SHF+IADD (alu)", out, 24);
  run<6>("FFMA+FADD", out, 16);
  run<7>("FFMA2+LOP3/IADD", out, 16);
  run<8>("FSET+LOP3", out, 16);
  run<9>("I2FP+LOP3", out, 16);
  run<10>("IMAD.WIDE+IADD+FADD2", out, 24);
  run<11>("FADD2+IMAD", out, 16);
  run<12>("FADD x2", out, 16);
  return 0;
}
