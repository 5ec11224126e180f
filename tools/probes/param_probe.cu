// Launch cost of a kernel against its parameter-block size (sm_100a):
// back-to-back launches of an empty-ish kernel with 256 B, 4 KB, 8 KB, 16 KB and
// 31 KB __grid_constant__ parameter structs, timed by events over 2000 launches;
// and a 148 x 3 CTA grid (one wave) per launch.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o param_probe param_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct Args { unsigned int w[N / 4]; };
template <int N>
__global__ void k(const __grid_constant__ Args<N> a, unsigned int* out) {
  if (a.w[threadIdx.x % (N / 4)] == 0xdeadbeefu) out[blockIdx.x] = 1;
}
template <int N> float run(unsigned int* d, int grid) {
  Args<N> a = {};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 100; ++i) k<N><<<grid, 256>>>(a, d);
  cudaEventRecord(e0);
  const int n = 2000;
  for (int i = 0; i < n; ++i) k<N><<<grid, 256>>>(a, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / n;
}
int main() {
  unsigned int* d;
  cudaMalloc(&d, 1 << 20);
  for (int grid : {1, 444, 10240}) {
    printf("grid %5d: 256B %.2f us  4KB %.2f  8KB %.2f  16KB %.2f  31KB %.2f\n", grid,
           run<256>(d, grid), run<4096>(d, grid), run<8192>(d, grid), run<16384>(d, grid),
           run<31744>(d, grid));
  }
  return 0;
}
