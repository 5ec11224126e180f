// TMA box latency on an otherwise idle GPU: one CTA per SM loads a 3D float box
// (W x H x D) from a 256^3 volume resident in L2 / HBM, timing issue -> mbarrier
// completion with clock64.  Rows = H x D, bytes = 4 W H D.  Answers whether the box
// wait of the warp kernel scales with rows (TMA requests) or bytes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
struct alignas(64) Args { CUtensorMap tm; int W, H, D; unsigned long long* out; int reps; };
extern __shared__ __align__(128) unsigned char smem[];
__global__ void probe(const __grid_constant__ Args a) {
  __shared__ __align__(8) unsigned long long mbar_s;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&mbar_s);
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem) + 127u) & ~127u;
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(1) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  unsigned long long tot = 0;
  for (int r = 0; r < a.reps; ++r) {
    const int x = ((blockIdx.x * 37 + r * 53) % 200) & ~3, y = (blockIdx.x * 11 + r * 29) % 200,
              z = (blockIdx.x * 7 + r * 17) % 200;
    const long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(a.W * a.H * a.D * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sbase), "l"(reinterpret_cast<uint64_t>(&a.tm)), "r"(x), "r"(y), "r"(z), "r"(mbar) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P; }" : "=r"(done) : "r"(mbar), "r"(r & 1) : "memory");
    tot += clock64() - t0;
  }
  a.out[blockIdx.x] = tot / a.reps;
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  const int n = 256;
  float* d; cudaMalloc(&d, (size_t)n * n * n * 4); cudaMemset(d, 0, (size_t)n * n * n * 4);
  unsigned long long* out; cudaMalloc(&out, 444 * 8);
  int shapes[][3] = {{24, 21, 22}, {24, 42, 11}, {48, 21, 11}, {96, 21, 6}, {24, 10, 22}, {8, 21, 22}, {64, 16, 16}, {32, 32, 16}};
  for (auto& s : shapes) {
    Args a{};
    cuuint64_t dims[3] = {n, n, n}; cuuint64_t strides[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};
    cuuint32_t box[3] = {(cuuint32_t)s[0], (cuuint32_t)s[1], (cuuint32_t)s[2]}, es[3] = {1, 1, 1};
    enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.W = s[0]; a.H = s[1]; a.D = s[2]; a.out = out; a.reps = 20;
    const int bytes = s[0] * s[1] * s[2] * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 256);
    for (int ctas : {1, 148, 444}) {
      probe<<<ctas, 32, bytes + 256>>>(a);
      cudaDeviceSynchronize();
      unsigned long long h[444]; cudaMemcpy(h, out, 8 * ctas, cudaMemcpyDeviceToHost);
      double m = 0; int k = ctas; for (int i = 0; i < k; ++i) m += h[i]; m /= k;
      printf("box %3dx%3dx%3d rows %4d bytes %6d  ctas %3d: %7.0f cycles per box (%s)\n", s[0], s[1], s[2], s[1] * s[2], bytes, ctas, m, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
