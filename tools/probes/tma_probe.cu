// Standalone probe of the TMA staging primitives used by warp3d_tma_kernel:
// a 4D tensor map in __grid_constant__ parameter space, box (W, R, 1, 1),
// mbarrier expect_tx / try_wait.  Prints per-case status.  (Debug tool.)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

struct alignas(64) Args {
  CUtensorMap tm;
  int x, y, z, v;
  int bytes;
  int* status;
  float* dump;
};

extern __shared__ __align__(16) unsigned char smem[];

__global__ void probe(const __grid_constant__ Args a) {
  __shared__ __align__(8) unsigned long long mbar_s;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&mbar_s);
  const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sbase = (sraw + 127u) & ~127u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(a.bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sbase),
        "l"(reinterpret_cast<uint64_t>(&a.tm)), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.v), "r"(mbar)
        : "memory");
  }
  uint32_t done = 0, tries = 0;
  for (; tries < (1u << 22) && !done; ++tries) {
    asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P; }"
                 : "=r"(done) : "r"(mbar), "r"(0u) : "memory");
  }
  if (threadIdx.x == 0) { a.status[0] = done; a.status[1] = tries; a.status[2] = sraw; }
  __syncthreads();
  const float* s = reinterpret_cast<const float*>(smem + (sbase - sraw));
  for (int i = threadIdx.x; i < 64; i += blockDim.x) a.dump[i] = s[i];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  printf("encode fn %p q=%d\n", p, (int)q);
  const int nx = 32, ny = 32, nz = 32, nv = 1;
  std::vector<float> h(nx * ny * nz * nv);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int* st; cudaMalloc(&st, 16); float* dump; cudaMalloc(&dump, 256);
  struct Case { int W, R, x, y, z; } cases[] = {{16, 4, 0, 0, 0}, {16, 4, -4, 0, 0}, {40, 4, 4, 5, 7}, {16, 4, 0, -1, -1}, {16, 4, 28, 30, 31}, {16, 4, -16, -2, 33}, {16, 4, 2, 0, 0}};
  for (auto c : cases) {
    Args a;
    const cuuint64_t dims[4] = {nx, ny, nz, nv};
    const cuuint64_t strides[3] = {nx * 4ull, nx * ny * 4ull, nx * ny * nz * 4ull};
    const cuuint32_t box[4] = {(cuuint32_t)c.W, (cuuint32_t)c.R, 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.x = c.x; a.y = c.y; a.z = c.z; a.v = 0; a.bytes = c.W * c.R * 4; a.status = st; a.dump = dump;
    cudaMemset(st, 0xff, 16);
    probe<<<1, 128, 8192>>>(a);
    cudaError_t e = cudaDeviceSynchronize();
    int hs[4]; float hd[8];
    cudaMemcpy(hs, st, 16, cudaMemcpyDeviceToHost); cudaMemcpy(hd, dump, 32, cudaMemcpyDeviceToHost);
    printf("W=%d R=%d at (%d,%d,%d): encode=%d launch=%s done=%d tries=%d sraw=%d  s[0..3]=%g %g %g %g\n",
           c.W, c.R, c.x, c.y, c.z, (int)r, cudaGetErrorString(e), hs[0], hs[1], hs[2], hd[0], hd[1], hd[2], hd[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
