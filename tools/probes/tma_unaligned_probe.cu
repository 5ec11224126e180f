// TMA 3D box loads with unaligned inner (x) origins: u8 and f32 maps.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
struct alignas(64) Args { CUtensorMap tm; int x, y, z, bytes; int* status; unsigned char* dump; };
extern __shared__ __align__(128) unsigned char smem[];
__global__ void probe(const __grid_constant__ Args a) {
  __shared__ __align__(8) unsigned long long mbar_s;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&mbar_s);
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem) + 127u) & ~127u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(a.bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sbase), "l"(reinterpret_cast<uint64_t>(&a.tm)), "r"(a.x), "r"(a.y), "r"(a.z), "r"(mbar) : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  for (uint32_t tries = 0; tries < (1u << 20) && !done; ++tries)
    asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P; }" : "=r"(done) : "r"(mbar), "r"(0u) : "memory");
  if (threadIdx.x == 0) *a.status = done ? 1 : 2;
  unsigned char* s = smem + (sbase - (uint32_t)__cvta_generic_to_shared(smem));
  for (int i = threadIdx.x; i < a.bytes; i += blockDim.x) a.dump[i] = s[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  const int nx = 128, ny = 64, nz = 8;
  for (int es : {1, 4}) {
    std::vector<unsigned char> h((size_t)nx * ny * nz * es);
    for (size_t i = 0; i < h.size() / es; ++i) {
      if (es == 1) h[i] = (unsigned char)(i * 7 + 3);
      else { float f = (float)i; memcpy(&h[i * 4], &f, 4); }
    }
    unsigned char* d; cudaMalloc(&d, h.size()); cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    int* st; cudaMalloc(&st, 4); unsigned char* dump; cudaMalloc(&dump, 1 << 16);
    const int bw = es == 1 ? 32 : 20, bh = 8, bd = 4;
    Args a{};
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t strides[2] = {(cuuint64_t)nx * es, (cuuint64_t)nx * ny * es};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd}, es3[3] = {1, 1, 1};
    CUresult r = enc(&a.tm, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es3,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("es %d encode %d\n", es, (int)r);
    for (int x0 : {0, 1, 3, 5, 13, -3, 120, 113}) {
      a.x = x0; a.y = 3; a.z = 2; a.bytes = bw * bh * bd * es; a.status = st; a.dump = dump;
      cudaMemset(st, 0, 4);
      probe<<<1, 128, a.bytes + 256>>>(a);
      cudaError_t e = cudaDeviceSynchronize();
      int s = -1; cudaMemcpy(&s, st, 4, cudaMemcpyDeviceToHost);
      std::vector<unsigned char> o(a.bytes); cudaMemcpy(o.data(), dump, a.bytes, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int z = 0; z < bd; ++z) for (int y = 0; y < bh; ++y) for (int x = 0; x < bw; ++x) {
        int gx = x0 + x, gy = 3 + y, gz = 2 + z;
        bool in = gx >= 0 && gx < nx;
        size_t gi = ((size_t)gz * ny + gy) * nx + gx;
        for (int b = 0; b < es; ++b) {
          unsigned char want = in ? h[gi * es + b] : 0, got = o[((size_t)(z * bh + y) * bw + x) * es + b];
          bad += want != got;
        }
      }
      printf("  es %d x0 %4d: err=%s status=%d mismatches=%d\n", es, x0, cudaGetErrorString(e), s, bad);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
