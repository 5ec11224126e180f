// Micro-benchmark: texture-unit gathers (tld4 on a tall 2D pitch-linear float
// texture) vs shared-memory gathers for the trilinear warp's corner fetch.
// Each thread walks output rows of a rotated sampling pattern like the C3
// train transforms; reports GVoxel/s for: 2 x tld4 (image) + 1 x tex (label).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void tex_kernel(cudaTextureObject_t ti, cudaTextureObject_t tl, int nx, int ny, int nz,
                           float a00, float a01, float a02, float a10, float a11, float a12,
                           float a20, float a21, float a22, float* out, int mode) {
  const int x = blockIdx.x * 16 + (threadIdx.x & 15);
  const int z = blockIdx.z * 16 + 2 * (threadIdx.x >> 5) + ((threadIdx.x >> 4) & 1);
  const int y0 = blockIdx.y * 16;
  float acc = 0.f;
  const float cx = 0.5f * nx, cy = 0.5f * ny, cz = 0.5f * nz;
  const float t0 = a00 * (x - cx) + a02 * (z - cz) + cx;
  const float t1 = a10 * (x - cx) + a12 * (z - cz) + cy;
  const float t2 = a20 * (x - cx) + a22 * (z - cz) + cz;
  for (int y = y0; y < y0 + 16; ++y) {
    const float px = fmaf(a01, y - cy, t0), py = fmaf(a11, y - cy, t1), pz = fmaf(a21, y - cy, t2);
    const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
    const float tx = px - fx, ty = py - fy, tz = pz - fz;
    const float u = fx + 1.0f, v = fmaf(fz, (float)ny, fy) + 1.0f;
    float4 g0 = tex2Dgather<float4>(ti, u, v, 0);
    float4 g1 = tex2Dgather<float4>(ti, u, v + ny, 0);
    // tld4 returns (x: (i, j+1), y: (i+1, j+1), z: (i+1, j), w: (i, j))
    const float c00 = fmaf(tx, g0.z - g0.w, g0.w), c10 = fmaf(tx, g0.y - g0.x, g0.x);
    const float c01 = fmaf(tx, g1.z - g1.w, g1.w), c11 = fmaf(tx, g1.y - g1.x, g1.x);
    const float c0 = fmaf(ty, c10 - c00, c00), c1 = fmaf(ty, c11 - c01, c01);
    acc += fmaf(tz, c1 - c0, c0);
    if (mode) {
      const float ru = fx + (tx >= 0.5f) + 0.5f, rv = fmaf(fz + (tz >= 0.5f), (float)ny, fy + (ty >= 0.5f)) + 0.5f;
      acc += tex2D<float>(tl, ru, rv);
    }
  }
  out[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x * 256 + blockIdx.x * 256 + threadIdx.x] = acc;
}

int main() {
  const int nx = 128, ny = 128, nz = 160;
  float* img; float* lbl; float* out;
  size_t pitch = nx * 4;
  cudaMalloc(&img, (size_t)nx * ny * nz * 4);
  cudaMalloc(&lbl, (size_t)nx * ny * nz * 4);
  cudaMemset(img, 0, (size_t)nx * ny * nz * 4);
  cudaMalloc(&out, 64 << 20);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypePitch2D;
  rd.res.pitch2D.devPtr = img;
  rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
  rd.res.pitch2D.width = nx;
  rd.res.pitch2D.height = ny * nz;
  rd.res.pitch2D.pitchInBytes = pitch;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t ti, tl;
  cudaError_t e = cudaCreateTextureObject(&ti, &rd, &td, nullptr);
  rd.res.pitch2D.devPtr = lbl;
  e = cudaCreateTextureObject(&tl, &rd, &td, nullptr);
  printf("tex create: %s\n", cudaGetErrorString(e));
  const float c = cosf(0.2f), s = sinf(0.2f);
  dim3 grid(nx / 16, ny / 16, nz / 16);
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it)
      tex_kernel<<<dim3(grid.x, grid.y, grid.z * 16), 256>>>(ti, tl, nx, ny, nz, c, -s, 0.1f, s, c, 0.05f, -0.1f, 0.08f, 1.0f, out, mode);
    cudaEventRecord(a);
    const int reps = 20;
    for (int it = 0; it < reps; ++it)
      tex_kernel<<<dim3(grid.x, grid.y, grid.z * 16), 256>>>(ti, tl, nx, ny, nz, c, -s, 0.1f, s, c, 0.05f, -0.1f, 0.08f, 1.0f, out, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double vox = (double)nx * ny * nz * 16 * reps;
    printf("mode %d (%s): %.1f GVoxel/s  err=%s\n", mode, mode ? "2 tld4 + tex" : "2 tld4", vox / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
