// warp3d_resample.cu -- resampling to r mm before the network (Rister et al.,
// arXiv 1811.11226, Sec. V.A):
// Gaussian lowpass g(x) ~ exp(-sum_k x_k^2 / sigma_k^2), sigma_k = (1/3)
// max(r/u_k - 1, 0), then interpolation at spacing r
// (trilinear image, nearest labels; labels are never smoothed).
//
// The 3D kernel is a product of 1D factors, so the smoothing runs as separable
// passes x, y, z (each an HBM-streaming stencil: every output voxel reads its
// 2R+1 neighbours along one axis through L1/L2, edge voxels replicated, fp32
// accumulation in tap order), and the interpolation is the warp kernel with a
// centre-aligned scale-only affine (warp3d_cube.cu).  Readings R22-R25.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "warp3d_internal.cuh"

namespace w3d {

namespace {

struct Taps {
  float w[kMaxTaps];  // w[0 .. 2R] for offsets -R .. R, normalised (sum 1 in double)
  int32_t R;
};

// out(x, y, z) = sum_t w[t] in(.., clamp(c + t - R), ..) along `Axis`.  One
// thread per output voxel, x fastest (coalesced for every axis).
template <int Axis>
__global__ void __launch_bounds__(256) smooth_axis_kernel(const float* __restrict__ in,
                                                          float* __restrict__ out, int nx, int ny,
                                                          int nz, const __grid_constant__ Taps t) {
  const int x = static_cast<int>(blockIdx.x) * 256 + static_cast<int>(threadIdx.x);
  const int y = static_cast<int>(blockIdx.y), z = static_cast<int>(blockIdx.z);
  if (x >= nx) return;
  const int n = Axis == 0 ? nx : (Axis == 1 ? ny : nz);
  const int c = Axis == 0 ? x : (Axis == 1 ? y : z);
  const int64_t stride = Axis == 0 ? 1 : (Axis == 1 ? int64_t(nx) : int64_t(nx) * ny);
  const int64_t base = (static_cast<int64_t>(z) * ny + y) * nx + x - int64_t(c) * stride;
  float acc = 0.0f;
  for (int k = 0; k <= 2 * t.R; ++k) {
    int j = c + k - t.R;
    j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
    acc = __fmaf_rn(t.w[k], __ldg(in + base + int64_t(j) * stride), acc);
  }
  out[(static_cast<int64_t>(z) * ny + y) * nx + x] = acc;
}

// Fused separable smoothing of one 32 x 8 x 8 output tile (radius <= kFuseR per
// axis): the input tile + halo (edge voxels replicated) is read once into shared
// memory, then the x, y and z passes run out of shared memory in the same
// order and fp32 arithmetic as smooth_axis_kernel (bit-identical results), and
// only the output tile is written back: one HBM read + one write per voxel
// instead of three of each.
constexpr int kFuseR = 8, FX = 32, FY = 8, FZ = 8;
struct Taps3 {
  float wx[2 * kFuseR + 1], wy[2 * kFuseR + 1], wz[2 * kFuseR + 1];
  int32_t rx, ry, rz;
};

extern __shared__ float fuse_smem[];

// RM: compile-time tap radius >= every axis' radius; an axis with a smaller
// radius has its weights centred and zero-padded (fma(0, v, acc) = acc exactly,
// so the result equals the per-axis passes bit for bit).
template <int RM>
__global__ void __launch_bounds__(256) smooth_fused_kernel(const float* __restrict__ in,
                                                           float* __restrict__ out, int nx, int ny,
                                                           int nz, const __grid_constant__ Taps3 t) {
  const int ox = static_cast<int>(blockIdx.x) * FX, oy = static_cast<int>(blockIdx.y) * FY,
            oz = static_cast<int>(blockIdx.z) * FZ;
  // halo RM on every axis (zero-weight taps read real, finite, edge-replicated data)
  constexpr int AX = FX + 2 * RM, AY = FY + 2 * RM, AZ = FZ + 2 * RM;
  float* A = fuse_smem;            // [AZ][AY][AX]  input + halo; later the y-pass result
  float* B = fuse_smem + AX * AY * AZ;  // [AZ][AY][FX] x-pass result
  // taps centred in 2 RM + 1 slots, zero-padded (registers)
  float wx[2 * RM + 1], wy[2 * RM + 1], wz[2 * RM + 1];
#pragma unroll
  for (int k = 0; k <= 2 * RM; ++k) {
    wx[k] = (k >= RM - t.rx && k <= RM + t.rx) ? t.wx[k - (RM - t.rx)] : 0.0f;
    wy[k] = (k >= RM - t.ry && k <= RM + t.ry) ? t.wy[k - (RM - t.ry)] : 0.0f;
    wz[k] = (k >= RM - t.rz && k <= RM + t.rz) ? t.wz[k - (RM - t.rz)] : 0.0f;
  }
  // lane = x (32 = FX), warp w walks rows (y, z) w, w + 8, ...: no per-element division
  const int lx = static_cast<int>(threadIdx.x & 31), w = static_cast<int>(threadIdx.x >> 5);
  const int gx0 = min(max(ox + lx - RM, 0), nx - 1);
  const int gx1 = min(max(ox + lx + 32 - RM, 0), nx - 1);
  const bool x1 = lx + 32 < AX;
  {
    int y = w, z = 0;
    while (y >= AY) { y -= AY; ++z; }
    for (int r = w; r < AY * AZ; r += 8) {
      const int gy = min(max(oy + y - RM, 0), ny - 1), gz = min(max(oz + z - RM, 0), nz - 1);
      const float* row = in + (static_cast<int64_t>(gz) * ny + gy) * nx;
      float* arow = A + r * AX;
      arow[lx] = __ldg(row + gx0);
      if (x1) arow[lx + 32] = __ldg(row + gx1);
      y += 8;
      while (y >= AY) { y -= AY; ++z; }
    }
  }
  __syncthreads();
  for (int r = w; r < AY * AZ; r += 8) {  // x pass: B[z][y][x], rows of A
    const float* a = A + r * AX + lx;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k <= 2 * RM; ++k) acc = __fmaf_rn(wx[k], a[k], acc);
    B[r * FX + lx] = acc;
  }
  __syncthreads();
  float* C = A;  // [AZ][FY][FX] y-pass result
  for (int r = w; r < FY * AZ; r += 8) {
    const int z = r / FY, y = r - z * FY;
    const float* b = B + (z * AY + y) * FX + lx;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k <= 2 * RM; ++k) acc = __fmaf_rn(wy[k], b[k * FX], acc);
    C[r * FX + lx] = acc;
  }
  __syncthreads();
  const int gx = ox + lx;
  for (int r = w; r < FY * FZ; r += 8) {  // z pass + store
    const int z = r / FY, y = r - z * FY;
    const int gy = oy + y, gz = oz + z;
    if (gx >= nx || gy >= ny || gz >= nz) continue;
    const float* c = C + r * FX + lx;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k <= 2 * RM; ++k) acc = __fmaf_rn(wz[k], c[k * FX * FY], acc);
    out[(static_cast<int64_t>(gz) * ny + gy) * nx + gx] = acc;
  }
}

void make_taps(double sigma, int R, float* w) {
  double d[kMaxTaps], sum = 0.0;
  for (int i = -R; i <= R; ++i) {
    d[i + R] = sigma > 0.0 ? std::exp(-double(i) * double(i) / (sigma * sigma)) : 1.0;
    sum += d[i + R];
  }
  for (int i = 0; i <= 2 * R; ++i) w[i] = static_cast<float>(d[i] / sum);
}

}  // namespace

int gauss_radius(double sigma) { return sigma > 0.0 ? static_cast<int>(std::ceil(3.0 * sigma)) : 0; }

cudaError_t launch_smooth_axis(int axis, const float* in, float* out, int nx, int ny, int nz,
                               double sigma, cudaStream_t s) {
  Taps t;
  t.R = gauss_radius(sigma);
  make_taps(sigma, t.R, t.w);
  const dim3 grid(static_cast<unsigned>((nx + 255) / 256), static_cast<unsigned>(ny),
                  static_cast<unsigned>(nz));
  if (axis == 0)
    smooth_axis_kernel<0><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  else if (axis == 1)
    smooth_axis_kernel<1><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  else
    smooth_axis_kernel<2><<<grid, 256, 0, s>>>(in, out, nx, ny, nz, t);
  note_launch();
  return cudaGetLastError();
}

bool smooth_fusable(const double sigma[3]) {
  for (int k = 0; k < 3; ++k)
    if (gauss_radius(sigma[k]) > kFuseR) return false;
  return true;
}

cudaError_t launch_smooth_fused(const float* in, float* out, int nx, int ny, int nz,
                                const double sigma[3], cudaStream_t s) {
  Taps3 t;
  t.rx = gauss_radius(sigma[0]);
  t.ry = gauss_radius(sigma[1]);
  t.rz = gauss_radius(sigma[2]);
  make_taps(sigma[0], t.rx, t.wx);
  make_taps(sigma[1], t.ry, t.wy);
  make_taps(sigma[2], t.rz, t.wz);
  const dim3 grid(static_cast<unsigned>((nx + FX - 1) / FX), static_cast<unsigned>((ny + FY - 1) / FY),
                  static_cast<unsigned>((nz + FZ - 1) / FZ));
  const int rmax = max(t.rx, max(t.ry, t.rz));
  const int RM = rmax <= 4 ? (rmax < 1 ? 1 : rmax) : (rmax <= 6 ? 6 : 8);
  const int AX = FX + 2 * RM, AY = FY + 2 * RM, AZ = FZ + 2 * RM;
  const size_t smem = sizeof(float) * (size_t(AX) * AY * AZ + size_t(FX) * AY * AZ);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kernel) {
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
    if (e == cudaSuccess) kernel<<<grid, 256, smem, s>>>(in, out, nx, ny, nz, t);
  };
  if (rmax <= 1) go(smooth_fused_kernel<1>);
  else if (rmax <= 2) go(smooth_fused_kernel<2>);
  else if (rmax <= 3) go(smooth_fused_kernel<3>);
  else if (rmax <= 4) go(smooth_fused_kernel<4>);
  else if (rmax <= 6) go(smooth_fused_kernel<6>);
  else go(smooth_fused_kernel<8>);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace w3d
