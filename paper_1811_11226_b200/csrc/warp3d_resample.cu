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

}  // namespace

int gauss_radius(double sigma) { return sigma > 0.0 ? static_cast<int>(std::ceil(3.0 * sigma)) : 0; }

cudaError_t launch_smooth_axis(int axis, const float* in, float* out, int nx, int ny, int nz,
                               double sigma, cudaStream_t s) {
  Taps t;
  t.R = gauss_radius(sigma);
  double w[kMaxTaps], sum = 0.0;
  for (int i = -t.R; i <= t.R; ++i) {
    w[i + t.R] = std::exp(-double(i) * double(i) / (sigma * sigma));
    sum += w[i + t.R];
  }
  for (int i = 0; i <= 2 * t.R; ++i) t.w[i] = static_cast<float>(w[i] / sum);
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

}  // namespace w3d
