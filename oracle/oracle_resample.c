/*
 * oracle_resample.c -- TEST INFRASTRUCTURE ONLY (see oracle_warp3d.h).
 *
 * The resampling step before the network (Rister et al., arXiv 1811.11226,
 * Sec. V.A): "Gaussian smoothing,
 * which serves as a lowpass filter to avoid aliasing artifacts, followed by
 * interpolation at the new resolution", with
 *
 *   g(x) proportional to exp(-sum_k x_k^2 / sigma_k^2)
 *   sigma_k = (1/3) max(r / u_k - 1, 0), r = 3 mm
 *
 * Readings (R22-R25): x_k in input voxels; the kernel is sampled at
 * integer offsets |i_k| <= ceil(3 sigma_k) and normalised to sum 1; voxels
 * beyond the volume replicate the nearest edge voxel (so smoothing a constant
 * returns the constant); output dims max(1, floor(n_k u_k / r + 1/2)); output
 * voxel j samples input coordinate c_in + (j - c_out) r / u_k (centre-aligned,
 * R3), trilinear for images, nearest for labels (never smoothed).
 *
 * The smoothing here is the 3D definition evaluated directly (one triple sum per
 * voxel, double precision), not the separable passes the CUDA path uses.
 */
#include <math.h>
#include <stdlib.h>

#include "oracle_warp3d.h"

void oracle_resample_sigma(const double u[3], double r, double sigma[3]) {
  for (int k = 0; k < 3; ++k) {
    const double q = r / u[k] - 1.0;
    sigma[k] = (q > 0.0 ? q : 0.0) / 3.0;
  }
}

void oracle_resample_dims(const int32_t in_dims[3], const double u[3], double r,
                          int32_t out_dims[3]) {
  for (int k = 0; k < 3; ++k) {
    const double m = floor((double)in_dims[k] * u[k] / r + 0.5);
    out_dims[k] = m < 1.0 ? 1 : (int32_t)m;
  }
}

int32_t oracle_gauss_radius(double sigma) { return sigma > 0.0 ? (int32_t)ceil(3.0 * sigma) : 0; }

/* Normalised 1D taps w[0 .. 2R] for offsets -R .. R. */
static void gauss_taps(double sigma, int32_t R, double* w) {
  double sum = 0.0;
  for (int32_t i = -R; i <= R; ++i) {
    w[i + R] = sigma > 0.0 ? exp(-(double)i * (double)i / (sigma * sigma)) : 1.0;
    sum += w[i + R];
  }
  for (int32_t i = 0; i <= 2 * R; ++i) w[i] /= sum;
}

static int32_t clampi(int32_t v, int32_t lo, int32_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* out(x) = sum_{i in box} g(i) in(clamp(x + i)), g(i) = prod_k w_k(i_k):
 * the 3D kernel of PAPER.md:487 sampled and normalised (sum of the product of
 * normalised 1D factors is 1). */
void oracle_smooth3d(const float* in, const int32_t dims[3], const double sigma[3],
                     double* out) {
  const int32_t nx = dims[0], ny = dims[1], nz = dims[2];
  int32_t R[3];
  double* w[3];
  for (int k = 0; k < 3; ++k) {
    R[k] = oracle_gauss_radius(sigma[k]);
    w[k] = (double*)malloc(sizeof(double) * (size_t)(2 * R[k] + 1));
    gauss_taps(sigma[k], R[k], w[k]);
  }
  for (int32_t z = 0; z < nz; ++z)
    for (int32_t y = 0; y < ny; ++y)
      for (int32_t x = 0; x < nx; ++x) {
        double acc = 0.0;
        for (int32_t k = -R[2]; k <= R[2]; ++k) {
          const int32_t zz = clampi(z + k, 0, nz - 1);
          for (int32_t j = -R[1]; j <= R[1]; ++j) {
            const int32_t yy = clampi(y + j, 0, ny - 1);
            for (int32_t i = -R[0]; i <= R[0]; ++i) {
              const int32_t xx = clampi(x + i, 0, nx - 1);
              const double g = w[0][i + R[0]] * w[1][j + R[1]] * w[2][k + R[2]];
              acc += g * (double)in[((size_t)zz * ny + yy) * nx + xx];
            }
          }
        }
        out[((size_t)z * ny + y) * nx + x] = acc;
      }
  for (int k = 0; k < 3; ++k) free(w[k]);
}

/* Centre-aligned scale map (R3, R25): A = diag(r / u_k), b = c_in - A c_out,
 * evaluated in double and rounded once to fp32 (as warp3d_compose_affine). */
void oracle_resample_affine(const int32_t in_dims[3], const int32_t out_dims[3], const double u[3],
                            double r, float A[12]) {
  for (int k = 0; k < 12; ++k) A[k] = 0.0f;
  for (int k = 0; k < 3; ++k) {
    const double s = r / u[k];
    const double c_in = 0.5 * ((double)in_dims[k] - 1.0), c_out = 0.5 * ((double)out_dims[k] - 1.0);
    A[4 * k + k] = (float)s;
    A[4 * k + 3] = (float)(c_in - s * c_out);
  }
}
