/*
 * oracle_warp3d.c -- TEST INFRASTRUCTURE ONLY (see oracle_warp3d.h).
 *
 * A plain single-threaded implementation of the per-output-voxel chain of
 * Rister et al., arXiv 1811.11226, Sec. IV:
 *
 *   occlusion test -> pull-back coordinate p = A x + b -> trilinear image /
 *   nearest label sample -> additive Gaussian noise -> window/clamp -> gamma
 *
 * Every step follows the paper's definition in the paper's order, in double
 * precision, except the coordinate p itself, which is evaluated by the fp32
 * FMA nesting fixed by DESIGN.md reading R4 (the paper does not state the
 * precision; bit-exact labels need one agreed rounding of p).  No blocking,
 * fusion, hoisting or reordering: one voxel at a time, z -> y -> x.
 *
 * Compile: gcc -O2 -ffp-contract=off -fPIC -shared (no fast-math).
 * Pins: tests/test_oracle_*.py.
 */
#include "oracle_warp3d.h"

#include <math.h>
#include <stddef.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), the counter-based RNG  */
/* that replaces the paper's per-thread cuRAND generators (*/
/* DESIGN.md reading R10).  Constants are the published Philox4x32 ones.     */
/* ------------------------------------------------------------------------ */
static const uint32_t PHILOX_M0 = 0xD2511F53u;
static const uint32_t PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u; /* golden ratio        */
static const uint32_t PHILOX_W1 = 0xBB67AE85u; /* sqrt(3) - 1         */

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PHILOX_W0; /* key schedule: bumped between rounds */
    k1 += PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Noise counter mapping (R10): output voxel (x, y, z) of a volume of
 * dims (mx, my, mz) uses Philox block q = x + mx * (floor(y/4) + Gy * z),
 * Gy = ceil(my/4), with counter (lo q, hi q, lo id, hi id) and key
 * (lo seed, hi seed); its lane is y mod 4.  Lanes 0,1 share words (r0, r1),
 * lanes 2,3 share (r2, r3).  u1 in (0,1) and s in [-1,1) are exact in fp32. */
void oracle_noise_uniforms(uint64_t seed, uint64_t volume_id, const int32_t dims[3],
                           int32_t x, int32_t y, int32_t z, double* u1, double* s) {
  uint64_t Gy = ((uint64_t)dims[1] + 3u) / 4u;
  uint64_t q = (uint64_t)x + (uint64_t)dims[0] * ((uint64_t)(y / 4) + Gy * (uint64_t)z);
  unsigned lane = (unsigned)(y % 4);
  uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), (uint32_t)volume_id,
                     (uint32_t)(volume_id >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  oracle_philox4x32_10(ctr, key, r);
  uint32_t ua = lane < 2 ? r[0] : r[2];
  uint32_t ub = lane < 2 ? r[1] : r[3];
  *u1 = (2.0 * (double)(ua >> 9) + 1.0) * ldexp(1.0, -24);
  *s = 2.0 * ((double)(ub >> 8) * ldexp(1.0, -24)) - 1.0;
}

/* Box-Muller: n = sqrt(-2 ln u1) * (cos | sin)(pi s); even lanes (y even) take
 * the cosine, odd lanes the sine.  Standard normal. */
double oracle_noise_normal(uint64_t seed, uint64_t volume_id, const int32_t dims[3],
                           int32_t x, int32_t y, int32_t z) {
  double u1, s;
  oracle_noise_uniforms(seed, volume_id, dims, x, y, z, &u1, &s);
  double R = sqrt(-2.0 * log(u1));
  double angle = M_PI * s;
  return (y % 2) ? R * sin(angle) : R * cos(angle);
}

void oracle_noise_field(float* out, const int32_t dims[3], float sigma, uint64_t seed,
                        uint64_t volume_id) {
  size_t idx = 0;
  for (int32_t z = 0; z < dims[2]; ++z)
    for (int32_t y = 0; y < dims[1]; ++y)
      for (int32_t x = 0; x < dims[0]; ++x, ++idx)
        out[idx] = (float)((double)sigma * oracle_noise_normal(seed, volume_id, dims, x, y, z));
}

/* ------------------------------------------------------------------------ */
/* Affine composition: A is a product of rotation,        */
/* scaling, shearing, reflection and generic affine factors; the order is    */
/* DESIGN.md reading R16: A = F Rz Ry Rx Sh S G.  b = c + d - A c, with       */
/* c = (n - 1)/2 per axis (R3); for different in/out dims b = c_in + d -     */
/* A c_out, so that A c_out + b = c_in + d.               */
/* ------------------------------------------------------------------------ */
static void matmul3(const double a[9], const double b[9], double c[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += a[3 * i + k] * b[3 * k + j];
      c[3 * i + j] = acc;
    }
}

void oracle_compose_affine(const orc_geom* g, const int32_t in_dims[3],
                           const int32_t out_dims[3], double affine_d[12],
                           float affine_f[12]) {
  double cx = cos(g->rot_rad[0]), sx = sin(g->rot_rad[0]);
  double cy = cos(g->rot_rad[1]), sy = sin(g->rot_rad[1]);
  double cz = cos(g->rot_rad[2]), sz = sin(g->rot_rad[2]);
  const double Rx[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
  const double Ry[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};
  const double Rz[9] = {cz, -sz, 0, sz, cz, 0, 0, 0, 1};
  const double Sh[9] = {1, g->shear[0], g->shear[1], 0, 1, g->shear[2], 0, 0, 1};
  const double S[9] = {g->scale[0], 0, 0, 0, g->scale[1], 0, 0, 0, g->scale[2]};
  const double F[9] = {g->flip[0] ? -1.0 : 1.0, 0, 0, 0, g->flip[1] ? -1.0 : 1.0, 0,
                       0, 0, g->flip[2] ? -1.0 : 1.0};
  double G[9];
  for (int i = 0; i < 9; ++i) G[i] = g->generic[i] + ((i % 4) == 0 ? 1.0 : 0.0);

  double t1[9], t2[9], A[9];
  matmul3(F, Rz, t1);   /* F Rz            */
  matmul3(t1, Ry, t2);  /* F Rz Ry         */
  matmul3(t2, Rx, t1);  /* F Rz Ry Rx      */
  matmul3(t1, Sh, t2);  /* ... Sh          */
  matmul3(t2, S, t1);   /* ... S           */
  matmul3(t1, G, A);    /* ... G           */

  double c_in[3], c_out[3];
  for (int k = 0; k < 3; ++k) {
    c_in[k] = 0.5 * ((double)in_dims[k] - 1.0);
    c_out[k] = 0.5 * ((double)out_dims[k] - 1.0);
  }
  for (int k = 0; k < 3; ++k) {
    double Ac = A[3 * k + 0] * c_out[0] + A[3 * k + 1] * c_out[1] + A[3 * k + 2] * c_out[2];
    double b = c_in[k] + g->disp[k] - Ac;
    for (int j = 0; j < 3; ++j) affine_d[4 * k + j] = A[3 * k + j];
    affine_d[4 * k + 3] = b;
  }
  for (int i = 0; i < 12; ++i) affine_f[i] = (float)affine_d[i];
}

/* ------------------------------------------------------------------------ */
/* Per-voxel chain                                                           */
/* ------------------------------------------------------------------------ */

/* Input voxel j = (jx, jy, jz) with per-corner out-of-bounds fill (R6). */
static double image_at(const float* in, const int32_t n[3], long jx, long jy, long jz,
                       float fill) {
  if (jx < 0 || jy < 0 || jz < 0 || jx >= n[0] || jy >= n[1] || jz >= n[2]) return fill;
  return in[((size_t)jz * (size_t)n[1] + (size_t)jy) * (size_t)n[0] + (size_t)jx];
}

static double lerp(double a, double b, double t) { return a + t * (b - a); }

typedef struct {
  double value;   /* image output */
  int label;      /* label output */
} voxel_result;

static voxel_result one_voxel(const float* in, const uint8_t* in_lbl, const int32_t n[3],
                              const float A[12], int32_t interp, float fill,
                              uint8_t label_fill, const orc_photometric* ph,
                              const int32_t m[3], int32_t x, int32_t y, int32_t z) {
  voxel_result r;
  uint32_t flags = ph ? ph->flags : 0u;

  /* Step 1 -- coordinate map p = A x + b, evaluated
   * as fmaf(A_k1, y, fmaf(A_k0, x, fmaf(A_k2, z, b_k))) in fp32 (R4). */
  float X = (float)x, Y = (float)y, Z = (float)z;
  float p[3];
  for (int k = 0; k < 3; ++k)
    p[k] = fmaf(A[4 * k + 1], Y, fmaf(A[4 * k + 0], X, fmaf(A[4 * k + 2], Z, A[4 * k + 3])));

  /* Label: nearest neighbour, round half up (R7),
   * label_fill when the nearest voxel is outside the volume (R8). */
  r.label = label_fill;
  if (in_lbl) {
    int inside = 1;
    long rr[3];
    for (int k = 0; k < 3; ++k) {
      if (!((double)p[k] >= -0.5 && (double)p[k] < (double)n[k] - 0.5)) { inside = 0; break; }
      double fl = floor((double)p[k]);
      rr[k] = (long)fl + (((double)p[k] - fl) >= 0.5 ? 1 : 0);
    }
    if (inside)
      r.label = in_lbl[((size_t)rr[2] * (size_t)n[1] + (size_t)rr[1]) * (size_t)n[0] +
                       (size_t)rr[0]];
  }

  /* Occlusion (reading R15): an occluded voxel's image is
   * exactly 0 and every later step is skipped; labels are untouched. */
  if ((flags & ORC_OCCLUDE) &&
      (double)z >= (double)ph->occ_z0 &&
      (double)z <= (double)ph->occ_z0 + (double)ph->occ_height) {
    r.value = 0.0;
    return r;
  }

  /* Step 2 -- image sample I_in(p). */
  double v;
  int any_far = 0;
  for (int k = 0; k < 3; ++k)
    if (!((double)p[k] > -1.0 && (double)p[k] < (double)n[k])) any_far = 1;
  if (any_far) {
    v = fill; /* every trilinear corner is out of bounds (R6) */
  } else {
    double fl[3], f[3];
    for (int k = 0; k < 3; ++k) { fl[k] = floor((double)p[k]); f[k] = (double)p[k] - fl[k]; }
    long i = (long)fl[0], j = (long)fl[1], k = (long)fl[2];
    if (interp == ORC_INTERP_NEAREST) {
      v = image_at(in, n, i + (f[0] >= 0.5), j + (f[1] >= 0.5), k + (f[2] >= 0.5), fill);
    } else {
      /* trilinear: along x, then y, then z (R5) */
      double c00 = lerp(image_at(in, n, i, j, k, fill), image_at(in, n, i + 1, j, k, fill), f[0]);
      double c10 = lerp(image_at(in, n, i, j + 1, k, fill), image_at(in, n, i + 1, j + 1, k, fill), f[0]);
      double c01 = lerp(image_at(in, n, i, j, k + 1, fill), image_at(in, n, i + 1, j, k + 1, fill), f[0]);
      double c11 = lerp(image_at(in, n, i, j + 1, k + 1, fill), image_at(in, n, i + 1, j + 1, k + 1, fill), f[0]);
      double c0 = lerp(c00, c10, f[1]);
      double c1 = lerp(c01, c11, f[1]);
      v = lerp(c0, c1, f[2]);
    }
  }

  /* Step 3 -- additive Gaussian noise I_noise = I + n, n ~ N(0, sigma^2)
   * (PAPER.md:440-446), on every voxel including fill voxels (R9). */
  if ((flags & ORC_NOISE) && ph->noise_sigma > 0.0f) {
    v += (double)ph->noise_sigma * oracle_noise_normal(ph->seed, ph->volume_id, m, x, y, z);
  }

  /* Step 4 -- window: (v - a)/(b - a), then clamp to [0,1]. */
  if (flags & ORC_WINDOW) {
    double a = ph->window_lo, b = ph->window_hi;
    v = (v - a) / (b - a);
    if (flags & ORC_CLAMP) v = fmin(fmax(v, 0.0), 1.0);
  }

  /* Step 5 -- gamma w^gamma on the clamped window (north star; R13). */
  if ((flags & ORC_GAMMA) && ph->gamma != 1.0f) v = pow(v, (double)ph->gamma);

  r.value = v;
  return r;
}

void oracle_warp_volume(const float* in, const uint8_t* in_lbl, const int32_t in_dims[3],
                        const float affine[12], int32_t interp, float fill,
                        uint8_t label_fill, const orc_photometric* ph, float* out,
                        uint8_t* out_lbl, const int32_t out_dims[3]) {
  size_t idx = 0;
  for (int32_t z = 0; z < out_dims[2]; ++z)
    for (int32_t y = 0; y < out_dims[1]; ++y)
      for (int32_t x = 0; x < out_dims[0]; ++x, ++idx) {
        voxel_result r = one_voxel(in, in_lbl, in_dims, affine, interp, fill, label_fill, ph,
                                   out_dims, x, y, z);
        out[idx] = (float)r.value;
        if (out_lbl) out_lbl[idx] = (uint8_t)r.label;
      }
}

void oracle_warp_points(const float* in, const uint8_t* in_lbl, const int32_t in_dims[3],
                        const float affine[12], int32_t interp, float fill,
                        uint8_t label_fill, const orc_photometric* ph,
                        const int32_t out_dims[3], const int32_t* xyz, int64_t n,
                        float* out_vals, uint8_t* out_lbls) {
  for (int64_t i = 0; i < n; ++i) {
    voxel_result r = one_voxel(in, in_lbl, in_dims, affine, interp, fill, label_fill, ph,
                               out_dims, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    out_vals[i] = (float)r.value;
    if (out_lbls) out_lbls[i] = (uint8_t)r.label;
  }
}
