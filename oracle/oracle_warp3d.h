/*
 * oracle_warp3d.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The oracle is a plain, slow, single-threaded C implementation of the
 * per-voxel augmentation of Rister et al., arXiv 1811.11226, Sec. IV
 * (PAPER.md:341-467).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant with the CUDA path (paper_1811_11226_b200/);
 * it has its own structs, declared here, which the Python test harness
 * mirrors with ctypes independently of the product binding.
 *
 * Notation: p = A x + b maps an OUTPUT voxel
 * coordinate x to the INPUT sampling coordinate p (pull-back).
 * Coordinates (x, y, z) <-> memory [z][y][x], x fastest.
 */
#ifndef ORACLE_WARP3D_H
#define ORACLE_WARP3D_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Photometric flag bits (oracle's own copy). */
#define ORC_NOISE   1u  /* additive Gaussian noise          */
#define ORC_WINDOW  2u  /* intensity affine (v-a)/(b-a)          */
#define ORC_CLAMP   4u  /* clamp to [0,1]                        */
#define ORC_GAMMA   8u  /* w^gamma (north-star addition, not in the paper)     */
#define ORC_OCCLUDE 16u /* occlusion prism in output z       */

#define ORC_INTERP_LINEAR  0
#define ORC_INTERP_NEAREST 1

typedef struct {
  uint32_t flags;
  float window_lo, window_hi; /* a < b, HU */
  float gamma;                /* > 0 */
  float noise_sigma;          /* >= 0, HU */
  uint32_t _pad0;
  uint64_t seed;              /* Philox key */
  uint64_t volume_id;         /* Philox counter high words */
  float occ_z0, occ_height;   /* occlusion prism z0 <= z <= z0 + delta */
} orc_photometric;

typedef struct {
  double rot_rad[3];  /* Euler angles about x, y, z                     */
  double scale[3];    /* per-axis scale                                 */
  double shear[3];    /* xy, xz, yz entries of unit upper-triangular Sh */
  int32_t flip[3];    /* 0/1 per axis -> F = diag(+-1)                  */
  int32_t _pad0;
  double generic[9];  /* G = I + generic (row-major)                    */
  double disp[3];     /* d in voxels                                    */
} orc_geom;

/* Philox4x32-10 (Salmon et al. 2011, "Parallel random numbers: as easy as
 * 1, 2, 3"): one block.  ctr[4], key[2] -> out[4]. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* The (u1, s) uniforms and the standard normal n used for output voxel
 * (x, y, z) of a volume of dims (mx, my, mz) with id `volume_id`
 * (reading R10). */
void oracle_noise_uniforms(uint64_t seed, uint64_t volume_id, const int32_t dims[3],
                           int32_t x, int32_t y, int32_t z, double* u1, double* s);
double oracle_noise_normal(uint64_t seed, uint64_t volume_id, const int32_t dims[3],
                           int32_t x, int32_t y, int32_t z);

/* A = F Rz Ry Rx Sh S G, b = c_in + d - A c_out.
 * Writes the double matrix [A|b] (row-major 3x4) and its fp32 rounding. */
void oracle_compose_affine(const orc_geom* g, const int32_t in_dims[3],
                           const int32_t out_dims[3], double affine_d[12],
                           float affine_f[12]);

/* One volume.  in: float [nz][ny][nx]; in_lbl: uint8 or NULL.
 * out: float [mz][my][mx]; out_lbl: uint8 or NULL (NULL iff in_lbl NULL).
 * ph may be NULL (no photometric step). */
void oracle_warp_volume(const float* in, const uint8_t* in_lbl, const int32_t in_dims[3],
                        const float affine[12], int32_t interp, float fill,
                        uint8_t label_fill, const orc_photometric* ph, float* out,
                        uint8_t* out_lbl, const int32_t out_dims[3]);

/* The same computation at n selected output voxels (x,y,z triples),
 * for sampled parity at sizes the full oracle would take too long on. */
void oracle_warp_points(const float* in, const uint8_t* in_lbl, const int32_t in_dims[3],
                        const float affine[12], int32_t interp, float fill,
                        uint8_t label_fill, const orc_photometric* ph,
                        const int32_t out_dims[3], const int32_t* xyz, int64_t n,
                        float* out_vals, uint8_t* out_lbls);

/* Standalone noise field sigma * n(v) over a volume of `dims`. */
void oracle_noise_field(float* out, const int32_t dims[3], float sigma, uint64_t seed,
                        uint64_t volume_id);

/* Resampling to r mm (oracle_resample.c). */
void oracle_resample_sigma(const double u[3], double r, double sigma[3]);
void oracle_resample_dims(const int32_t in_dims[3], const double u[3], double r,
                          int32_t out_dims[3]);
int32_t oracle_gauss_radius(double sigma);
void oracle_smooth3d(const float* in, const int32_t dims[3], const double sigma[3], double* out);
void oracle_resample_affine(const int32_t in_dims[3], const int32_t out_dims[3], const double u[3],
                            double r, float A[12]);

#ifdef __cplusplus
}
#endif

#endif
