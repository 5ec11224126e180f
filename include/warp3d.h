/*
 * warp3d.h -- C ABI of the B200 (sm_100a) 3D CT augmentation library.
 *
 * Implements the per-training-iteration augmentation of Rister et al.,
 * "CT organ segmentation using GPU data augmentation, unsupervised labels and
 * IOU loss", arXiv 1811.11226, Sec. IV:
 *
 *   I_affine(x) = I_in(A x + b)
 *   image: trilinear; labels: nearest neighbour
 *   I_occ(x)    = 0 inside an axis-aligned prism in z
 *   I_noise(x)  = I_occ(x) + n(x), n ~ N(0, sigma^2) iid
 *   I_window(x) = min(max((I_noise(x) - a)/(b - a), 0), 1) PAPER.md:455-467
 *   gamma: w <- w^gamma (north-star addition; not in the paper)
 *
 * The arithmetic contract the paper leaves open (voxel centres, border mode,
 * rounding of p, tie rule, RNG mapping, ...) is DESIGN.md readings R1-R21;
 * the numbers below (R4, R6, ...) refer to them.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 * - Layout: volumes are dense [batch][nz][ny][nx], x fastest (R1).  Voxel
 *   (x,y,z) has its centre at integer coordinates.  w3d_dims is (nx, ny, nz).
 * - Pointers named in/out/labels/ctr are DEVICE pointers owned by the caller;
 *   structs and the affine of warp3d_affine are HOST pointers, read before the
 *   call returns.  The library never allocates, frees or synchronises on the
 *   hot path; launches are asynchronous on `stream` (a cudaStream_t; NULL =
 *   legacy default stream).
 * - Errors: every function returns a w3d_status.  Invalid arguments are
 *   rejected BEFORE any launch with W3D_ERR_INVALID_ARG; a failed launch
 *   returns W3D_ERR_CUDA.  warp3d_last_error() gives a thread-local message
 *   for the last non-OK status.  Asynchronous kernel faults surface at the
 *   caller's next synchronisation.  No C++ exception crosses this ABI.
 * - Output must not overlap input (gathers read arbitrary input voxels).
 */
#ifndef WARP3D_H
#define WARP3D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 3: + warp3d_pipeline_create_ex / warp3d_pipeline_vols_per_job (multi-volume jobs),
 *      warp3d_compose_params_batched, warp3d_params_from_arrays (additive) */
#define WARP3D_ABI_VERSION 3

typedef enum {
  W3D_OK = 0,
  W3D_ERR_INVALID_ARG = 1, /* bad pointer / dims / params; nothing launched   */
  W3D_ERR_UNSUPPORTED = 2, /* valid but outside this build (e.g. > 2^31 voxels
                              per volume)                                      */
  W3D_ERR_CUDA = 3,        /* a CUDA runtime call or launch failed              */
  W3D_ERR_INTERNAL = 4
} w3d_status;

typedef enum {
  W3D_INTERP_LINEAR = 0,   /* trilinear                        */
  W3D_INTERP_NEAREST = 1   /* nearest, round half up (R7)                        */
} w3d_interp;

/* Kernel variant selector for warp3d_affine_batched_ex (tests / benchmarks).
   Both variants compute bit-identical results (same arithmetic, R4-R14).     */
typedef enum {
  W3D_KERNEL_AUTO = 0,     /* library choice: STAGED for the volumes whose
                              16-row tile box fits the staging buffer; the others
                              (large rotations / scales) in their own launches of
                              16 x 8 x 16 tiles with fixed-dims TMA boxes (half the
                              box height), GATHER when even those do not fit     */
  W3D_KERNEL_GATHER = 1,   /* every corner gathered through L1/L2 (__ldg) with
                              per-corner bounds                                  */
  W3D_KERNEL_STAGED = 2    /* per-tile source footprint staged in shared memory
                              (16 x 16 x 16 output tiles): volumes whose worst-
                              case tile box fits the buffer load one fixed-dims
                              box per tile by TMA (cp.async.bulk.tensor; image
                              and, when its 16 B aligned box fits beside it,
                              labels -- else labels by cp.async); other volumes
                              use per-tile exact boxes by cp.async, split into
                              2 / 4 y-parts when larger than the buffer,
                              gathered beyond that.  Layouts without 16 B chunks
                              (nx % 4 != 0, unaligned input) and dims >= 2^21
                              gather.                         */
} w3d_kernel;

typedef struct {
  int32_t nx, ny, nz;      /* each in [1, 2^24); nx*ny*nz < 2^31                 */
} w3d_dims;

/* Photometric flag bits (w3d_photometric.flags). */
enum {
  W3D_PH_NOISE = 1u,   /* v += sigma * n, Philox4x32-10 + Box-Muller (R10)       */
  W3D_PH_WINDOW = 2u,  /* v = (v - a)/(b - a)  (R14)               */
  W3D_PH_CLAMP = 4u,   /* v = min(max(v, 0), 1); requires WINDOW                 */
  W3D_PH_GAMMA = 8u,   /* v = v^gamma; requires WINDOW|CLAMP (R13)               */
  W3D_PH_OCCLUDE = 16u /* image = 0 for occ_z0 <= z <= occ_z0 + occ_height, all
                          later steps skipped, labels untouched (R15)            */
};

typedef struct {
  uint32_t flags;      /* W3D_PH_* bits; unknown bits -> INVALID_ARG              */
  float window_lo;     /* a (HU), finite; a < b when WINDOW        */
  float window_hi;     /* b (HU), finite                                          */
  float gamma;         /* > 0, finite when GAMMA; gamma == 1 skips the step       */
  float noise_sigma;   /* >= 0, finite, HU                     */
  uint32_t _reserved;  /* must be 0                                               */
  uint64_t seed;       /* Philox key (key0 = low 32 bits, key1 = high)            */
  uint64_t volume_id;  /* GLOBAL sample index: Philox counter words 2,3 (R10)     */
  float occ_z0;        /* occlusion prism start (output z), finite                */
  float occ_height;    /* delta >= 0, finite                                      */
} w3d_photometric;     /* 48 bytes */

typedef struct {
  float affine[12];    /* row-major [A | b]: OUTPUT voxel coords -> INPUT coords,
                          p_k = fma(A_k1, y, fma(A_k0, x, fma(A_k2, z, b_k))) in
                          fp32 (R4).  Finite, |A_kj| <= 2^20, |b_k| <= 2^30.      */
  w3d_photometric ph;
} w3d_volume_params;   /* 96 bytes */

/* Host-side description of a random geometric transform. */
typedef struct {
  double rot_rad[3];   /* Euler angles about x, y, z                            */
  double scale[3];     /* per-axis, > 0                                         */
  double shear[3];     /* xy, xz, yz entries of a unit upper-triangular Sh      */
  int32_t flip[3];     /* 0/1 per axis -> F = diag(+-1) (footnote PAPER.md:408)  */
  int32_t _reserved;
  double generic[9];   /* G = I + generic, row-major ("generic affine warping") */
  double disp[3];      /* d (voxels): output centre maps to input centre + d     */
} w3d_geom;

/*
 * warp3d_affine -- one volume.  out(x) = photometric(I_in(A x + b)).
 *   in       device float [in.nz][in.ny][in.nx]
 *   affine   host float[12], see w3d_volume_params.affine
 *   interp   image interpolation (trilinear per PAPER.md:416-417, or nearest)
 *   fill     image value of out-of-volume trilinear corners (R6), finite
 *   ph       host, NULL = no photometric step
 *   out      device float [out.nz][out.ny][out.nx], must not overlap `in`
 */
w3d_status warp3d_affine(const float* in, w3d_dims in_dims, const float affine[12],
                         w3d_interp interp, float fill, const w3d_photometric* ph,
                         float* out, w3d_dims out_dims, void* stream);

/*
 * warp3d_affine_batched -- `batch` volumes of identical in_dims / out_dims,
 * each with its own transform and photometric parameters (PAPER.md:406-410,
 * 445-446, 460-461: parameters are drawn per training example), plus the
 * matching nearest-neighbour label warp.
 *   in         device float [batch][in]
 *   in_labels  device uint8 [batch][in], or NULL (no label warp)
 *   params     host array [batch]
 *   label_fill label of voxels whose nearest input voxel is outside (R8)
 *   out        device float [batch][out]
 *   out_labels device uint8 [batch][out]; NULL iff in_labels is NULL
 * Volume i's noise stream is keyed by params[i].ph.(seed, volume_id) only,
 * so results do not depend on batch size, order, split or GPU count.
 */
w3d_status warp3d_affine_batched(int32_t batch, const float* in, const uint8_t* in_labels,
                                 w3d_dims in_dims, const w3d_volume_params* params,
                                 w3d_interp interp, float fill, uint8_t label_fill,
                                 float* out, uint8_t* out_labels, w3d_dims out_dims,
                                 void* stream);

/* Same, with an explicit kernel variant (results are identical by contract). */
w3d_status warp3d_affine_batched_ex(int32_t batch, const float* in, const uint8_t* in_labels,
                                    w3d_dims in_dims, const w3d_volume_params* params,
                                    w3d_interp interp, float fill, uint8_t label_fill,
                                    float* out, uint8_t* out_labels, w3d_dims out_dims,
                                    w3d_kernel variant, void* stream);

/*
 * warp3d_affine_batched_v -- a batch of volumes of DIFFERENT dims (NEXT-4:
 * "CT scans vary in resolution and number of slices"), each a
 * separate device allocation, warped into one uniform output batch (the
 * paper's fixed training crop).
 *   in_type      element type of every image: W3D_IN_F32 or W3D_IN_I16.
 *   in           host array [batch] of device pointers to the images
 *                [nz_i][ny_i][nx_i] (caller-owned).
 *   in_labels    host array [batch] of device uint8 label pointers, or NULL.
 *   in_dims      host array [batch] of the volumes' dims.
 *   params, interp, fill, label_fill, out, out_labels, out_dims: as
 *                warp3d_affine_batched (out = [batch][out_dims], slot i = volume i).
 * Volumes with equal dims share a launch (one per distinct dims); the result
 * of each volume equals warp3d_affine_batched on that volume alone.
 */
typedef enum { W3D_IN_F32 = 0, W3D_IN_I16 = 1 } w3d_in_type;
w3d_status warp3d_affine_batched_v(int32_t batch, w3d_in_type in_type, const void* const* in,
                                   const uint8_t* const* in_labels, const w3d_dims* in_dims,
                                   const w3d_volume_params* params, w3d_interp interp, float fill,
                                   uint8_t label_fill, float* out, uint8_t* out_labels,
                                   w3d_dims out_dims, void* stream);

/*
 * warp3d_affine_batched_i16[_ex] -- the batched warp with an int16 image input
 * (CT is 12-bit HU; 2 B per input voxel instead
 * of 4).  Identical to warp3d_affine_batched[_ex] except that `in` is int16
 * [batch][nz][ny][nx] (2-byte aligned); every input voxel converts to float
 * exactly (R17b) and the rest of the chain is unchanged, so the result equals
 * warp3d_affine_batched on the same volume stored as float32, bit for bit.
 * Staged paths need nx % 8 == 0, a 16 B aligned input and an integral `fill` in
 * int16 range (others gather).
 */
w3d_status warp3d_affine_batched_i16(int32_t batch, const int16_t* in, const uint8_t* in_labels,
                                     w3d_dims in_dims, const w3d_volume_params* params,
                                     w3d_interp interp, float fill, uint8_t label_fill, float* out,
                                     uint8_t* out_labels, w3d_dims out_dims, void* stream);
w3d_status warp3d_affine_batched_i16_ex(int32_t batch, const int16_t* in, const uint8_t* in_labels,
                                        w3d_dims in_dims, const w3d_volume_params* params,
                                        w3d_interp interp, float fill, uint8_t label_fill,
                                        float* out, uint8_t* out_labels, w3d_dims out_dims,
                                        w3d_kernel variant, void* stream);

/*
 * warp3d_compose_affine -- host only (no GPU needed).  A = F Rz Ry Rx Sh S G
 * (R16), b = c_in + d - A c_out with c = (n - 1)/2 per axis (PAPER.md:411-413,
 * R3), evaluated in double and rounded once to fp32 into affine_out[12].
 */
w3d_status warp3d_compose_affine(const w3d_geom* g, w3d_dims in_dims, w3d_dims out_dims,
                                 float affine_out[12]);

/*
 * warp3d_compose_params_batched -- host only: out[i].affine = warp3d_compose_affine(
 * geoms[i]) and out[i].ph = ph[i] for i < n (one call per training batch instead of
 * one per volume; the per-volume draws of PAPER.md:403-446 stay the caller's).
 * Arrays of n elements, caller-owned; the photometric fields are validated as
 * warp3d_affine_batched would.  W3D_ERR_INVALID_ARG names the first bad volume.
 */
w3d_status warp3d_compose_params_batched(int32_t n, const w3d_geom* geoms,
                                         const w3d_photometric* ph, w3d_dims in_dims,
                                         w3d_dims out_dims, w3d_volume_params* out);

/*
 * warp3d_params_from_arrays -- host only: the same from per-volume arrays (a training
 * loop's draws as numpy columns, no structs to fill): rot / scale / shear / disp
 * double [n][3] (x, y, z), flip uint8 [n][3] (nonzero = flip), generic double [n][9]
 * (G - I, row-major) or NULL, window double [n][2] (lo, hi), gamma / sigma double [n],
 * volume_ids uint64 [n] or NULL (0 .. n-1), occ_z0 / occ_height double [n] or NULL
 * (occ_height[i] >= 0 adds W3D_PH_OCCLUDE to `flags` for volume i); the photometric
 * values are rounded to the float32 fields of w3d_photometric.  shear, flip,
 * disp: NULL = zeros.  Validation and errors as warp3d_compose_params_batched.
 */
w3d_status warp3d_params_from_arrays(int32_t n, w3d_dims in_dims, w3d_dims out_dims,
                                     const double* rot, const double* scale, const double* shear,
                                     const uint8_t* flip, const double* disp,
                                     const double* generic, uint32_t flags,
                                     const double* window, const double* gamma, const double* sigma,
                                     uint64_t seed, const uint64_t* volume_ids,
                                     const double* occ_z0, const double* occ_height,
                                     w3d_volume_params* out);

/*
 * warp3d_noise -- test hook: out[v] = sigma * n(seed, volume_id, v) over a
 * dense volume of `dims` (the noise term of PAPER.md:442 alone, R10).
 */
w3d_status warp3d_noise(float* out, w3d_dims dims, float sigma, uint64_t seed,
                        uint64_t volume_id, void* stream);

/*
 * warp3d_philox4x32_10 -- test hook: n independent Philox4x32-10 blocks.
 *   ctr  device uint32 [n][4];  out device uint32 [n][4];  key = (lo, hi) of `key`.
 */
w3d_status warp3d_philox4x32_10(const uint32_t* ctr, uint64_t key, uint32_t* out, int64_t n,
                                void* stream);

/*
 * warp3d_footprint_batched -- measurement helper (not on the hot path).
 * Counts the distinct input voxels the warp touches: counts[0] = #F_img
 * (in-volume trilinear corners with nonzero extent, i.e. every corner of every
 * sample whose p is not fully out of bounds), counts[1] = #F_lbl (in-volume
 * nearest voxels).  marks: device uint8 scratch [2][batch][in] (overwritten);
 * counts: device uint64 [2] (overwritten).  Used for the algorithmic-bytes
 * roofline.
 */
w3d_status warp3d_footprint_batched(int32_t batch, w3d_dims in_dims,
                                    const w3d_volume_params* params, w3d_dims out_dims,
                                    uint8_t* marks, unsigned long long* counts, void* stream);

/*
 * Resampling to r mm before the network ("Resampling consists
 * of Gaussian smoothing, which serves as a lowpass filter to avoid aliasing
 * artifacts, followed by interpolation at the new resolution").
 * spacing_mm = (u_x, u_y, u_z) of the input voxels, target_mm = r (the paper's 3).
 * Readings (R22-R25):
 *   sigma_k = max(r / u_k - 1, 0) / 3
 *   g(x) ~ exp(-sum_k x_k^2 / sigma_k^2), x in input voxels,
 *   sampled at |i_k| <= ceil(3 sigma_k), normalised to sum 1 per axis; voxels
 *   beyond the volume replicate the nearest edge voxel (a constant stays constant)
 *   out dims_k = max(1, floor(n_k u_k / r + 1/2))
 *   output voxel j samples input c_in + (j - c_out) r / u_k (centre-aligned, R3):
 *   trilinear for the image, nearest for the labels (never smoothed), border fill
 *   (R6, R8) for the rare samples beyond the edge.
 */
/* sigma_out[3] (host only). */
w3d_status warp3d_resample_sigma(const double spacing_mm[3], double target_mm,
                                 double sigma_out[3]);
/* Output dims (host only). */
w3d_status warp3d_resample_dims(w3d_dims in_dims, const double spacing_mm[3], double target_mm,
                                w3d_dims* out_dims);
/* The centre-aligned scale map [A|b] (host only; R4 contract of warp3d_affine). */
w3d_status warp3d_resample_affine(w3d_dims in_dims, w3d_dims out_dims, const double spacing_mm[3],
                                  double target_mm, float affine_out[12]);
/*
 * warp3d_smooth3d -- the separable Gaussian lowpass alone.  in, out, tmp: device
 * float32 [nz][ny][nx], caller-owned, pairwise disjoint (tmp = scratch).
 * sigma: host double[3] per axis (x, y, z), >= 0; at most 63 taps per axis
 * (sigma <= 10.33, else W3D_ERR_UNSUPPORTED); ny, nz <= 65535.  Passes x, y, z
 * (axes with sigma 0 skipped), fp32 accumulation in tap order.  Async on stream.
 */
w3d_status warp3d_smooth3d(const float* in, w3d_dims dims, const double sigma[3], float* out,
                           float* tmp, void* stream);
/*
 * warp3d_resample -- smoothing + interpolation of one volume (and its labels).
 * in / in_labels: device [in_dims] (labels nullable); out / out_labels: device
 * [out_dims], out_dims must equal warp3d_resample_dims(); tmp: device float32
 * scratch of 2 * in_dims voxels; all disjoint.  fill / label_fill: values beyond
 * the input (R6, R8).  Async on stream.
 */
w3d_status warp3d_resample(const float* in, const uint8_t* in_labels, w3d_dims in_dims,
                           const double spacing_mm[3], double target_mm, float fill,
                           uint8_t label_fill, float* out, uint8_t* out_labels,
                           w3d_dims out_dims, float* tmp, void* stream);

/*
 * FIFO pipeline ("a first-in first-out (FIFO) queue to
 * pipeline jobs ... while one image is being processed, the next has already
 * begun transferring"): augments a batch held in HOST memory.  A job is
 * vols_per_job consecutive volumes of the batch (the last job of a call may
 * hold fewer); job j uses device slot j % depth: copy-in stream (one H2D of the
 * job's images, one of its labels) -> compute stream (warp3d_affine_batched on
 * the slot) -> copy-out stream (D2H), each ordered by events, so H2D of job
 * j+1, the warp of job j and the D2H of job j-1 overlap.  The paper's jobs are
 * single volumes (vols_per_job = 1); warp3d_pipeline_create picks vols_per_job
 * automatically (jobs of >= 96 MB of input, at most 8 volumes: with both copy
 * directions busy, per-volume copies of a 13 MB volume reach 47 GB/s per
 * direction on a B200 host link, 4-volume copies 49), warp3d_pipeline_create_ex
 * takes it as an argument (0 = automatic; 1 .. 104; else W3D_ERR_INVALID_ARG)
 * and warp3d_pipeline_vols_per_job reports it.  Host buffers should be pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous.
 *
 * warp3d_pipeline_create allocates the slots' device buffers, streams and
 * events (not on the hot path); warp3d_pipeline_run performs no allocation: it
 * enqueues all jobs, makes them start after the work already queued on
 * `stream` and makes `stream` wait for the last copy-out, and returns without
 * synchronising (the outputs are valid after `stream` completes).
 * `flags` (create): W3D_PIPE_LABELS (= 1, the former with_labels) allocates
 * label slots; W3D_PIPE_CHAIN (= 2) orders each call after the previous calls
 * on the same pipeline only (slot by slot), not after everything queued on
 * `stream`: the next batch's copy-in then overlaps the previous batch's
 * warp and copy-out instead of waiting for it to drain.  With CHAIN the caller
 * guarantees that in_host holds its data when the call is made and that no
 * pending device work still reads out_host; the first call of a pipeline
 * still starts after the work queued on `stream`.  Unknown bits:
 * W3D_ERR_INVALID_ARG.
 *   in_host          float [batch][in]   (read)
 *   in_labels_host   uint8 [batch][in] or NULL (requires with_labels)
 *   out_host         float [batch][out]  (written)
 *   out_labels_host  uint8 [batch][out]; NULL iff in_labels_host is NULL
 */
typedef struct w3d_pipeline w3d_pipeline;
enum { W3D_PIPE_LABELS = 1, W3D_PIPE_CHAIN = 2 };
w3d_status warp3d_pipeline_create(int32_t depth, w3d_dims in_dims, w3d_dims out_dims,
                                  int32_t flags, w3d_pipeline** out);
w3d_status warp3d_pipeline_create_ex(int32_t depth, int32_t vols_per_job, w3d_dims in_dims,
                                     w3d_dims out_dims, int32_t flags, w3d_pipeline** out);
int32_t warp3d_pipeline_vols_per_job(const w3d_pipeline* p);
w3d_status warp3d_pipeline_run(w3d_pipeline* p, int32_t batch, const float* in_host,
                               const uint8_t* in_labels_host, const w3d_volume_params* params,
                               w3d_interp interp, float fill, uint8_t label_fill,
                               float* out_host, uint8_t* out_labels_host, void* stream);
w3d_status warp3d_pipeline_destroy(w3d_pipeline* p);

/* Number of kernels this library has launched in this process (evidence for
 * bench.py's gpu_launches). */
uint64_t warp3d_launch_count(void);

/* Diagnostics: out[0] = output tiles computed from a staged shared-memory box,
 * out[1] = tiles computed by gathers (variant GATHER, unaligned inputs, or a
 * footprint larger than the staging buffer), out[2] = the staged tiles whose box
 * came by TMA, out[3] = the staged tiles split into y-parts; cumulative in this
 * process.  Synchronises the device (not for the hot path). */
w3d_status warp3d_tile_stats(uint64_t out[4]);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* warp3d_last_error(void);

int warp3d_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WARP3D_H */
