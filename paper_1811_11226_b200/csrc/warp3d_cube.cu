// warp3d_cube.cu -- host side of the warp kernel: layout
// checks, launch dispatch into the instantiation units (cube_inst_*.cu, one per
// image type x parameter block, compiled in parallel), the per-volume staging
// box (cube_cp_box) and the tile counters.  The kernel itself is
// cube_kernel.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "cube_config.cuh"
#include "warp3d_internal.cuh"

namespace w3d {
namespace cube {
template <class T, int NV>
cudaError_t launch_typed_nv(const WarpArgsT<NV>& a, bool gather_only, cudaStream_t s);
template <class T, int NV>
cudaError_t read_stats_nv(unsigned long long out[4]);

template <class T>
static cudaError_t launch_typed(const WarpArgs& a, bool gather_only, cudaStream_t s) {
  if (a.nvol > kSmallVol) return launch_typed_nv<T, kMaxVolPerLaunch>(a, gather_only, s);
  WarpArgsSmall b;  // launches of at most kSmallVol volumes pass the small parameter block
  std::memcpy(&b, &a, sizeof(b));  // header, tensor maps and vol[0, kSmallVol)
  return launch_typed_nv<T, kSmallVol>(b, gather_only, s);
}
}  // namespace cube

// Staged layouts: 16 B chunks (nx and the volume stride multiples of the chunk,
// 16 B aligned input), coordinates below 2^21 (magic-number floor), and for
// int16 input a fill that int16 represents (the staged box holds fill).
bool cube_supported(const WarpArgs& a) {
  const int chunk = a.in16 ? 8 : 4;
  const bool fill_ok = !a.in16 || (a.fill == std::nearbyint(a.fill) && a.fill >= -32768.0f &&
                                   a.fill <= 32767.0f);
  return (a.nx % chunk == 0) && a.in_aligned && fill_ok && a.nx < (1 << 21) &&
         a.ny < (1 << 21) && a.nz < (1 << 21);
}

// gather_only (W3D_KERNEL_GATHER, or layouts cube_supported() rejects): every
// tile through L1/L2 gathers.
cudaError_t launch_cube(const WarpArgs& a, bool gather_only, cudaStream_t s) {
  gather_only = gather_only || !cube_supported(a);
  const cudaError_t e = a.in16 ? cube::launch_typed<int16_t>(a, gather_only, s)
                               : cube::launch_typed<float>(a, gather_only, s);
  note_launch();
  return e;
}

// TMA image boxes: 16 B aligned global strides and volume bases (the staged
// layout), one tensor map per volume in the first kTmaVolPerLaunch volumes.
bool cube_tma_supported(const WarpArgs& a) { return cube_supported(a); }

// Staging box of one volume's tiles (TMA image box and cp.async boxes) and its
// origin offsets: the footprint of a 16 x kTY x 16 tile has extent
// ext_k = sum_j |A_kj| span_j; from the origin floor(p0 + box_mlo) the tile
// needs at most floor(ext_k + 2 margin) + 3 elements per axis (floor of the
// lower bound, the +1 trilinear corner, rounding inside the margin; the margin
// covers 16 ulp of the largest |p| of any tile voxel), plus chunk - 1 in x for
// the 16 B aligned row start.  Rows per plane padded (and the row widened by
// one chunk when no padding works) so the plane pitch spreads the two
// half-warps over the banks (tools/model_tiles.py); cp_p = cp_w * cp_h, so the
// TMA box (cp_w, cp_h, cp_d) lands with the same pitches.  cp_rows = kTY when
// the box fits the buffer, else 0 (per-tile exact boxes, parts, gathers).
// Bank model of the staged corner loads (tools/bank_model.py): a warp's 32 lanes
// (16 output x by 2 output z) read floor(p) + W floor(p_y) + W h floor(p_z) (+ a
// corner offset, which rotates every lane's bank alike), so the shared-memory
// wavefronts of a load depend on the plane pitch (W, W h) and on A.  kBankSamples
// warp-rows of two sample tiles; their floors do not depend on the pitch.
#ifndef W3D_BANK_SAMPLES
#define W3D_BANK_SAMPLES 4
#endif
constexpr int kBankSamples = W3D_BANK_SAMPLES;
struct BankFloors {
  int32_t f[kBankSamples][3][32];
};
static void bank_floors(const float A[12], const int out[3], int tile_rows, BankFloors& F) {
  const int tiles[3] = {(out[0] + 15) / 16, (out[1] + tile_rows - 1) / tile_rows, (out[2] + 15) / 16};
  for (int smp = 0; smp < kBankSamples; ++smp) {
    const int q = smp < kBankSamples / 2 ? 1 : 3;  // tiles at 1/4 and 3/4 of the grid
    const int ox = 16 * ((tiles[0] * q) / 4), oy = tile_rows * ((tiles[1] * q) / 4);
    const int oz = 16 * ((tiles[2] * q) / 4);
    const int w = (5 * smp + 2 * (smp & 1)) % (cube::THREADS / 32);
    const int r = (smp & 1) ? tile_rows - 1 : (smp * tile_rows) / (2 * kBankSamples);
    for (int l = 0; l < 32; ++l) {
      const float x = float(ox + (l & 15)), y = float(oy + r), z = float(oz + 2 * w + (l >> 4));
      for (int k = 0; k < 3; ++k) {  // clamped (no overflowing cast), floor inline (no libm)
        float q = A[4 * k] * x + A[4 * k + 1] * y + A[4 * k + 2] * z + A[4 * k + 3];
        q = q < -1073741824.0f ? -1073741824.0f : (q > 1073741824.0f ? 1073741824.0f : q);
        const int32_t t = static_cast<int32_t>(q);
        F.f[smp][k][l] = t - (q < static_cast<float>(t) ? 1 : 0);
      }
    }
  }
}
// mean over the samples of max over banks of the distinct words addressed: per bank a
// 64-bit set of the words' rows (word >> 5) mod 64 -- branch-free; rows 2048 words
// apart would alias, farther than one warp's loads reach in a staged box;
// eshift: log2 of the elements per 4-byte word (0 for float32, 1 for int16)
static int bank_cost(const BankFloors& F, int W, int h, int eshift, int bound = 1 << 30) {
  const uint32_t Wu = static_cast<uint32_t>(W), Pu = static_cast<uint32_t>(W * h);
  int tot = 0;
  for (int smp = 0; smp < kBankSamples && tot <= bound; ++smp) {  // stop once worse
    uint64_t rows[32] = {};
    for (int l = 0; l < 32; ++l) {
      // modulo 2^32 (unsigned: only the bank and equality matter)
      const uint32_t idx = (static_cast<uint32_t>(F.f[smp][0][l]) +
                            Wu * static_cast<uint32_t>(F.f[smp][1][l]) +
                            Pu * static_cast<uint32_t>(F.f[smp][2][l])) >>
                           eshift;
      rows[idx & 31] |= uint64_t(1) << ((idx >> 5) & 63);
    }
    int worst = 1;
    for (int bk = 0; bk < 32; ++bk) worst = std::max(worst, __builtin_popcountll(rows[bk]));
    tot += worst;
  }
  return tot;  // in units of 1 / kBankSamples wavefronts per load
}

void cube_cp_box(const float A[12], VolDev& P, int elem_bytes, const int /*in*/[3],
                 const int out[3], int tile_rows) {
  using namespace cube;
  const int kC = 16 / elem_bytes;
  const int cap = kCapVox * 5 / (elem_bytes + 1);
  P.cp_w = P.cp_h = P.cp_d = P.cp_rows = 0;
  P.cp_abs = 0;
  P.cp_p = 0;
  P.cp_w_bytes = P.cp_p_bytes = 0;
  P.box_w = P.box_h = P.box_d = P.box_wl = 0;
  int d[3];
  const double span[3] = {TX - 1.0, tile_rows - 1.0, TZ - 1.0};
  bool ok = true;
  for (int k = 0; k < 3; ++k) {
    double mag = std::fabs(double(A[4 * k + 3])), ext = 0.0, mlo = 0.0, mhi = 0.0;
    for (int j = 0; j < 3; ++j) {
      const double a = double(A[4 * k + j]) * span[j];
      ext += std::fabs(a);
      mlo += a < 0.0 ? a : 0.0;
      mhi += a > 0.0 ? a : 0.0;
      mag += std::fabs(double(A[4 * k + j])) * (out[j] + 16.0);  // any voxel of any tile
    }
    const double margin = 16.0 * mag * 0x1.0p-24 + 1e-3;
    P.box_mlo[k] = static_cast<float>(mlo - margin);
    P.box_mhi[k] = std::nextafter(static_cast<float>(mhi + margin), INFINITY);  // rounded up
    if (ext > 200.0) ok = false;
    d[k] = ok ? static_cast<int>(std::floor(ext + 2.0 * margin)) + 3 : 0;
  }
  if (!ok) return;
  const int W0 = (d[0] + kC - 1 + kC - 1) & ~(kC - 1), H0 = d[1], D = d[2];
  // TMA label box candidate: rows of Wl bytes from the 16 B aligned x origin
  // (lo & ~15 >= lo - 15), H0 rows per plane
  const int Wl = (d[0] + 15 + 15) & ~15;
  const int64_t lbl_bytes = int64_t(Wl) * H0 * D;
  auto img_bytes_of = [&](int64_t plane) {
    return (int64_t(elem_bytes) * plane * D + 127) & ~int64_t(127);
  };
  // smallest bank-spreading padding; one that also leaves room for the TMA
  // label box wins over a smaller one that does not (labels by cp.async cost
  // more than the bank conflicts the padding saves), and the unpadded layout
  // wins when it alone makes the label box fit
  int best_w = 0, best_h = 0;
  int64_t best = INT64_MAX;
  bool best_lbl = false;
  const int64_t room = int64_t(kCapVox) * 5;
  for (int W = W0; W <= W0 + kC; W += kC)
    for (int h = H0; h < H0 + 8; ++h) {
      const int res = (W * h) & 31;
      const bool spread = elem_bytes == 4 ? (res == 12 || res == 16 || res == 20 || res == 24)
                                          : res == 16;
      if (!spread || int64_t(W) * h * D > cap) continue;
      const bool lbl = img_bytes_of(int64_t(W) * h) + lbl_bytes <= room && Wl <= 256;
      if ((lbl && !best_lbl) || (lbl == best_lbl && int64_t(W) * h < best)) {
        best = int64_t(W) * h;
        best_w = W;
        best_h = h;
        best_lbl = lbl;
      }
    }
  const bool plain_lbl = img_bytes_of(int64_t(W0) * H0) + lbl_bytes <= room && Wl <= 256;
  if (best_w == 0 || (!best_lbl && plain_lbl)) {  // unpadded
    best_w = W0;
    best_h = H0;
  }
  // the pitch the bank model prefers among the widths W0, W0 + chunk and up to 7 rows
  // of padding, keeping the label box beside the image box if the rule above did
  // (f32 16-row boxes; W3D_BANK_MODEL=0 restores the residue rule alone)
  static const bool bank_model = !(getenv("W3D_BANK_MODEL") && getenv("W3D_BANK_MODEL")[0] == '0');
  // (float32 only: for int16 boxes the model's pick measured no change, 282.9 vs 282.9)
  // (float32 boxes of volumes with >= 256 output tiles: for a few tiles the call is
  // launch- and host-bound and the ~5 us of modelling would show)
  const int64_t ntiles = int64_t((out[0] + TX - 1) / TX) * ((out[1] + tile_rows - 1) / tile_rows) *
                         ((out[2] + TZ - 1) / TZ);
  if (bank_model && elem_bytes == 4 && ntiles >= 256) {
    const int eshift = 0;
    BankFloors F;
    bank_floors(A, out, tile_rows, F);
    const bool want_lbl = img_bytes_of(int64_t(best_w) * best_h) + lbl_bytes <= room && Wl <= 256;
    int bc = bank_cost(F, best_w, best_h, eshift);
    // search only when the rule's pitch averages more than 2 wavefronts per load (the
    // volumes with the costly conflicts; ~5 us of host time per searched volume)
    static const bool always = getenv("W3D_BANK_MODEL") && getenv("W3D_BANK_MODEL")[0] == '2';
    const bool search = always || bc > 2 * kBankSamples;
    // a candidate's banks depend on (W mod 32, W h mod 32) only (up to rare equal
    // addresses): one evaluation per residue pair, the smallest box first
    uint32_t seen[8] = {};
    seen[(best_w & 31) >> 2] |= 1u << ((best_w * best_h) & 31);
    for (int Wc = W0; search && Wc <= W0 + kC && bc > kBankSamples; Wc += kC)
      for (int h = H0; h < H0 + 8 && bc > kBankSamples; ++h) {
        if (int64_t(Wc) * h * D > cap || (Wc == best_w && h == best_h)) continue;
        const bool lbl = img_bytes_of(int64_t(Wc) * h) + lbl_bytes <= room && Wl <= 256;
        if (want_lbl && !lbl) continue;
        uint32_t& sw = seen[(Wc & 31) >> 2];
        const uint32_t bit = 1u << ((Wc * h) & 31);
        if (sw & bit) continue;
        sw |= bit;
        const int c = bank_cost(F, Wc, h, eshift, bc);
        if (c < bc || (c == bc && int64_t(Wc) * h < int64_t(best_w) * best_h)) {
          bc = c;
          best_w = Wc;
          best_h = h;
        }
      }
  }
  const int64_t Pp = int64_t(best_w) * best_h;
  if (Pp * D > cap || best_w > 4 * THREADS || best_w > 256 || best_h > 256 || D > 256) return;
  // the staged index in absolute coordinates (cube_kernel.cuh sample2 kAbs):
  // |fx + W fy + P fz| < 2^22 (the magic-number index kM +- 2^22) for every p of
  // the output volume (p is affine: its range is spanned by the 8 output corners;
  // + the rounding margin, the +1 corner and the box slack).  Otherwise the
  // volume takes the per-tile boxes.
  {
    double lim = 0.0;
    // the image and (TMA) label pitches, whichever is larger
    const double pitch[3] = {1.0, double(std::max(best_w, Wl)),
                             double(std::max<int64_t>(Pp, int64_t(Wl) * H0))};
    for (int k = 0; k < 3; ++k) {
      double lo = A[4 * k + 3], hi = A[4 * k + 3];
      for (int j = 0; j < 3; ++j) {
        const double t = double(A[4 * k + j]) * (out[j] - 1);
        lo += t < 0.0 ? t : 0.0;
        hi += t > 0.0 ? t : 0.0;
      }
      lim += pitch[k] * (std::max(std::fabs(lo), std::fabs(hi)) + 8.0);
    }
    if (!(lim < 4194304.0)) return;
  }
  P.cp_abs = 1;
  P.cp_w = static_cast<uint16_t>(best_w);
  P.cp_h = static_cast<uint16_t>(best_h);
  P.cp_d = static_cast<uint16_t>(D);
  P.cp_p = static_cast<int32_t>(Pp);
  P.cp_rows = static_cast<uint16_t>(tile_rows);
  P.cp_w_bytes = static_cast<uint16_t>(best_w * elem_bytes);
  P.cp_p_bytes = static_cast<uint16_t>(Pp * elem_bytes);
  // the TMA label box, used when it fits beside the image box (and
  // prepare_tma makes its tensor map)
  if (img_bytes_of(Pp) + lbl_bytes <= room && Wl <= 256) {
    P.box_wl = static_cast<uint16_t>(Wl);
    P.box_h = static_cast<uint16_t>(H0);
  }
}

cudaError_t read_cube_stats(unsigned long long out[4]) {
  using namespace cube;
  cudaError_t (*const parts[4])(unsigned long long*) = {
      read_stats_nv<float, kSmallVol>, read_stats_nv<float, kMaxVolPerLaunch>,
      read_stats_nv<int16_t, kSmallVol>, read_stats_nv<int16_t, kMaxVolPerLaunch>};
  for (int k = 0; k < 4; ++k) out[k] = 0;
  for (auto* f : parts) {
    unsigned long long v[4];
    const cudaError_t e = f(v);
    if (e != cudaSuccess) return e;
    for (int k = 0; k < 4; ++k) out[k] += v[k];
  }
  out[0] += out[2];  // staged = cp.async + TMA
  return cudaSuccess;
}

}  // namespace w3d
