// warp3d_host.cu -- C-ABI entry points (include/warp3d.h): argument
// validation, per-volume parameter derivation, launch chunking, errors.
//
// Validation rejects everything outside the contract BEFORE launching
// (W3D_ERR_INVALID_ARG).  Per-volume parameters travel by value as a
// __grid_constant__ kernel argument (up to kMaxVolPerLaunch volumes per
// launch), so the hot path performs no allocation, copy or synchronisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <tuple>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "philox.cuh"
#include "warp3d.h"
#include "warp3d_internal.cuh"
#include "cube_config.cuh"

namespace w3d {
// tile heights of the staged warp kernel: kTY rows, or half as many for launches
// whose kTY-row boxes do not fit the staging buffer (AUTO, launch_group)
constexpr int kTileRows = cube::kTY, kTileRowsSmall = cube::kTY / 2;

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

static w3d_status fail(w3d_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

static w3d_status ok() {
  g_last_error.clear();
  return W3D_OK;
}

static w3d_status cuda_fail(cudaError_t e, const char* what) {
  return fail(W3D_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

constexpr int32_t kMaxDim = 1 << 23;  // n - 0.5 exact in fp32 (R8)
constexpr int64_t kMaxVoxels = (int64_t(1) << 31) - 1;

static w3d_status check_dims(const w3d_dims& d, const char* name) {
  if (d.nx < 1 || d.ny < 1 || d.nz < 1 || d.nx >= kMaxDim || d.ny >= kMaxDim || d.nz >= kMaxDim)
    return fail(W3D_ERR_INVALID_ARG, "%s = (%d, %d, %d): each must be in [1, 2^23)", name, d.nx,
                d.ny, d.nz);
  const int64_t n = int64_t(d.nx) * d.ny * d.nz;
  if (n > kMaxVoxels)
    return fail(W3D_ERR_UNSUPPORTED, "%s has %lld voxels (> 2^31 - 1 per volume)", name,
                static_cast<long long>(n));
  return W3D_OK;
}

static int64_t nvox(const w3d_dims& d) { return int64_t(d.nx) * d.ny * d.nz; }

static bool overlap(const void* a, int64_t abytes, const void* b, int64_t bbytes) {
  if (!a || !b) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + static_cast<uintptr_t>(bbytes) && b0 < a0 + static_cast<uintptr_t>(abytes);
}

static w3d_status check_affine(const float* A, int i) {
  for (int k = 0; k < 12; ++k) {
    const float v = A[k];
    const float lim = (k % 4 == 3) ? 1073741824.0f /* 2^30 */ : 1048576.0f /* 2^20 */;
    if (!std::isfinite(v) || std::fabs(v) > lim)
      return fail(W3D_ERR_INVALID_ARG,
                  "volume %d: affine[%d] = %g (must be finite, |A| <= 2^20, |b| <= 2^30)", i, k,
                  static_cast<double>(v));
  }
  return W3D_OK;
}

static w3d_status check_ph(const w3d_photometric& ph, int i) {
  const uint32_t known = W3D_PH_NOISE | W3D_PH_WINDOW | W3D_PH_CLAMP | W3D_PH_GAMMA |
                         W3D_PH_OCCLUDE;
  if (ph.flags & ~known) return fail(W3D_ERR_INVALID_ARG, "volume %d: unknown flags 0x%x", i, ph.flags);
  if (ph._reserved != 0) return fail(W3D_ERR_INVALID_ARG, "volume %d: _reserved must be 0", i);
  if ((ph.flags & W3D_PH_CLAMP) && !(ph.flags & W3D_PH_WINDOW))
    return fail(W3D_ERR_INVALID_ARG, "volume %d: CLAMP requires WINDOW", i);
  if ((ph.flags & W3D_PH_GAMMA) && !((ph.flags & W3D_PH_WINDOW) && (ph.flags & W3D_PH_CLAMP)))
    return fail(W3D_ERR_INVALID_ARG, "volume %d: GAMMA requires WINDOW and CLAMP", i);
  if (ph.flags & W3D_PH_WINDOW) {
    if (!std::isfinite(ph.window_lo) || !std::isfinite(ph.window_hi) ||
        !(ph.window_lo < ph.window_hi))
      return fail(W3D_ERR_INVALID_ARG, "volume %d: window needs finite a < b (a=%g, b=%g)", i,
                  double(ph.window_lo), double(ph.window_hi));
    const double s = 1.0 / (double(ph.window_hi) - double(ph.window_lo));
    if (!std::isfinite(static_cast<float>(s)))
      return fail(W3D_ERR_INVALID_ARG, "volume %d: 1/(b-a) overflows fp32", i);
  }
  if ((ph.flags & W3D_PH_GAMMA) && !(std::isfinite(ph.gamma) && ph.gamma > 0.0f))
    return fail(W3D_ERR_INVALID_ARG, "volume %d: gamma must be finite and > 0", i);
  if ((ph.flags & W3D_PH_NOISE) && !(std::isfinite(ph.noise_sigma) && ph.noise_sigma >= 0.0f))
    return fail(W3D_ERR_INVALID_ARG, "volume %d: noise_sigma must be finite and >= 0", i);
  if ((ph.flags & W3D_PH_OCCLUDE) &&
      !(std::isfinite(ph.occ_z0) && std::isfinite(ph.occ_height) && ph.occ_height >= 0.0f))
    return fail(W3D_ERR_INVALID_ARG, "volume %d: occlusion needs finite z0 and height >= 0", i);
  return W3D_OK;
}

// Host-side derivation of the kernel's per-volume parameters.
static VolDev derive(const float* A, const w3d_photometric* ph) {
  VolDev P;
  std::memset(&P, 0, sizeof(P));
  std::memcpy(P.A, A, sizeof(P.A));
  P.gamma = 1.0f;
  P.win_s = 1.0f;
  P.win_off = 0.0f;
  P.clamp_lo = -INFINITY;
  P.clamp_hi = INFINITY;
  if (!ph) return P;
  uint32_t f = 0;
  if ((ph->flags & W3D_PH_NOISE) && ph->noise_sigma > 0.0f) {
    f |= kNoise;
    P.sigma = ph->noise_sigma;
  }
  if (ph->flags & W3D_PH_WINDOW) {
    const double a = ph->window_lo, b = ph->window_hi;
    P.win_s = static_cast<float>(1.0 / (b - a));
    P.win_off = static_cast<float>(-a * double(P.win_s));
  }
  if (ph->flags & W3D_PH_CLAMP) {
    P.clamp_lo = 0.0f;
    P.clamp_hi = 1.0f;
  }
  if ((ph->flags & W3D_PH_GAMMA) && ph->gamma != 1.0f) {
    f |= kGamma;
    P.gamma = ph->gamma;
  }
  if (ph->flags & W3D_PH_OCCLUDE) {
    // z0 <= z <= z0 + delta over integer z  <=>  ceil(z0) <= z <= floor(z0 + delta),
    // the sum in double exactly as the oracle evaluates it (R15).
    const double lo = std::ceil(double(ph->occ_z0));
    const double hi = std::floor(double(ph->occ_z0) + double(ph->occ_height));
    const double clo = lo < -2e9 ? -2e9 : (lo > 2e9 ? 2e9 : lo);
    const double chi = hi < -2e9 ? -2e9 : (hi > 2e9 ? 2e9 : hi);
    P.occ_lo = static_cast<int32_t>(clo);
    P.occ_hi = static_cast<int32_t>(chi);
    if (P.occ_lo <= P.occ_hi) f |= kOcclude;
  }
  P.flags = f;
  const uint32_t key0 = static_cast<uint32_t>(ph->seed);
  const uint32_t key1 = static_cast<uint32_t>(ph->seed >> 32);
  const uint32_t vid0 = static_cast<uint32_t>(ph->volume_id);
  const uint32_t vid1 = static_cast<uint32_t>(ph->volume_id >> 32);
  for (int r = 0; r < 10; ++r) {  // Philox key schedule (philox.cuh); rk*[0] = the key
    P.rk0[r] = key0 + static_cast<uint32_t>(r) * 0x9E3779B9u;
    P.rk1[r] = key1 + static_cast<uint32_t>(r) * 0xBB67AE85u;
  }
  const PhiloxPrefix pp = philox_prefix(vid0, vid1, key0, key1);
  P.ph_K0 = pp.K0;
  P.ph_K1 = pp.K1;
  P.ph_K2 = pp.K2;
  P.ph_U3 = pp.U3;
  return P;
}

// ---------------------------------------------------------------------------
// TMA tensor maps: one 3D map per volume for the image (float32) and one for
// the labels (uint8), box dims = the volume's tile footprint (cube_tma_box).
// Encoded with the driver's cuTensorMapEncodeTiled (fetched through the
// runtime); a per-slot cache skips re-encoding identical maps.
// ---------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// elem: 1 = uint8 labels, 2 = int16 image, 4 = float32 image
static bool encode_3d(CUtensorMap* m, int elem, const void* base, const WarpArgs& a, uint32_t bw,
                      uint32_t bh, uint32_t bd) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const cuuint64_t es = static_cast<cuuint64_t>(elem);
  const CUtensorMapDataType dt = elem == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16  // raw int16 bits
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const cuuint64_t dims[3] = {cuuint64_t(a.nx), cuuint64_t(a.ny), cuuint64_t(a.nz)};
  const cuuint64_t strides[2] = {cuuint64_t(a.nx) * es, cuuint64_t(a.nx) * a.ny * es};
  const cuuint32_t box[3] = {bw, bh, bd};
  const cuuint32_t estr[3] = {1, 1, 1};
  // no L2 promotion: a box row is 24-48 elements, and promoting its sector reads to
  // 256 B fetched DRAM bytes no sample uses (C4: 214.6 GVoxel/s without, 199.0 with
  // 256 B; C3 / C5 / C2 / int16 unchanged).  A/B knob W3D_L2PROMO: 0 none (default),
  // 1 64 B, 2 128 B, 3 256 B.
  static const int promo = getenv("W3D_L2PROMO") ? atoi(getenv("W3D_L2PROMO")) : 0;
  const CUtensorMapL2promotion pr =
      promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                 : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                              : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  return enc(m, dt, 3,
             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct MapKey {
  const void* base = nullptr;
  int32_t nx = 0, ny = 0, nz = 0;
  uint32_t bw = 0, bh = 0, bd = 0;
  int32_t elem = 0;
  bool operator==(const MapKey& o) const {
    return base == o.base && nx == o.nx && ny == o.ny && nz == o.nz && bw == o.bw &&
           bh == o.bh && bd == o.bd && elem == o.elem;
  }
};

// Encoded maps by key, direct-mapped (per host thread): a training loop's new
// transforms change the box dims every step, but over the steps the same few hundred
// (address, dims, box) combinations recur, and a hit is a 128 B copy instead of a
// cuTensorMapEncodeTiled call (~1 us; 32 per C3 launch).
static bool encode_cached(CUtensorMap* dst, const MapKey& k, const WarpArgs& a) {
  struct Entry {
    MapKey key;
    CUtensorMap map;
  };
  constexpr int kEntries = 1024;
  static thread_local Entry* table = new Entry[kEntries]();
  uint64_t h = reinterpret_cast<uint64_t>(k.base) * 0x9E3779B97F4A7C15ull;
  for (const uint32_t v : {uint32_t(k.nx), uint32_t(k.ny), uint32_t(k.nz), k.bw, k.bh, k.bd,
                           uint32_t(k.elem)})
    h = (h ^ v) * 0x100000001B3ull;
  Entry& e = table[(h >> 20) & (kEntries - 1)];
  if (e.key == k && k.base != nullptr) {
    std::memcpy(dst, &e.map, sizeof(CUtensorMap));
    return true;
  }
  if (!encode_3d(dst, k.elem, k.base, a, k.bw, k.bh, k.bd)) return false;
  e.key = k;
  std::memcpy(&e.map, dst, sizeof(CUtensorMap));
  return true;
}

// Image tensor maps of the launch chunk in `args` (volumes whose staging box
// fits, cube_cp_box); returns false (and clears every box) when encoding is
// unavailable.
static bool prepare_tma(WarpArgs& args) {
  static thread_local MapKey key_img[kTmaVolPerLaunch], key_lbl[kTmaVolPerLaunch];
  bool ok = get_encode() != nullptr;
  const int eb = args.in16 ? 2 : 4;
  // label maps: 16 B aligned rows and bases
  static const bool no_tma_lbl = getenv("W3D_NO_TMA_LBL") && getenv("W3D_NO_TMA_LBL")[0] == '1';
  bool lbl_ok = args.in_lbl != nullptr && args.nx % 16 == 0 && !no_tma_lbl;
  for (int32_t i = 0; lbl_ok && i < args.nvol; ++i) lbl_ok = args.vol[i].lbl_addr % 16 == 0;
  for (int32_t i = 0; i < args.nvol && i < kTmaVolPerLaunch && ok; ++i) {
    VolDev& P = args.vol[i];
    P.box_w = P.box_d = 0;
    if (P.cp_rows == 0) {
      P.box_wl = 0;
      continue;
    }
    const void* base = reinterpret_cast<const void*>(P.in_addr);
    MapKey ki{base, args.nx, args.ny, args.nz, P.cp_w, P.cp_h, P.cp_d, eb};
    if (!(ki == key_img[i])) {
      key_img[i] = MapKey();
      ok = encode_cached(&args.tm[2 * i], ki, args);
      if (ok) key_img[i] = ki;
    }
    if (ok) {
      P.box_w = P.cp_w;
      P.box_d = P.cp_d;
    }
    if (ok && lbl_ok && P.box_wl != 0) {
      MapKey kl{reinterpret_cast<const void*>(P.lbl_addr), args.nx, args.ny, args.nz, P.box_wl,
                P.box_h, P.cp_d, 1};
      bool lok = true;
      if (!(kl == key_lbl[i])) {
        key_lbl[i] = MapKey();
        lok = encode_cached(&args.tm[2 * i + 1], kl, args);
        if (lok) key_lbl[i] = kl;
      }
      if (!lok) P.box_wl = 0;
    } else {
      P.box_wl = 0;
    }
  }
  if (!ok)
    for (int32_t i = 0; i < args.nvol; ++i) args.vol[i].box_w = args.vol[i].box_wl = 0;
  return ok;
}

// Tile order of a launch (WarpArgs::brick): volumes much larger than L2 whose
// footprint boxes are large (the 8-row launches: large rotations) traverse the
// output in bricks of 2^s x 2^s x 2^s tiles (y doubled for 8-row tiles), so the
// input a wave reads is compact and its reuse by neighbouring tiles hits in L2.
// Needs power-of-two tile counts per brick row / column (else 0: launch order).
// W3D_BRICK=<log2 tiles> overrides (0 = off; experiments).
static int32_t brick_order(const WarpArgs& a, bool gather) {
  static const int env = getenv("W3D_BRICK") ? atoi(getenv("W3D_BRICK")) : -1;
  const int s = env >= 0 ? env : (a.tile_rows != kTileRows && !gather ? 2 : 0);
  if (s <= 0) return 0;
  const int sy = s + (a.tile_rows == kTileRows ? 0 : 1);
  const int64_t tx = (a.mx + cube::TX - 1) / cube::TX, ty = (a.my + a.tile_rows - 1) / a.tile_rows;
  const int64_t tz = (a.mz + cube::TZ - 1) / cube::TZ;
  auto lg = [](int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return (int64_t(1) << l) == v ? l : -1;
  };
  if (tx % (1 << s) || ty % (1 << sy) || tz % (1 << s)) return 0;
  const int lbx = lg(tx >> s), lby = lg(ty >> sy);
  if (lbx < 0 || lby < 0 || lbx > 15 || lby > 15 || s > 15 || sy > 15) return 0;
  return int32_t(0x80000000u | uint32_t(s) | uint32_t(sy) << 4 | uint32_t(s) << 8 |
                 uint32_t(lbx) << 12 | uint32_t(lby) << 16);
}

// One group of volumes with the same in_dims, already validated; chunks of
// kMaxVolPerLaunch (kTmaVolPerLaunch with TMA) volumes.  Volume i reads
// vols[i] (image: float32 if elem == 4, int16 if elem == 2; labels nullable)
// and writes output slot vols[i].slot of the uniform output batch out[].
struct VolIn {
  const void* img;
  const uint8_t* lbl;
  int32_t slot;
};

static w3d_status launch_group(int32_t batch, const VolIn* vols, int elem, w3d_dims in_dims,
                               const float* const* affines, const w3d_photometric* const* phs,
                               w3d_interp interp, float fill, uint8_t label_fill, float* out,
                               uint8_t* out_labels, w3d_dims out_dims, w3d_kernel variant,
                               cudaStream_t stream) {
  static thread_local WarpArgs args;  // ~31 KB: keep off the stack
  const int64_t in_n = nvox(in_dims), out_n = nvox(out_dims);
  static const bool no_tma = getenv("W3D_NO_TMA") && getenv("W3D_NO_TMA")[0] == '1';
  const bool want_tma = variant != W3D_KERNEL_GATHER && !no_tma;
  const int32_t chunk = want_tma ? kTmaVolPerLaunch : kMaxVolPerLaunch;
  const bool labels = vols[0].lbl != nullptr;
  const int id[3] = {in_dims.nx, in_dims.ny, in_dims.nz};
  const int od[3] = {out_dims.nx, out_dims.ny, out_dims.nz};
  // AUTO splits a batch by box size: the volumes whose 16-row box fits the staging
  // buffer first, then the others (their own launches: 8-row tiles),
  // so one large-footprint volume does not send a whole chunk to the slow paths.  Each
  // volume carries its own output slot, so the order is free.
  static thread_local std::vector<int32_t> order;
  static thread_local std::vector<VolDev> pre;  // per volume, derived once per call
  order.resize(static_cast<size_t>(batch));
  pre.resize(static_cast<size_t>(batch));
  for (int32_t i = 0; i < batch; ++i) {
    VolDev& P = pre[i];
    P = derive(affines[i], phs[i]);
    P.in_addr = reinterpret_cast<uint64_t>(vols[i].img);
    P.lbl_addr = reinterpret_cast<uint64_t>(vols[i].lbl);
    P.out_slot = vols[i].slot;
    cube_cp_box(affines[i], P, elem, id, od, kTileRows);
  }
  int32_t n16 = batch;
  if (variant == W3D_KERNEL_AUTO && interp == W3D_INTERP_LINEAR && want_tma) {
    int32_t lo = 0;
    static thread_local std::vector<int32_t> big;
    big.clear();
    for (int32_t i = 0; i < batch; ++i) {
      if (pre[i].cp_rows != 0)
        order[lo++] = i;
      else
        big.push_back(i);
    }
    for (int32_t i : big) order[lo++] = i;
    n16 = batch - static_cast<int32_t>(big.size());
  } else {
    for (int32_t i = 0; i < batch; ++i) order[i] = i;
  }
  // chunks never straddle the two classes
  auto next_chunk = [&](int32_t v0) {
    const int32_t end = v0 < n16 ? n16 : batch;
    return (end - v0 < chunk) ? end - v0 : chunk;
  };
  for (int32_t v0 = 0; v0 < batch; v0 += next_chunk(v0)) {
    const int32_t nv = next_chunk(v0);
    // type flags (the kernels read every address from vol[i])
    args.in = elem == 4 ? static_cast<const float*>(vols[order[v0]].img) : nullptr;
    args.in16 = elem == 2 ? static_cast<const int16_t*>(vols[order[v0]].img) : nullptr;
    {
      const float f = std::nearbyint(fill) == fill && fill >= -32768.0f && fill <= 32767.0f
                          ? fill
                          : 0.0f;
      const uint32_t h = static_cast<uint16_t>(static_cast<int16_t>(f));
      args.fill16_pair = h | (h << 16);
    }
    args.in_lbl = labels ? vols[order[v0]].lbl : nullptr;
    args.out = out;
    args.out_lbl = out_labels;
    args.nx = in_dims.nx; args.ny = in_dims.ny; args.nz = in_dims.nz;
    args.mx = out_dims.nx; args.my = out_dims.ny; args.mz = out_dims.nz;
    args.in_stride = in_n;
    args.out_stride = out_n;
    args.out_row_bytes = 4 * int64_t(out_dims.nx);
    args.out_lrow_bytes = out_dims.nx;
    args.fill = fill;
    args.label_fill = label_fill;
    args.interp = interp;
    args.nvol = nv;
    args.in_aligned = 1;
    for (int32_t i = 0; i < nv; ++i) {
      const VolDev& P = args.vol[i] = pre[order[v0 + i]];
      if (P.in_addr % 16 || P.lbl_addr % 8) args.in_aligned = 0;
    }
    // AUTO: when no volume's 16-row box fits the buffer (large rotations / scales),
    // 8-row tiles (half the box height) usually do: stage those by TMA rather than
    // gathering every corner through L1 (C4)
    args.tile_rows = kTileRows;
    if (variant == W3D_KERNEL_AUTO && interp == W3D_INTERP_LINEAR) {
      bool any16 = false, any8 = false;
      for (int32_t i = 0; i < nv; ++i) any16 |= args.vol[i].cp_rows != 0;
      static const int force8 = getenv("W3D_TILE_ROWS") ? atoi(getenv("W3D_TILE_ROWS")) : 0;
      if (force8 == kTileRowsSmall) any16 = false;  // A/B knob
      if (!any16) {
        for (int32_t i = 0; i < nv; ++i) {
          cube_cp_box(affines[order[v0 + i]], args.vol[i], elem, id, od, kTileRowsSmall);
          any8 |= args.vol[i].cp_rows != 0;
        }
        if (any8) {
          args.tile_rows = kTileRowsSmall;
        } else {  // neither fits: back to the 16-row offsets (the gather kernel's tile classes)
          for (int32_t i = 0; i < nv; ++i) {
            cube_cp_box(affines[order[v0 + i]], args.vol[i], elem, id, od, kTileRows);
          }
        }
      }
    }
    for (int r = 0; r < 10; ++r) {  // volume 0's key schedule (used when all seeds agree)
      args.rk0[r] = args.vol[0].rk0[r];
      args.rk1[r] = args.vol[0].rk1[r];
    }
    args.use_tma = 0;
    if (want_tma && cube_tma_supported(args))
      args.use_tma = prepare_tma(args) ? 1 : 0;
    // STAGED: the staged cube kernel (it gathers by itself when the layout
    // does not allow 16 B chunks); GATHER: every tile gathered.  AUTO: staged,
    // unless no volume of the chunk has a staging box that fits the buffer
    // (large rotations / scales): then its tiles would mostly go in y-parts,
    // and the gather kernel, which keeps the whole L1 (no staging carve-out),
    // is faster (C4: 138.0 vs 133.7 GVoxel/s)
    bool gather = variant == W3D_KERNEL_GATHER;
    if (variant == W3D_KERNEL_AUTO) {
      bool any_box = false;
      for (int32_t i = 0; i < nv; ++i) any_box |= args.vol[i].cp_rows != 0;
      gather = !any_box;
    }
    args.brick = brick_order(args, gather);
    {  // L2 prefetch one resident wave ahead (8-row launches; W3D_PREFETCH=<CTAs> overrides)
      static const int pf = getenv("W3D_PREFETCH") ? atoi(getenv("W3D_PREFETCH")) : -1;
      args.prefetch_ahead = pf >= 0 ? pf : 0;
    }
    args.pdl = v0 > 0 ? 1 : 0;  // the first chunk waits for all prior work on the stream
    const cudaError_t e = launch_cube(args, gather, stream);
    if (e != cudaSuccess) return cuda_fail(e, "warp3d kernel launch");
  }
  return ok();
}

// A uniform batch: volume i at in + i * nvox(in_dims), output slot i.
static w3d_status run_batched_t(int32_t batch, const void* in, int elem, const uint8_t* in_labels,
                                w3d_dims in_dims, const float* const* affines,
                                const w3d_photometric* const* phs, w3d_interp interp, float fill,
                                uint8_t label_fill, float* out, uint8_t* out_labels,
                                w3d_dims out_dims, w3d_kernel variant, cudaStream_t stream) {
  static thread_local std::vector<VolIn> vols;
  vols.resize(static_cast<size_t>(batch));
  const int64_t in_n = nvox(in_dims);
  for (int32_t i = 0; i < batch; ++i)
    vols[i] = VolIn{static_cast<const char*>(in) + i * in_n * elem,
                    in_labels ? in_labels + i * in_n : nullptr, i};
  return launch_group(batch, vols.data(), elem, in_dims, affines, phs, interp, fill, label_fill,
                      out, out_labels, out_dims, variant, stream);
}

static w3d_status run_batched(int32_t batch, const float* in, const uint8_t* in_labels,
                              w3d_dims in_dims, const float* const* affines,
                              const w3d_photometric* const* phs, w3d_interp interp, float fill,
                              uint8_t label_fill, float* out, uint8_t* out_labels,
                              w3d_dims out_dims, w3d_kernel variant, cudaStream_t stream) {
  return run_batched_t(batch, in, 4, in_labels, in_dims, affines, phs, interp, fill, label_fill,
                       out, out_labels, out_dims, variant, stream);
}

static w3d_status check_common(const void* in, w3d_dims in_dims, w3d_interp interp, float fill,
                               float* out, w3d_dims out_dims, int in_bytes = 4) {
  if (!in || !out) return fail(W3D_ERR_INVALID_ARG, "in/out must be non-NULL device pointers");
  if (reinterpret_cast<uintptr_t>(in) % in_bytes || reinterpret_cast<uintptr_t>(out) % 4)
    return fail(W3D_ERR_INVALID_ARG, "in/out must be aligned to their element size");
  w3d_status st = check_dims(in_dims, "in_dims");
  if (st != W3D_OK) return st;
  st = check_dims(out_dims, "out_dims");
  if (st != W3D_OK) return st;
  if (interp != W3D_INTERP_LINEAR && interp != W3D_INTERP_NEAREST)
    return fail(W3D_ERR_INVALID_ARG, "interp = %d is not a w3d_interp", int(interp));
  if (!std::isfinite(fill)) return fail(W3D_ERR_INVALID_ARG, "fill must be finite");
  return W3D_OK;
}

}  // namespace w3d

using namespace w3d;

extern "C" {

int warp3d_abi_version(void) { return WARP3D_ABI_VERSION; }

const char* warp3d_last_error(void) { return g_last_error.c_str(); }

uint64_t warp3d_launch_count(void) { return g_launches.load(); }

w3d_status warp3d_tile_stats(uint64_t out[4]) {
  if (!out) return fail(W3D_ERR_INVALID_ARG, "out must be non-NULL");
  unsigned long long v[4] = {0, 0, 0, 0};
  const cudaError_t e = read_cube_stats(v);
  if (e != cudaSuccess) return cuda_fail(e, "warp3d_tile_stats");
  for (int k = 0; k < 4; ++k) out[k] = v[k];
  return ok();
}

w3d_status warp3d_affine(const float* in, w3d_dims in_dims, const float affine[12],
                         w3d_interp interp, float fill, const w3d_photometric* ph, float* out,
                         w3d_dims out_dims, void* stream) {
  w3d_status st = check_common(in, in_dims, interp, fill, out, out_dims);
  if (st != W3D_OK) return st;
  if (!affine) return fail(W3D_ERR_INVALID_ARG, "affine must be a non-NULL host pointer");
  if ((st = check_affine(affine, 0)) != W3D_OK) return st;
  if (ph && (st = check_ph(*ph, 0)) != W3D_OK) return st;
  if (overlap(in, nvox(in_dims) * 4, out, nvox(out_dims) * 4))
    return fail(W3D_ERR_INVALID_ARG, "out overlaps in (in-place warps are not allowed)");
  const float* A = affine;
  return run_batched(1, in, nullptr, in_dims, &A, &ph, interp, fill, 0, out, nullptr, out_dims,
                     W3D_KERNEL_AUTO, static_cast<cudaStream_t>(stream));
}

static w3d_status batched_impl(int32_t batch, const float* in, const int16_t* in16,
                               const uint8_t* in_labels, w3d_dims in_dims,
                               const w3d_volume_params* params, w3d_interp interp, float fill,
                               uint8_t label_fill, float* out, uint8_t* out_labels,
                               w3d_dims out_dims, w3d_kernel variant, void* stream) {
  if (batch < 1) return fail(W3D_ERR_INVALID_ARG, "batch = %d must be >= 1", batch);
  const int eb = in16 ? 2 : 4;
  const void* inp = in16 ? static_cast<const void*>(in16) : static_cast<const void*>(in);
  w3d_status st = check_common(inp, in_dims, interp, fill, out, out_dims, eb);
  if (st != W3D_OK) return st;
  if (!params) return fail(W3D_ERR_INVALID_ARG, "params must be a non-NULL host array");
  if ((in_labels == nullptr) != (out_labels == nullptr))
    return fail(W3D_ERR_INVALID_ARG, "out_labels must be NULL iff in_labels is NULL");
  if (variant != W3D_KERNEL_AUTO && variant != W3D_KERNEL_GATHER && variant != W3D_KERNEL_STAGED)
    return fail(W3D_ERR_INVALID_ARG, "variant = %d is not a w3d_kernel", int(variant));
  for (int32_t i = 0; i < batch; ++i) {
    if ((st = check_affine(params[i].affine, i)) != W3D_OK) return st;
    if ((st = check_ph(params[i].ph, i)) != W3D_OK) return st;
  }
  const int64_t in_b = int64_t(batch) * nvox(in_dims), out_b = int64_t(batch) * nvox(out_dims);
  if (overlap(inp, in_b * eb, out, out_b * 4) || overlap(in_labels, in_b, out_labels, out_b) ||
      overlap(inp, in_b * eb, out_labels, out_b) || overlap(in_labels, in_b, out, out_b * 4) ||
      overlap(out, out_b * 4, out_labels, out_b))
    return fail(W3D_ERR_INVALID_ARG, "output buffers overlap inputs or each other");
  const int n = batch;
  static thread_local const float* A[1 << 16];
  static thread_local const w3d_photometric* P[1 << 16];
  for (int32_t v0 = 0; v0 < n; v0 += (1 << 16)) {
    const int32_t nv = (n - v0 < (1 << 16)) ? n - v0 : (1 << 16);
    for (int32_t i = 0; i < nv; ++i) {
      A[i] = params[v0 + i].affine;
      P[i] = &params[v0 + i].ph;
    }
    const void* base = in16 ? static_cast<const void*>(in16 + int64_t(v0) * nvox(in_dims))
                            : static_cast<const void*>(in + int64_t(v0) * nvox(in_dims));
    st = run_batched_t(nv, base, eb,
                       in_labels ? in_labels + int64_t(v0) * nvox(in_dims) : nullptr, in_dims, A,
                       P, interp, fill, label_fill, out + int64_t(v0) * nvox(out_dims),
                       out_labels ? out_labels + int64_t(v0) * nvox(out_dims) : nullptr, out_dims,
                       variant, static_cast<cudaStream_t>(stream));
    if (st != W3D_OK) return st;
  }
  return ok();
}

w3d_status warp3d_affine_batched_ex(int32_t batch, const float* in, const uint8_t* in_labels,
                                    w3d_dims in_dims, const w3d_volume_params* params,
                                    w3d_interp interp, float fill, uint8_t label_fill,
                                    float* out, uint8_t* out_labels, w3d_dims out_dims,
                                    w3d_kernel variant, void* stream) {
  return batched_impl(batch, in, nullptr, in_labels, in_dims, params, interp, fill, label_fill,
                      out, out_labels, out_dims, variant, stream);
}

w3d_status warp3d_affine_batched_i16_ex(int32_t batch, const int16_t* in, const uint8_t* in_labels,
                                        w3d_dims in_dims, const w3d_volume_params* params,
                                        w3d_interp interp, float fill, uint8_t label_fill,
                                        float* out, uint8_t* out_labels, w3d_dims out_dims,
                                        w3d_kernel variant, void* stream) {
  return batched_impl(batch, nullptr, in, in_labels, in_dims, params, interp, fill, label_fill,
                      out, out_labels, out_dims, variant, stream);
}

w3d_status warp3d_affine_batched_i16(int32_t batch, const int16_t* in, const uint8_t* in_labels,
                                     w3d_dims in_dims, const w3d_volume_params* params,
                                     w3d_interp interp, float fill, uint8_t label_fill, float* out,
                                     uint8_t* out_labels, w3d_dims out_dims, void* stream) {
  return batched_impl(batch, nullptr, in, in_labels, in_dims, params, interp, fill, label_fill,
                      out, out_labels, out_dims, W3D_KERNEL_AUTO, stream);
}

w3d_status warp3d_affine_batched(int32_t batch, const float* in, const uint8_t* in_labels,
                                 w3d_dims in_dims, const w3d_volume_params* params,
                                 w3d_interp interp, float fill, uint8_t label_fill, float* out,
                                 uint8_t* out_labels, w3d_dims out_dims, void* stream) {
  return warp3d_affine_batched_ex(batch, in, in_labels, in_dims, params, interp, fill, label_fill,
                                  out, out_labels, out_dims, W3D_KERNEL_AUTO, stream);
}

// Per-volume inputs of different dims (NEXT-4): volumes grouped by in_dims, one
// launch group per distinct dims, each volume writing its own slot of out[].
w3d_status warp3d_affine_batched_v(int32_t batch, w3d_in_type in_type, const void* const* in,
                                   const uint8_t* const* in_labels, const w3d_dims* in_dims,
                                   const w3d_volume_params* params, w3d_interp interp, float fill,
                                   uint8_t label_fill, float* out, uint8_t* out_labels,
                                   w3d_dims out_dims, void* stream) {
  if (batch < 1) return fail(W3D_ERR_INVALID_ARG, "batch = %d must be >= 1", batch);
  if (in_type != W3D_IN_F32 && in_type != W3D_IN_I16)
    return fail(W3D_ERR_INVALID_ARG, "in_type = %d is not a w3d_in_type", int(in_type));
  if (!in || !in_dims || !params)
    return fail(W3D_ERR_INVALID_ARG, "in, in_dims and params must be non-NULL host arrays");
  if ((in_labels == nullptr) != (out_labels == nullptr))
    return fail(W3D_ERR_INVALID_ARG, "out_labels must be NULL iff in_labels is NULL");
  const int eb = in_type == W3D_IN_I16 ? 2 : 4;
  const int64_t out_b = int64_t(batch) * nvox(out_dims);
  w3d_status st;
  for (int32_t i = 0; i < batch; ++i) {
    if ((st = check_common(in[i], in_dims[i], interp, fill, out, out_dims, eb)) != W3D_OK)
      return fail(st, "volume %d: %s", i, g_last_error.c_str());
    if (in_labels && !in_labels[i])
      return fail(W3D_ERR_INVALID_ARG, "in_labels[%d] is NULL", i);
    if ((st = check_affine(params[i].affine, i)) != W3D_OK) return st;
    if ((st = check_ph(params[i].ph, i)) != W3D_OK) return st;
    const int64_t n = nvox(in_dims[i]);
    if (overlap(in[i], n * eb, out, out_b * 4) ||
        (in_labels && (overlap(in_labels[i], n, out_labels, out_b) ||
                       overlap(in_labels[i], n, out, out_b * 4) ||
                       overlap(in[i], n * eb, out_labels, out_b))))
      return fail(W3D_ERR_INVALID_ARG, "volume %d: input overlaps the outputs", i);
  }
  if (out_labels && overlap(out, out_b * 4, out_labels, out_b))
    return fail(W3D_ERR_INVALID_ARG, "out and out_labels overlap");
  std::vector<int32_t> order(static_cast<size_t>(batch));
  for (int32_t i = 0; i < batch; ++i) order[i] = i;
  auto key = [&](int32_t i) {
    return std::make_tuple(in_dims[i].nz, in_dims[i].ny, in_dims[i].nx);
  };
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return key(a) < key(b); });
  std::vector<VolIn> vols;
  std::vector<const float*> A;
  std::vector<const w3d_photometric*> P;
  for (size_t g0 = 0; g0 < order.size();) {
    size_t g1 = g0;
    while (g1 < order.size() && key(order[g1]) == key(order[g0])) ++g1;
    vols.clear();
    A.clear();
    P.clear();
    for (size_t k = g0; k < g1; ++k) {
      const int32_t i = order[k];
      vols.push_back(VolIn{in[i], in_labels ? in_labels[i] : nullptr, i});
      A.push_back(params[i].affine);
      P.push_back(&params[i].ph);
    }
    st = launch_group(static_cast<int32_t>(g1 - g0), vols.data(), eb, in_dims[order[g0]],
                      A.data(), P.data(), interp, fill, label_fill, out, out_labels, out_dims,
                      W3D_KERNEL_AUTO, static_cast<cudaStream_t>(stream));
    if (st != W3D_OK) return st;
    g0 = g1;
  }
  return ok();
}

// A = F Rz Ry Rx Sh S G (R16), b = c_in + d - A c_out, double.
w3d_status warp3d_compose_affine(const w3d_geom* g, w3d_dims in_dims, w3d_dims out_dims,
                                 float affine_out[12]) {
  if (!g || !affine_out) return fail(W3D_ERR_INVALID_ARG, "g and affine_out must be non-NULL");
  w3d_status st = check_dims(in_dims, "in_dims");
  if (st != W3D_OK) return st;
  if ((st = check_dims(out_dims, "out_dims")) != W3D_OK) return st;
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(g->rot_rad[k]) || !std::isfinite(g->scale[k]) || !(g->scale[k] > 0) ||
        !std::isfinite(g->shear[k]) || !std::isfinite(g->disp[k]))
      return fail(W3D_ERR_INVALID_ARG, "geom: non-finite entry or scale <= 0 on axis %d", k);
  for (int k = 0; k < 9; ++k)
    if (!std::isfinite(g->generic[k])) return fail(W3D_ERR_INVALID_ARG, "geom: generic[%d]", k);
  struct M3 {
    double m[3][3];
  };
  auto mul = [](const M3& a, const M3& b) {
    M3 c;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        c.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
    return c;
  };
  const double cx = std::cos(g->rot_rad[0]), sx = std::sin(g->rot_rad[0]);
  const double cy = std::cos(g->rot_rad[1]), sy = std::sin(g->rot_rad[1]);
  const double cz = std::cos(g->rot_rad[2]), sz = std::sin(g->rot_rad[2]);
  const M3 F{{{g->flip[0] ? -1.0 : 1.0, 0, 0}, {0, g->flip[1] ? -1.0 : 1.0, 0},
              {0, 0, g->flip[2] ? -1.0 : 1.0}}};
  const M3 Rz{{{cz, -sz, 0}, {sz, cz, 0}, {0, 0, 1}}};
  const M3 Ry{{{cy, 0, sy}, {0, 1, 0}, {-sy, 0, cy}}};
  const M3 Rx{{{1, 0, 0}, {0, cx, -sx}, {0, sx, cx}}};
  const M3 Sh{{{1, g->shear[0], g->shear[1]}, {0, 1, g->shear[2]}, {0, 0, 1}}};
  const M3 S{{{g->scale[0], 0, 0}, {0, g->scale[1], 0}, {0, 0, g->scale[2]}}};
  M3 G;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) G.m[i][j] = g->generic[3 * i + j] + (i == j ? 1.0 : 0.0);
  const M3 A = mul(mul(mul(mul(mul(mul(F, Rz), Ry), Rx), Sh), S), G);
  const double n_in[3] = {double(in_dims.nx), double(in_dims.ny), double(in_dims.nz)};
  const double n_out[3] = {double(out_dims.nx), double(out_dims.ny), double(out_dims.nz)};
  for (int k = 0; k < 3; ++k) {
    double Ac = 0.0;
    for (int j = 0; j < 3; ++j) Ac += A.m[k][j] * 0.5 * (n_out[j] - 1.0);
    const double b = 0.5 * (n_in[k] - 1.0) + g->disp[k] - Ac;
    for (int j = 0; j < 3; ++j) affine_out[4 * k + j] = static_cast<float>(A.m[k][j]);
    affine_out[4 * k + 3] = static_cast<float>(b);
  }
  return ok();
}

w3d_status warp3d_compose_params_batched(int32_t n, const w3d_geom* geoms,
                                         const w3d_photometric* ph, w3d_dims in_dims,
                                         w3d_dims out_dims, w3d_volume_params* out) {
  if (n < 0 || (n > 0 && (!geoms || !ph || !out)))
    return fail(W3D_ERR_INVALID_ARG, "n >= 0 and non-NULL geoms / ph / out");
  for (int32_t i = 0; i < n; ++i) {
    w3d_status st = check_ph(ph[i], i);
    if (st != W3D_OK) return st;
    if ((st = warp3d_compose_affine(&geoms[i], in_dims, out_dims, out[i].affine)) != W3D_OK)
      return st;
    out[i].ph = ph[i];
  }
  return ok();
}

w3d_status warp3d_params_from_arrays(int32_t n, w3d_dims in_dims, w3d_dims out_dims,
                                     const double* rot, const double* scale, const double* shear,
                                     const uint8_t* flip, const double* disp,
                                     const double* generic, uint32_t flags,
                                     const double* window, const double* gamma, const double* sigma,
                                     uint64_t seed, const uint64_t* volume_ids,
                                     const double* occ_z0, const double* occ_height,
                                     w3d_volume_params* out) {
  if (n < 0 || (n > 0 && (!rot || !scale || !window || !gamma || !sigma || !out)))
    return fail(W3D_ERR_INVALID_ARG, "n >= 0 and non-NULL rot / scale / window / gamma / sigma / out");
  for (int32_t i = 0; i < n; ++i) {
    w3d_geom g;
    std::memset(&g, 0, sizeof(g));
    for (int k = 0; k < 3; ++k) {
      g.rot_rad[k] = rot[3 * i + k];
      g.scale[k] = scale[3 * i + k];
      g.shear[k] = shear ? shear[3 * i + k] : 0.0;
      g.flip[k] = flip ? (flip[3 * i + k] != 0) : 0;
      g.disp[k] = disp ? disp[3 * i + k] : 0.0;
    }
    if (generic)
      for (int k = 0; k < 9; ++k) g.generic[k] = generic[9 * i + k];
    w3d_photometric ph;
    std::memset(&ph, 0, sizeof(ph));
    const bool occ = occ_height && occ_height[i] >= 0.0;
    ph.flags = flags | (occ ? uint32_t(W3D_PH_OCCLUDE) : 0u);
    ph.window_lo = static_cast<float>(window[2 * i]);
    ph.window_hi = static_cast<float>(window[2 * i + 1]);
    ph.gamma = static_cast<float>(gamma[i]);
    ph.noise_sigma = static_cast<float>(sigma[i]);
    ph.seed = seed;
    ph.volume_id = volume_ids ? volume_ids[i] : uint64_t(i);
    ph.occ_z0 = occ_z0 ? static_cast<float>(occ_z0[i]) : 0.0f;
    ph.occ_height = occ ? static_cast<float>(occ_height[i]) : 0.0f;
    w3d_status st = check_ph(ph, i);
    if (st != W3D_OK) return st;
    if ((st = warp3d_compose_affine(&g, in_dims, out_dims, out[i].affine)) != W3D_OK) return st;
    out[i].ph = ph;
  }
  return ok();
}

// ---------------------------------------------------------------------------
// Resampling to r mm (NEXT-3; readings R22-R25)
// ---------------------------------------------------------------------------
static w3d_status check_spacing(const double* u, double r) {
  if (!u) return fail(W3D_ERR_INVALID_ARG, "spacing_mm must be a non-NULL host array[3]");
  for (int k = 0; k < 3; ++k)
    if (!(std::isfinite(u[k]) && u[k] > 0.0))
      return fail(W3D_ERR_INVALID_ARG, "spacing_mm[%d] = %g must be finite and > 0", k, u[k]);
  if (!(std::isfinite(r) && r > 0.0))
    return fail(W3D_ERR_INVALID_ARG, "target_mm = %g must be finite and > 0", r);
  return W3D_OK;
}

w3d_status warp3d_resample_sigma(const double spacing_mm[3], double target_mm,
                                 double sigma_out[3]) {
  w3d_status st = check_spacing(spacing_mm, target_mm);
  if (st != W3D_OK) return st;
  if (!sigma_out) return fail(W3D_ERR_INVALID_ARG, "sigma_out must be non-NULL");
  for (int k = 0; k < 3; ++k) sigma_out[k] = std::max(target_mm / spacing_mm[k] - 1.0, 0.0) / 3.0;
  return ok();
}

w3d_status warp3d_resample_dims(w3d_dims in_dims, const double spacing_mm[3], double target_mm,
                                w3d_dims* out_dims) {
  w3d_status st = check_spacing(spacing_mm, target_mm);
  if (st != W3D_OK) return st;
  if ((st = check_dims(in_dims, "in_dims")) != W3D_OK) return st;
  if (!out_dims) return fail(W3D_ERR_INVALID_ARG, "out_dims must be non-NULL");
  const int32_t n[3] = {in_dims.nx, in_dims.ny, in_dims.nz};
  int32_t m[3];
  for (int k = 0; k < 3; ++k) {
    const double v = std::floor(double(n[k]) * spacing_mm[k] / target_mm + 0.5);
    if (v >= double(kMaxDim)) return fail(W3D_ERR_UNSUPPORTED, "resampled dim %d too large", k);
    m[k] = v < 1.0 ? 1 : static_cast<int32_t>(v);
  }
  out_dims->nx = m[0];
  out_dims->ny = m[1];
  out_dims->nz = m[2];
  return ok();
}

// Centre-aligned scale map: A = diag(r/u), b = c_in - A c_out (double, one fp32 rounding).
w3d_status warp3d_resample_affine(w3d_dims in_dims, w3d_dims out_dims, const double spacing_mm[3],
                                  double target_mm, float affine_out[12]) {
  w3d_status st = check_spacing(spacing_mm, target_mm);
  if (st != W3D_OK) return st;
  if ((st = check_dims(in_dims, "in_dims")) != W3D_OK) return st;
  if ((st = check_dims(out_dims, "out_dims")) != W3D_OK) return st;
  if (!affine_out) return fail(W3D_ERR_INVALID_ARG, "affine_out must be non-NULL");
  const double n_in[3] = {double(in_dims.nx), double(in_dims.ny), double(in_dims.nz)};
  const double n_out[3] = {double(out_dims.nx), double(out_dims.ny), double(out_dims.nz)};
  for (int k = 0; k < 12; ++k) affine_out[k] = 0.0f;
  for (int k = 0; k < 3; ++k) {
    const double a = target_mm / spacing_mm[k];
    affine_out[4 * k + k] = static_cast<float>(a);
    affine_out[4 * k + 3] = static_cast<float>(0.5 * (n_in[k] - 1.0) - a * 0.5 * (n_out[k] - 1.0));
  }
  return ok();
}

// Separable passes over the axes with sigma > 0: in -> ... -> result; with an
// odd number of passes the first writes `out`, else `tmp`, so the last lands in
// `out` (0 passes: a copy).
static w3d_status smooth_passes(const float* in, w3d_dims d, const double sigma[3], float* out,
                                float* tmp, cudaStream_t s) {
  int axes[3], na = 0;
  for (int k = 0; k < 3; ++k)
    if (sigma[k] > 0.0) axes[na++] = k;
  if (na == 0) {
    const cudaError_t e = cudaMemcpyAsync(out, in, size_t(nvox(d)) * 4, cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? ok() : cuda_fail(e, "warp3d_smooth3d copy");
  }
  static const bool no_fuse = getenv("W3D_SMOOTH_PASSES") && getenv("W3D_SMOOTH_PASSES")[0] == '1';
  if (smooth_fusable(sigma) && !no_fuse) {
    const cudaError_t e = launch_smooth_fused(in, out, d.nx, d.ny, d.nz, sigma, s);
    return e == cudaSuccess ? ok() : cuda_fail(e, "warp3d_smooth3d launch");
  }
  const float* src = in;
  float* dst = (na % 2 == 1) ? out : tmp;
  for (int i = 0; i < na; ++i) {
    const cudaError_t e = launch_smooth_axis(axes[i], src, dst, d.nx, d.ny, d.nz, sigma[axes[i]], s);
    if (e != cudaSuccess) return cuda_fail(e, "warp3d_smooth3d launch");
    src = dst;
    dst = (dst == out) ? tmp : out;
  }
  return ok();
}

static w3d_status check_sigma(const double* sigma, w3d_dims d) {
  if (!sigma) return fail(W3D_ERR_INVALID_ARG, "sigma must be a non-NULL host array[3]");
  for (int k = 0; k < 3; ++k) {
    if (!(std::isfinite(sigma[k]) && sigma[k] >= 0.0))
      return fail(W3D_ERR_INVALID_ARG, "sigma[%d] = %g must be finite and >= 0", k, sigma[k]);
    if (2 * gauss_radius(sigma[k]) + 1 > kMaxTaps)
      return fail(W3D_ERR_UNSUPPORTED, "sigma[%d] = %g: more than %d taps", k, sigma[k], kMaxTaps);
  }
  if (d.ny > 65535 || d.nz > 65535)
    return fail(W3D_ERR_UNSUPPORTED, "smoothing needs ny, nz <= 65535");
  return W3D_OK;
}

w3d_status warp3d_smooth3d(const float* in, w3d_dims dims, const double sigma[3], float* out,
                           float* tmp, void* stream) {
  w3d_status st = check_dims(dims, "dims");
  if (st != W3D_OK) return st;
  if (!in || !out || !tmp) return fail(W3D_ERR_INVALID_ARG, "in/out/tmp must be non-NULL");
  if ((st = check_sigma(sigma, dims)) != W3D_OK) return st;
  const int64_t b = nvox(dims) * 4;
  if (overlap(in, b, out, b) || overlap(in, b, tmp, b) || overlap(out, b, tmp, b))
    return fail(W3D_ERR_INVALID_ARG, "in, out and tmp must not overlap");
  return smooth_passes(in, dims, sigma, out, tmp, static_cast<cudaStream_t>(stream));
}

w3d_status warp3d_resample(const float* in, const uint8_t* in_labels, w3d_dims in_dims,
                           const double spacing_mm[3], double target_mm, float fill,
                           uint8_t label_fill, float* out, uint8_t* out_labels,
                           w3d_dims out_dims, float* tmp, void* stream) {
  w3d_status st = check_common(in, in_dims, W3D_INTERP_LINEAR, fill, out, out_dims);
  if (st != W3D_OK) return st;
  if ((st = check_spacing(spacing_mm, target_mm)) != W3D_OK) return st;
  if ((in_labels == nullptr) != (out_labels == nullptr))
    return fail(W3D_ERR_INVALID_ARG, "out_labels must be NULL iff in_labels is NULL");
  if (!tmp) return fail(W3D_ERR_INVALID_ARG, "tmp (2 x in_dims floats) must be non-NULL");
  w3d_dims expect;
  if ((st = warp3d_resample_dims(in_dims, spacing_mm, target_mm, &expect)) != W3D_OK) return st;
  if (expect.nx != out_dims.nx || expect.ny != out_dims.ny || expect.nz != out_dims.nz)
    return fail(W3D_ERR_INVALID_ARG, "out_dims must be warp3d_resample_dims() = (%d, %d, %d)",
                expect.nx, expect.ny, expect.nz);
  double sigma[3];
  warp3d_resample_sigma(spacing_mm, target_mm, sigma);
  if ((st = check_sigma(sigma, in_dims)) != W3D_OK) return st;
  const int64_t bi = nvox(in_dims), bo = nvox(out_dims);
  if (overlap(tmp, 2 * bi * 4, in, bi * 4) || overlap(tmp, 2 * bi * 4, out, bo * 4) ||
      overlap(in, bi * 4, out, bo * 4) || overlap(in_labels, bi, out_labels, bo))
    return fail(W3D_ERR_INVALID_ARG, "buffers overlap");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  float A[12];
  warp3d_resample_affine(in_dims, out_dims, spacing_mm, target_mm, A);
  // smoothed image in tmp[0 .. bi) (scratch tmp[bi .. 2 bi)), never the labels
  const float* src = in;
  if (sigma[0] > 0.0 || sigma[1] > 0.0 || sigma[2] > 0.0) {
    // The interpolation reads the smoothed image only at the trilinear corners of the
    // output grid: p_k = fma(a_k, j, b_k) (R4 with a diagonal affine: the zero terms are
    // exact), corners floor(p_k) and floor(p_k) + 1.  With the fused lowpass only those
    // coordinates are computed and stored (the rest of tmp is left as it was); the
    // values that are computed are the full lowpass's, bit for bit.
    static const bool dense = getenv("W3D_RESAMPLE_DENSE") && getenv("W3D_RESAMPLE_DENSE")[0] == '1';
    const int nin[3] = {in_dims.nx, in_dims.ny, in_dims.nz};
    const int nout[3] = {out_dims.nx, out_dims.ny, out_dims.nz};
    const bool maskable = !dense && smooth_fusable(sigma) && nin[0] <= kSmoothMaskMax &&
                          nin[1] <= kSmoothMaskMax && nin[2] <= kSmoothMaskMax;
    if (maskable) {
      constexpr int kW = kSmoothMaskMax / 32;
      static thread_local uint32_t mask[3 * kW];
      std::memset(mask, 0, sizeof(mask));
      for (int k = 0; k < 3; ++k) {
        const float a = A[4 * k + k], b = A[4 * k + 3];
        for (int j = 0; j < nout[k]; ++j) {
          const float pk = std::fmaf(a, static_cast<float>(j), b);
          const double f = std::floor(static_cast<double>(pk));
          for (int c = 0; c < 2; ++c) {
            const double i = f + c;
            if (i >= 0.0 && i < nin[k]) {
              const int ii = static_cast<int>(i);
              mask[k * kW + (ii >> 5)] |= 1u << (ii & 31);
            }
          }
        }
      }
      const cudaError_t e =
          launch_smooth_fused(in, tmp, in_dims.nx, in_dims.ny, in_dims.nz, sigma, s, mask);
      if (e != cudaSuccess) return cuda_fail(e, "warp3d_resample lowpass");
    } else if ((st = smooth_passes(in, in_dims, sigma, tmp, tmp + bi, s)) != W3D_OK) {
      return st;
    }
    src = tmp;
  }
  const float* Ap = A;
  const w3d_photometric* none = nullptr;
  return run_batched(1, src, in_labels, in_dims, &Ap, &none, W3D_INTERP_LINEAR, fill, label_fill,
                     out, out_labels, out_dims, W3D_KERNEL_AUTO, s);
}

w3d_status warp3d_noise(float* out, w3d_dims dims, float sigma, uint64_t seed, uint64_t volume_id,
                        void* stream) {
  if (!out) return fail(W3D_ERR_INVALID_ARG, "out must be non-NULL");
  w3d_status st = check_dims(dims, "dims");
  if (st != W3D_OK) return st;
  if (!(std::isfinite(sigma) && sigma >= 0.0f))
    return fail(W3D_ERR_INVALID_ARG, "sigma must be finite and >= 0");
  const cudaError_t e = launch_noise(out, dims.nx, dims.ny, dims.nz, sigma, uint32_t(seed),
                                     uint32_t(seed >> 32), uint32_t(volume_id),
                                     uint32_t(volume_id >> 32), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "warp3d_noise launch");
  return ok();
}

w3d_status warp3d_philox4x32_10(const uint32_t* ctr, uint64_t key, uint32_t* out, int64_t n,
                                void* stream) {
  if (!ctr || !out) return fail(W3D_ERR_INVALID_ARG, "ctr/out must be non-NULL");
  if (n < 0) return fail(W3D_ERR_INVALID_ARG, "n must be >= 0");
  if (reinterpret_cast<uintptr_t>(ctr) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
    return fail(W3D_ERR_INVALID_ARG, "ctr/out must be 16-byte aligned");
  if (n == 0) return ok();
  if (overlap(ctr, n * 16, out, n * 16) && ctr != out)
    return fail(W3D_ERR_INVALID_ARG, "ctr and out partially overlap");
  const cudaError_t e = launch_philox(ctr, uint32_t(key), uint32_t(key >> 32), out, n,
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "warp3d_philox4x32_10 launch");
  return ok();
}

w3d_status warp3d_footprint_batched(int32_t batch, w3d_dims in_dims,
                                    const w3d_volume_params* params, w3d_dims out_dims,
                                    uint8_t* marks, unsigned long long* counts, void* stream) {
  if (batch < 1 || !params || !marks || !counts)
    return fail(W3D_ERR_INVALID_ARG, "footprint: batch >= 1 and non-NULL params/marks/counts");
  if (batch > kMaxVolPerLaunch)
    return fail(W3D_ERR_UNSUPPORTED, "footprint: batch <= %d", kMaxVolPerLaunch);
  w3d_status st = check_dims(in_dims, "in_dims");
  if (st != W3D_OK) return st;
  if ((st = check_dims(out_dims, "out_dims")) != W3D_OK) return st;
  for (int32_t i = 0; i < batch; ++i) {
    if ((st = check_affine(params[i].affine, i)) != W3D_OK) return st;
    if ((st = check_ph(params[i].ph, i)) != W3D_OK) return st;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  static thread_local WarpArgs args;
  std::memset(&args, 0, sizeof(args));
  args.nx = in_dims.nx; args.ny = in_dims.ny; args.nz = in_dims.nz;
  args.mx = out_dims.nx; args.my = out_dims.ny; args.mz = out_dims.nz;
  args.in_stride = nvox(in_dims);
  args.out_stride = nvox(out_dims);
  args.interp = W3D_INTERP_LINEAR;
  args.nvol = batch;
  for (int32_t i = 0; i < batch; ++i) args.vol[i] = derive(params[i].affine, &params[i].ph);
  const int64_t total = args.in_stride * batch;
  cudaError_t e = cudaMemsetAsync(marks, 0, size_t(total) * 2, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = launch_footprint(args, marks, s);
  if (e == cudaSuccess) e = launch_count_marks(marks, total, counts, s);
  if (e == cudaSuccess) e = launch_count_marks(marks + total, total, counts + 1, s);
  if (e != cudaSuccess) return cuda_fail(e, "warp3d_footprint_batched");
  return ok();
}

// ---------------------------------------------------------------------------
// FIFO pipeline
// ---------------------------------------------------------------------------
struct w3d_pipeline {
  int32_t depth = 0;
  w3d_dims in_dims{}, out_dims{};
  bool labels = false;
  void* mem = nullptr;                    // all slots, one allocation
  float* in_img[8] = {};
  uint8_t* in_lbl[8] = {};
  float* out_img[8] = {};
  uint8_t* out_lbl[8] = {};
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[8] = {}, ev_comp[8] = {}, ev_out[8] = {};
  cudaEvent_t ev_start = nullptr;
  bool chain = false;   // W3D_PIPE_CHAIN: calls ordered after the previous calls only
  int64_t seq = 0;      // jobs submitted so far (slot of job j = j % depth, across calls)
  int32_t vols = 1;     // volumes per job (one H2D / warp / D2H per job)
};

// Volumes per job when the caller leaves it to the library: jobs of at least
// kJobBytes of input (image + labels), at most 8 volumes.  Per-volume copies of a
// C3 volume (13 MB each way) reach 47.1 GB/s per direction on a B200 box with both
// directions busy, 4-volume copies 49.1, one 210 MB copy 49.9 (tools/pcie_probe.py);
// C3 end to end: 8.67 GVoxel/s in jobs of 1 volume, 9.18 of 2, 9.35 of 4, 9.46 of 8.
static int32_t auto_vols_per_job(size_t in_bytes_per_volume) {
  constexpr size_t kJobBytes = size_t(96) << 20;
  const size_t k = (kJobBytes + in_bytes_per_volume - 1) / std::max<size_t>(in_bytes_per_volume, 1);
  return static_cast<int32_t>(std::min<size_t>(8, std::max<size_t>(1, k)));
}

static void pipeline_free(w3d_pipeline* p) {
  if (!p) return;
  for (int i = 0; i < 8; ++i) {
    if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
    if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
    if (p->ev_out[i]) cudaEventDestroy(p->ev_out[i]);
  }
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  if (p->s_in) cudaStreamDestroy(p->s_in);
  if (p->s_comp) cudaStreamDestroy(p->s_comp);
  if (p->s_out) cudaStreamDestroy(p->s_out);
  if (p->mem) cudaFree(p->mem);
  delete p;
}

w3d_status warp3d_pipeline_create(int32_t depth, w3d_dims in_dims, w3d_dims out_dims,
                                  int32_t flags, w3d_pipeline** out) {
  return warp3d_pipeline_create_ex(depth, 0, in_dims, out_dims, flags, out);
}

w3d_status warp3d_pipeline_create_ex(int32_t depth, int32_t vols_per_job, w3d_dims in_dims,
                                     w3d_dims out_dims, int32_t flags, w3d_pipeline** out) {
  if (!out) return fail(W3D_ERR_INVALID_ARG, "out must be non-NULL");
  *out = nullptr;
  if (depth < 1 || depth > 8) return fail(W3D_ERR_INVALID_ARG, "depth = %d must be in [1, 8]", depth);
  if (vols_per_job < 0 || vols_per_job > kMaxVolPerLaunch)
    return fail(W3D_ERR_INVALID_ARG, "vols_per_job = %d must be in [0, %d]", vols_per_job,
                kMaxVolPerLaunch);
  w3d_status st = check_dims(in_dims, "in_dims");
  if (st != W3D_OK) return st;
  if ((st = check_dims(out_dims, "out_dims")) != W3D_OK) return st;
  if (flags & ~(W3D_PIPE_LABELS | W3D_PIPE_CHAIN))
    return fail(W3D_ERR_INVALID_ARG, "flags = %d: unknown bits", flags);
  w3d_pipeline* p = new w3d_pipeline;
  p->depth = depth;
  p->in_dims = in_dims;
  p->out_dims = out_dims;
  p->labels = (flags & W3D_PIPE_LABELS) != 0;
  p->chain = (flags & W3D_PIPE_CHAIN) != 0;
  p->vols = vols_per_job > 0
                ? vols_per_job
                : auto_vols_per_job(size_t(nvox(in_dims)) * (p->labels ? 5 : 4));
  auto round256 = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t k = size_t(p->vols);  // a slot holds one job's volumes, contiguous
  const size_t bi = round256(k * size_t(nvox(in_dims)) * 4);
  const size_t bo = round256(k * size_t(nvox(out_dims)) * 4);
  const size_t bli = p->labels ? round256(k * size_t(nvox(in_dims))) : 0;
  const size_t blo = p->labels ? round256(k * size_t(nvox(out_dims))) : 0;
  const size_t per = bi + bo + bli + blo;
  cudaError_t e = cudaMalloc(&p->mem, per * size_t(depth));
  if (e == cudaSuccess) {
    char* base = static_cast<char*>(p->mem);
    for (int i = 0; i < depth; ++i) {
      char* q = base + per * size_t(i);
      p->in_img[i] = reinterpret_cast<float*>(q);
      p->out_img[i] = reinterpret_cast<float*>(q + bi);
      if (p->labels) {
        p->in_lbl[i] = reinterpret_cast<uint8_t*>(q + bi + bo);
        p->out_lbl[i] = reinterpret_cast<uint8_t*>(q + bi + bo + bli);
      }
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming);
  for (int i = 0; i < depth && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_out[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    pipeline_free(p);
    return cuda_fail(e, "warp3d_pipeline_create");
  }
  *out = p;
  return ok();
}

w3d_status warp3d_pipeline_run(w3d_pipeline* p, int32_t batch, const float* in_host,
                               const uint8_t* in_labels_host, const w3d_volume_params* params,
                               w3d_interp interp, float fill, uint8_t label_fill,
                               float* out_host, uint8_t* out_labels_host, void* stream) {
  if (!p) return fail(W3D_ERR_INVALID_ARG, "pipeline must be non-NULL");
  if (batch < 1) return fail(W3D_ERR_INVALID_ARG, "batch = %d must be >= 1", batch);
  if (!in_host || !out_host || !params)
    return fail(W3D_ERR_INVALID_ARG, "in_host, out_host and params must be non-NULL");
  if ((in_labels_host == nullptr) != (out_labels_host == nullptr))
    return fail(W3D_ERR_INVALID_ARG, "out_labels_host must be NULL iff in_labels_host is NULL");
  if (in_labels_host && !p->labels)
    return fail(W3D_ERR_INVALID_ARG, "pipeline created without label buffers");
  if (interp != W3D_INTERP_LINEAR && interp != W3D_INTERP_NEAREST)
    return fail(W3D_ERR_INVALID_ARG, "interp = %d is not a w3d_interp", int(interp));
  if (!std::isfinite(fill)) return fail(W3D_ERR_INVALID_ARG, "fill must be finite");
  w3d_status st;
  for (int32_t i = 0; i < batch; ++i) {
    if ((st = check_affine(params[i].affine, i)) != W3D_OK) return st;
    if ((st = check_ph(params[i].ph, i)) != W3D_OK) return st;
  }
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  const size_t ni = size_t(nvox(p->in_dims)), no = size_t(nvox(p->out_dims));
  const bool lab = in_labels_host != nullptr;
  cudaError_t e = cudaSuccess;
  if (!p->chain || p->seq == 0) {  // after the work already queued on `stream`
    e = cudaEventRecord(p->ev_start, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_in, p->ev_start, 0);
  }
  int64_t j = p->seq;  // job number across calls
  for (int32_t i = 0; i < batch && e == cudaSuccess; i += p->vols, ++j) {
    const int32_t kk = std::min(p->vols, batch - i);  // volumes i .. i + kk - 1
    const int s = static_cast<int>(j % p->depth);
    if (j >= p->depth) e = cudaStreamWaitEvent(p->s_in, p->ev_out[s], 0);  // slot free again
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->in_img[s], in_host + ni * size_t(i), ni * 4 * size_t(kk),
                          cudaMemcpyHostToDevice, p->s_in);
    if (e == cudaSuccess && lab)
      e = cudaMemcpyAsync(p->in_lbl[s], in_labels_host + ni * size_t(i), ni * size_t(kk),
                          cudaMemcpyHostToDevice, p->s_in);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_in[s], p->s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, p->ev_in[s], 0);
    if (e != cudaSuccess) break;
    st = warp3d_affine_batched(kk, p->in_img[s], lab ? p->in_lbl[s] : nullptr, p->in_dims,
                               params + i, interp, fill, label_fill, p->out_img[s],
                               lab ? p->out_lbl[s] : nullptr, p->out_dims, p->s_comp);
    if (st != W3D_OK) return st;
    e = cudaEventRecord(p->ev_comp[s], p->s_comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_out, p->ev_comp[s], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out_host + no * size_t(i), p->out_img[s], no * 4 * size_t(kk),
                          cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess && lab)
      e = cudaMemcpyAsync(out_labels_host + no * size_t(i), p->out_lbl[s], no * size_t(kk),
                          cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[s], p->s_out);
  }
  if (e == cudaSuccess) e = cudaStreamWaitEvent(user, p->ev_out[(j - 1) % p->depth], 0);
  p->seq = j;
  if (e != cudaSuccess) return cuda_fail(e, "warp3d_pipeline_run");
  return ok();
}

int32_t warp3d_pipeline_vols_per_job(const w3d_pipeline* p) { return p ? p->vols : 0; }

w3d_status warp3d_pipeline_destroy(w3d_pipeline* p) {
  if (!p) return ok();
  cudaStreamSynchronize(p->s_in);
  cudaStreamSynchronize(p->s_comp);
  cudaStreamSynchronize(p->s_out);
  pipeline_free(p);
  return ok();
}

}  // extern "C"
