// K2-K7: damping + block inverses, the fused power-series term, the camera
// reduction / U^-1 / stop test, back-substitution and the operator passes.
//
// Reference (paths relative to /root/reference/pkg/src/powerba/):
//   DampedSystem.__init__      blocks.py:164-192, _spd_block_inverse blocks.py:277-285
//   apply_w / apply_wt         blocks.py:214-236
//   apply_u_inv / apply_v_inv  blocks.py:238-246, apply_u / apply_schur 248-254
//   b_tilde                    blocks.py:256-260
//   series_terms / power_series_solve / stop_criterion  power_series.py:29-77
//   apply_series_inverse       power_series.py:80-91
//   back_substitute            power_series.py:94-100
//
// One series term is ONE pass over the observation store: per landmark tile
// the kernel computes y_l = sum_o J_l^T (J_p t_c), z_l = V_l^-1 y_l and, with
// the Jacobians still in registers, g_o = J_p^T (J_l z_l); the per-camera sum
// of g_o is reduced in shared memory into chunk-local camera slots in a fixed
// order and written once per (chunk, camera).  A second, small kernel merges
// the chunk partials per camera (fixed order), applies U^-1, accumulates the
// partial sum x and evaluates the stop test on the device.
#include <algorithm>
#include <limits>
#include <vector>

#include "poba_internal.h"

namespace poba {

namespace {

enum TermMode { kModeTerm = 0, kModeBt = 1, kModeW = 2 };
enum CamMode { kCamMerge = 0, kCamTerm = 1, kCamBt = 2 };
enum WtOut { kOutWt = 0, kOutZ = 1, kOutBack = 2 };

__device__ __forceinline__ int pk9(int i, int j) {  // packed upper-triangle index, i <= j
  return i * 9 - i * (i - 1) / 2 + (j - i);
}
__device__ __forceinline__ int sym9(int i, int j) { return i <= j ? pk9(i, j) : pk9(j, i); }

// z = V y with V packed [00,01,02,11,12,22]
__device__ __forceinline__ void sym3_mv(const double* __restrict__ V, const double y[3], double z[3]) {
  const double v00 = V[0], v01 = V[1], v02 = V[2], v11 = V[3], v12 = V[4], v22 = V[5];
  z[0] = v00 * y[0] + v01 * y[1] + v02 * y[2];
  z[1] = v01 * y[0] + v11 * y[1] + v12 * y[2];
  z[2] = v02 * y[0] + v12 * y[1] + v22 * y[2];
}

// ---------------------------------------------------------------------------
// damping + Cholesky inverses
// ---------------------------------------------------------------------------

__global__ void k_damp_u(const double* __restrict__ U0, const double* __restrict__ Dp, int64_t n_cam,
                         double lam, int identity, double* __restrict__ Ud, double* __restrict__ Uinv,
                         int* __restrict__ fail_flag) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cam) return;
  double U[45];
#pragma unroll
  for (int q = 0; q < 45; ++q) U[q] = U0[c * 45 + q];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double d = identity ? 1.0 : Dp[c * 9 + i];
    U[pk9(i, i)] += lam * (d * d);
  }
#pragma unroll
  for (int q = 0; q < 45; ++q) Ud[c * 45 + q] = U[q];
  // Cholesky U = L L^T (lower, stored row-major packed by rows i>=j into L[i*(i+1)/2 + j])
  double L[45];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    double d = U[pk9(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
    if (!(d > 0.0)) ok = false;
    const double ljj = sqrt(d);
    L[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
    for (int i = j + 1; i < 9; ++i) {
      double v = U[pk9(j, i)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
      L[i * (i + 1) / 2 + j] = v / ljj;
    }
  }
  if (!ok) {
    atomicOr(fail_flag, 1);
    return;
  }
  // L^-1 (lower)
  double Li[45];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    Li[i * (i + 1) / 2 + i] = 1.0 / L[i * (i + 1) / 2 + i];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double v = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) v += L[i * (i + 1) / 2 + k] * Li[k * (k + 1) / 2 + j];
      Li[i * (i + 1) / 2 + j] = -v / L[i * (i + 1) / 2 + i];
    }
  }
  // U^-1 = L^-T L^-1 :  (i,j) = sum_{k >= max(i,j)} Li[k][i] Li[k][j]
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) {
      double v = 0.0;
#pragma unroll
      for (int k = j; k < 9; ++k) v += Li[k * (k + 1) / 2 + i] * Li[k * (k + 1) / 2 + j];
      Uinv[c * 45 + pk9(i, j)] = v;
    }
}

__global__ void k_damp_v(const double* __restrict__ V0, const double* __restrict__ Dl, int64_t n_lm, double lam,
                         int identity, double* __restrict__ Vd, double* __restrict__ Vinv,
                         int* __restrict__ fail_flag) {
  int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= n_lm) return;
  double a[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) a[q] = V0[l * 6 + q];
  const int dg[3] = {0, 3, 5};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double d = identity ? 1.0 : Dl[l * 3 + i];
    a[dg[i]] += lam * (d * d);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) Vd[l * 6 + q] = a[q];
  // Cholesky of [[a0,a1,a2],[a1,a3,a4],[a2,a4,a5]]
  const double d0 = a[0];
  const double l00 = sqrt(d0);
  const double l10 = a[1] / l00, l20 = a[2] / l00;
  const double d1 = a[3] - l10 * l10;
  const double l11 = sqrt(d1);
  const double l21 = (a[4] - l20 * l10) / l11;
  const double d2 = a[5] - l20 * l20 - l21 * l21;
  const double l22 = sqrt(d2);
  if (!(d0 > 0.0) || !(d1 > 0.0) || !(d2 > 0.0)) {
    atomicOr(fail_flag, 2);
    return;
  }
  const double i00 = 1.0 / l00, i11 = 1.0 / l11, i22 = 1.0 / l22;
  const double i10 = -(l10 * i00) / l11;
  const double i21 = -(l21 * i11) / l22;
  const double i20 = -(l20 * i00 + l21 * i10) / l22;
  double* o = Vinv + l * 6;
  o[0] = i00 * i00 + i10 * i10 + i20 * i20;
  o[1] = i10 * i11 + i20 * i21;
  o[2] = i20 * i22;
  o[3] = i11 * i11 + i21 * i21;
  o[4] = i21 * i22;
  o[5] = i22 * i22;
}

// ---------------------------------------------------------------------------
// the fused term kernel: bulk-copy (TMA) pipeline over tiles, one CTA per SM
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// consumer release: this thread's prior shared-memory reads are ordered before
// the arrival (mbarrier.arrive has release semantics)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// streamed-once data: evict-first in L2 so the chunk accumulators stay resident
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// named barriers 1..kTermWarps pass the apply turn between consecutive warps
// (64 threads: the arriving warp and the waiting warp)
__device__ __forceinline__ void turn_pass(int to_warp) {
  asm volatile("bar.arrive %0, 64;" ::"r"(1 + to_warp) : "memory");
}
__device__ __forceinline__ void turn_wait(int warp) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + warp) : "memory");
}

struct TermArgs {
  const TileK* tk;         // per warp-tile kernel descriptors
  const int2* cta_tiles;   // tile range of each CTA
  const int* cam_s;        // camera of each slot (gathered two tiles ahead; unused with kChunkT)
  const int* part_cam;     // camera of each partial = of each chunk slot (kChunkT: fills the chunk's term-record table)
  const void* J;           // slot rows (double2, or float2 at precision 32)
  const double* tin;       // camera vector (kModeTerm)
  const double* lvec;      // b_l (kModeBt) or landmark input (kModeW)
  const double* Vinv;
  const double* zlong;     // landmark-indexed z of long landmarks (kModeTerm)
  double* partials;
  const SeriesState* st;
  int check_stop;
  int n_cam, n_partials, n_lm;  // bounds for the checked build (POBA_DEVICE_CHECKS)
};

// One CTA per SM streams a contiguous range of warp-tiles; warp w of the CTA
// takes tiles range.x + w, + w + kTermWarps, ... through its own one-stage bulk-copy
// pipeline (the stage is released as soon as the tile's rows are in
// registers, so the next tile's copy overlaps the whole tile's math).
//   phase 1  u_o = J_p t_c, with t_c either from the warp's gathered camera
//            records (CT = false: five lanes per 80-B record, 16-B loads, one
//            tile ahead) or read by slot from the chunk's term-record table
//            (CT = true: loaded by all warps at the chunk's first round,
//            between two CTA barriers); see TermShape in poba_internal.h,
//            w_o = J_l^T u_o, landmark sums y_l by a segmented warp scan
//   phase 2  z_l = V_l^-1 y_l on each landmark's last lane, shuffled back
//   phase 3  g_o = J_p^T (J_l z_l), nine doubles in registers
//   apply    g_o is added into the CTA's shared-memory accumulator record of
//            its camera slot.  Tiles apply strictly in tile order: the turn
//            is passed from warp to warp through named barriers (arrive /
//            sync pairs, no memory fences), so every camera sum is formed
//            in one fixed order -- no atomics, bitwise reproducible.  A warp
//            holds its tile's g_o in registers and applies it only after it
//            has computed its NEXT tile, so the turn's round trip overlaps a
//            whole tile of math.  A camera seen twice in one tile is
//            pre-summed in lane order; each distinct camera's contribution is
//            then shuffled to its apply lane (host-planned per tile so that the
//            slots of an eight-lane quarter differ mod 8: no bank replays).
// After the last tile of a chunk its warp writes the table out once (one 80-B
// partial per (chunk, camera)) and clears it before passing the turn on.
template <int MODE, bool F32, bool CT>
__global__ void __launch_bounds__(TermShape<CT>::kWarps * 32, kTermCtas) k_term(const TermArgs a) {
  constexpr int kTermWarps = TermShape<CT>::kWarps;  // (shadows the gather layout's global constant)
  constexpr int kTermCtl = TermShape<CT>::kCtl;
  constexpr int kWarpSmem = TermShape<CT>::kWarpSmem;
  constexpr int kAccSlots = TermShape<CT>::kAccSlots;
  constexpr bool kChunkT = CT;
  extern __shared__ __align__(128) uint8_t smraw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (a.check_stop && a.st->stopped) return;
  const int2 range = a.cta_tiles[blockIdx.x];
  uint8_t* ctl = smraw + kTermWarps * kWarpSmem;
  uint64_t* stage_bar = reinterpret_cast<uint64_t*>(ctl);  // [kTermWarps] full (copy landed)
  uint64_t* free_bar = stage_bar + kTermWarps;             // [kTermWarps] empty (all lanes read it)
  double2* acc = reinterpret_cast<double2*>(ctl + kTermCtl);                              // [kAccSlots][5]
  double2* ttc = acc + kAccSlots * 5;  // kChunkT: [kAccSlots][5] term records of the current chunk's cameras
  for (int k = threadIdx.x; k < kAccSlots * 5; k += blockDim.x) acc[k] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int w = 0; w < kTermWarps; ++w) {
      mbar_init(&stage_bar[w], 1);
      mbar_init(&free_bar[w], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int t_first = range.x + wid;
  if (t_first >= range.y) return;
  const int nq = (range.y - t_first + kTermWarps - 1) / kTermWarps;
  uint8_t* stg = smraw + wid * kWarpSmem;
  double2* ttab = reinterpret_cast<double2*>(stg + kStageBytes);  // [32 observations][5] camera records (!kChunkT)
  constexpr bool kGather = MODE == kModeTerm && !kChunkT;  // per-tile record gather
  constexpr bool kTable = MODE == kModeTerm && kChunkT;    // per-chunk record table
  int cur_part0 = -1;
  uint64_t* sbar = &stage_bar[wid];
  uint64_t* fbar = &free_bar[wid];
  const uint64_t pol = policy_evict_first();

  auto issue = [&](int ti, int n, int nlm, int lm0) {  // lane 0
    const uint32_t vbytes = (MODE != kModeW) ? (uint32_t)(nlm * 48) : 0u;
    const uint32_t rbytes = tile_copy_bytes<F32>(n);  // metadata + planes up to plane 11's last slot
    const char* src = static_cast<const char*>(a.J) + (int64_t)ti * tile_block_bytes<F32>();
    mbar_expect_tx(sbar, rbytes + 32u + vbytes);
    bulk_g2s_stream(stg, src, rbytes, sbar, pol);
    bulk_g2s(stg + kStDesc, a.tk + ti, 32, sbar);
    if (vbytes) bulk_g2s(stg + kStVinv, a.Vinv + (int64_t)lm0 * 6, vbytes, sbar);
  };
  auto gather = [&](int cam_lane, double2* tp) {  // 5 x 16-B pieces of the tile's 32 camera records
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int k = 32 * r + lane;
      const int cam = __shfl_sync(0xffffffffu, cam_lane, k / 5);
      POBA_DCHECK(cam >= 0 && cam < a.n_cam);
      tp[r] = reinterpret_cast<const double2*>(a.tin + (int64_t)cam * kTStride)[k % 5];
    }
  };
  if (lane == 0) {
    const int4 d = *reinterpret_cast<const int4*>(a.tk + t_first);
    issue(t_first, d.x, d.z, d.y);
  }
  double2 tp[5];  // camera-record pieces of the next tile, in flight (five lanes per 80-B record)
  int cam_next = 0;
  if (kGather) {
    gather(a.cam_s[(int64_t)t_first * kTile + lane], tp);
#pragma unroll
    for (int r = 0; r < 5; ++r) ttab[32 * r + lane] = tp[r];
    if (nq > 1) cam_next = a.cam_s[(int64_t)(t_first + kTermWarps) * kTile + lane];
  }
  __syncwarp();

  // the previous tile's contributions, applied after this tile's math
  double hg[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int h_slot = 0, h_ti = -1, h_flags = 0, h_part0 = 0, h_nslot = 0;
  bool h_apply = false;
  auto rmw = [&](int sl, const double* v) {
    POBA_DCHECK(sl >= 0 && sl < kAccSlots);
    double2* r = acc + sl * 5;
    const double2 o0 = r[0], o1 = r[1], o2 = r[2], o3 = r[3], o4 = r[4];
    r[0] = make_double2(o0.x + v[0], o0.y + v[1]);
    r[1] = make_double2(o1.x + v[2], o1.y + v[3]);
    r[2] = make_double2(o2.x + v[4], o2.y + v[5]);
    r[3] = make_double2(o3.x + v[6], o3.y + v[7]);
    r[4] = make_double2(o4.x + v[8], o4.y);
  };
  auto apply_held = [&]() {
    if (h_ti != range.x) turn_wait(wid);
    if (h_apply) rmw(h_slot, hg);
    __syncwarp();
    if (h_flags & kTileChunkLast) {  // write the chunk's partials, clear the table
      POBA_DCHECK(h_part0 >= 0 && h_nslot <= kAccSlots && h_part0 + h_nslot <= a.n_partials);
      double2* out = reinterpret_cast<double2*>(a.partials) + (int64_t)h_part0 * 5;
      for (int k = lane; k < h_nslot * 5; k += 32) {
        out[k] = acc[k];
        acc[k] = make_double2(0.0, 0.0);
      }
      __syncwarp();
    }
    if (h_ti + 1 < range.y) turn_pass((wid + 1) % kTermWarps);
  };

  for (int q = 0; q < nq; ++q) {
    const int ti = t_first + q * kTermWarps;
    mbar_wait(sbar, (uint32_t)(q & 1));
    const TileK t = *reinterpret_cast<const TileK*>(stg + kStDesc);
    if (kTable && t.part0 != cur_part0) {
      // first round of a chunk (chunks start at rounds, so every warp that has
      // a tile in this round is here): once all of them are past their reads
      // of the previous chunk's records, they load the new chunk's together
      const int nact = min(kTermWarps, range.y - range.x - q * kTermWarps);
      asm volatile("bar.sync 15, %0;" ::"r"(nact * 32) : "memory");
      for (int k = wid * 32 + lane; k < t.nslot * 5; k += nact * 32) {
        const int cam = a.part_cam[t.part0 + k / 5];
        POBA_DCHECK(cam < a.n_cam);
        ttc[k] = cam >= 0 ? __ldg(reinterpret_cast<const double2*>(a.tin + (int64_t)cam * kTStride) + k % 5)
                          : make_double2(0.0, 0.0);
      }
      asm volatile("bar.sync 15, %0;" ::"r"(nact * 32) : "memory");
      cur_part0 = t.part0;
    }
    const bool valid = lane < t.n;
    const bool is_long = t.flags & kTileLong;
    int slot = 0, li = 0, first = lane, last = lane;
    // the tile's metadata word of this lane (padding lanes carry an apply lane too)
    const uint32_t mv = reinterpret_cast<const uint32_t*>(stg)[lane];
    if (valid) {  // slot, landmark run
      slot = meta_slot(mv);
      li = meta_li(mv);
      POBA_DCHECK(slot < t.nslot && li < kTileLm && t.lm0 + li < a.n_lm);
      first = meta_first(mv);
      last = meta_last(mv);
    }
    const bool is_last = valid && lane == last;
    double vi[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (MODE != kModeW && is_last && !(MODE == kModeTerm && is_long)) {
      const double2* vs = reinterpret_cast<const double2*>(stg + kStVinv) + li * 3;
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const double2 v = vs[p];
        vi[2 * p] = v.x;
        vi[2 * p + 1] = v.y;
      }
    }
    // Lanes past the tile's end read stale stage entries: harmless, since
    // they are never a landmark's last lane, the segmented scan only pulls
    // from lower lanes, and they apply nothing (no select needed).
    double2 jr[kJPlanes];
#pragma unroll
    for (int p = 0; p < kJPlanes; ++p) {
      if (F32) {
        const float2 v = reinterpret_cast<const float2*>(stg + kMetaBytes)[p * kTile + lane];
        jr[p] = make_double2((double)v.x, (double)v.y);
      } else {
        jr[p] = reinterpret_cast<const double2*>(stg + kMetaBytes)[p * kTile + lane];
      }
    }
    // Refill the stage with this warp's next tile.  The bulk copy writes
    // through the async proxy, which is not ordered behind the lanes' generic
    // shared-memory reads of the stage by __syncwarp alone (with the rows
    // L2-resident the copy could land before reads still queued in the LSU).
    // The warp barrier orders every lane's reads before lane 0's arrival on
    // the warp's empty barrier (mbarrier.arrive: release), and lane 0
    // acquires that phase (try_wait: acquire) before it issues the copy -- the
    // consumer-release / producer-acquire pattern of a TMA pipeline, without
    // a full memory barrier.
    __syncwarp();
    if (lane == 0) mbar_arrive(fbar);
    // the next tile's camera records, in flight during this tile's math
    if (kGather && q + 1 < nq) {
      gather(cam_next, tp);
      cam_next = (q + 2 < nq) ? a.cam_s[(int64_t)(ti + 2 * kTermWarps) * kTile + lane] : 0;
    }
    // phase 1: this lane's camera record from the warp's record table (filled
    // at the end of the previous tile)
    double tc[10];
    if (MODE == kModeTerm) {
      const double2* rec = kChunkT ? ttc + slot * 5 : ttab + lane * 5;
#pragma unroll
      for (int p = 0; p < 5; ++p) {
        const double2 v = rec[p];
        tc[2 * p] = v.x;
        tc[2 * p + 1] = v.y;
      }
    }
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    if (MODE == kModeTerm && valid && !is_long) {
      double u0 = 0.0, u1 = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        u0 = fma(jr[j].x, tc[j], u0);
        u1 = fma(jr[j].y, tc[j], u1);
      }
      w0 = fma(jr[9].x, u0, jr[9].y * u1);
      w1 = fma(jr[10].x, u0, jr[10].y * u1);
      w2 = fma(jr[11].x, u0, jr[11].y * u1);
    }
    // lane 0 acquires the released stage and issues the refill here, a few
    // instructions after the arrivals, so the phase has usually completed and
    // the wait does not stall the warp
    if (lane == 0 && q + 1 < nq) {
      mbar_wait(fbar, (uint32_t)(q & 1));
      issue(ti + kTermWarps, t.nx_n & 0xff, t.nx_n >> 8, t.nx_lm0);
    }
    if (MODE == kModeTerm) {
      const int steps = (t.flags >> kTileScanShift) & 7;  // ceil(log2(longest landmark run of the tile))
#pragma unroll
      for (int i = 0, d = 1; i < 5; ++i, d <<= 1) {
        if (i >= steps) break;
        const double o0 = __shfl_up_sync(0xffffffffu, w0, d);
        const double o1 = __shfl_up_sync(0xffffffffu, w1, d);
        const double o2 = __shfl_up_sync(0xffffffffu, w2, d);
        if (lane - d >= first) {
          w0 += o0;
          w1 += o1;
          w2 += o2;
        }
      }
    }
    // phase 2
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    if (is_last) {
      const int lm = t.lm0 + li;
      if (MODE == kModeW) {
        z0 = a.lvec[lm * 3]; z1 = a.lvec[lm * 3 + 1]; z2 = a.lvec[lm * 3 + 2];
      } else if (MODE == kModeTerm && is_long) {
        z0 = a.zlong[lm * 3]; z1 = a.zlong[lm * 3 + 1]; z2 = a.zlong[lm * 3 + 2];
      } else {
        double y[3], z[3];
        if (MODE == kModeBt) {
          y[0] = a.lvec[lm * 3]; y[1] = a.lvec[lm * 3 + 1]; y[2] = a.lvec[lm * 3 + 2];
        } else {
          y[0] = w0; y[1] = w1; y[2] = w2;
        }
        sym3_mv(vi, y, z);
        z0 = z[0]; z1 = z[1]; z2 = z[2];
      }
    }
    const int src = valid ? last : lane;
    z0 = __shfl_sync(0xffffffffu, z0, src);
    z1 = __shfl_sync(0xffffffffu, z1, src);
    z2 = __shfl_sync(0xffffffffu, z2, src);
    // phase 3
    double g[9];
    {
      const double v0 = fma(jr[9].x, z0, fma(jr[10].x, z1, jr[11].x * z2));
      const double v1 = fma(jr[9].y, z0, fma(jr[10].y, z1, jr[11].y * z2));
#pragma unroll
      for (int j = 0; j < 9; ++j) g[j] = fma(jr[j].x, v0, jr[j].y * v1);
    }
    bool apply = valid;
    if (t.flags & kTileDupCam) {  // cameras seen twice in this tile: pre-sum on the lowest lane, lane order
      const unsigned grp = __match_any_sync(0xffffffffu, valid ? slot : -1 - lane);
      const int leader = __ffs(grp) - 1;
      unsigned pend = (valid && lane == leader) ? (grp & ~(1u << lane)) : 0u;
      apply = valid && lane == leader;
      while (__any_sync(0xffffffffu, pend != 0u)) {
        const int from = pend ? __ffs(pend) - 1 : lane;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          const double v = __shfl_sync(0xffffffffu, g[j], from);
          if (pend) g[j] += v;
        }
        pend &= pend - 1u;
      }
    }
    if (q > 0) apply_held();
    // hand each distinct camera's contribution to its apply lane (host-planned
    // permutation: the slots of a quarter differ mod 8, so the 16-B accumulator
    // accesses of a quarter do not collide); shuffles instead of bank replays
    {
      const int from = meta_apply_src(mv);
#pragma unroll
      for (int j = 0; j < 9; ++j) hg[j] = __shfl_sync(0xffffffffu, g[j], from);
      h_slot = __shfl_sync(0xffffffffu, slot, from);
      h_apply = meta_apply_on(mv);
#ifdef POBA_DEVICE_CHECKS
      const int src_applies = __shfl_sync(0xffffffffu, (int)apply, from);  // every lane takes part
      POBA_DCHECK(!h_apply || src_applies);
#endif
    }
    h_ti = ti;
    h_flags = t.flags;
    h_part0 = t.part0;
    h_nslot = t.nslot;
    if (kGather && q + 1 < nq) {
#pragma unroll
      for (int r = 0; r < 5; ++r) ttab[32 * r + lane] = tp[r];
    }
    __syncwarp();
  }
  apply_held();
}

// ---------------------------------------------------------------------------
// camera side: merge chunk partials, U^-1, partial sums, stop test
// ---------------------------------------------------------------------------

struct CamArgs {
  const int* part_cam_off;
  const int* part_idx;
  const double* partials;
  const double* rin;      // reduced vector when not merging
  double* rout;           // kCamMerge output
  const double* Uinv;
  const double* bp;
  double* bt;
  double* tvec;
  double* xvec;
  double* blk;            // per-block [dd, xx, nonfinite, nonzero]
  SeriesState* st;
  double* ratios;
  int n_cam;
  int order;
  double eps;
  int check_stop;
  // sliced camera step (sharded contexts): this rank's cameras [c0, c1), the
  // R received slices (ls cameras x 9 each) of the ranks' partial sums
  const double* recv;
  int nranks, ls, c0, c1;
};

enum CamSrc { kSrcPartials = 0, kSrcFull = 1, kSrcSlices = 2 };

// stop logic of the series at one order from the reduced norms
// (power_series.py:29-42, 62-77); one thread
template <int MODE>
__device__ void series_stop(const CamArgs& a, double DD, double XX, double NF, double NZ) {
  SeriesState* st = a.st;
  if (MODE == kCamBt) {
    if (NZ == 0.0) {  // zero right-hand side (power_series.py:64-65)
      st->stopped = 1;
      st->converged = 1;
      st->order_used = 0;
      st->any_nonzero = -1;  // marks the zero-rhs shortcut
    } else if (NF > 0.0) {
      st->stopped = 1;
      st->error = POBA_ENONFINITE;
      st->error_order = 0;
    }
  } else {
    const int i = a.order;
    if (NF > 0.0) {
      st->stopped = 1;
      st->error = POBA_ENONFINITE;
      st->error_order = i;
    } else {
      st->order_used = i;
      if (a.check_stop) {
        if (XX == 0.0) {
          st->stopped = 1;
          st->error = POBA_EVANISH;
          st->error_order = i;
        } else {
          const double ratio = (double)(i + 1) * sqrt(DD) / sqrt(XX);
          if (a.ratios) a.ratios[i] = ratio;
          if (ratio < a.eps) {
            st->stopped = 1;
            st->converged = 1;
          }
        }
      }
    }
  }
}

// One warp per camera: the camera's reduced vector r (from the chunk partials,
// a full vector, or -- sliced -- the rank-order sum of the R received slices),
// then b_tilde / t = U^-1 r / x += t and the norms of the stop test.  The
// norms are reduced in a fixed order (lanes, warps, blocks in the last block);
// on a slice the last block leaves its four totals in the pad doubles of the
// slice's first four t records (all-gathered with t), and k_stop finishes.
template <int MODE, int SRC>
__global__ void __launch_bounds__(256) k_cam(const CamArgs a) {
  __shared__ double red[8][4];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cam = (SRC == kSrcSlices ? a.c0 : 0) + blockIdx.x * 8 + warp;
  const int cam_end = SRC == kSrcSlices ? a.c1 : a.n_cam;
  if (MODE == kCamTerm && a.st->stopped) return;
  double r[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) r[j] = 0.0;
  if (cam < cam_end) {
    if (SRC == kSrcSlices) {  // rank-order sum of the received slices
      const int64_t off = (int64_t)(cam - a.c0) * 9;
#pragma unroll
      for (int j = 0; j < 9; ++j) r[j] = a.recv[off + j];
      for (int rk = 1; rk < a.nranks; ++rk)
#pragma unroll
        for (int j = 0; j < 9; ++j) r[j] += a.recv[(int64_t)rk * a.ls * 9 + off + j];
    } else if (SRC == kSrcPartials) {
      const int p0 = a.part_cam_off[cam], p1 = a.part_cam_off[cam + 1];
      for (int p = p0 + lane; p < p1; p += 32) {  // 80-B partial records: five 16-B loads
        POBA_DCHECK(a.part_idx[p] >= 0);
        const double2* src = reinterpret_cast<const double2*>(a.partials + (int64_t)a.part_idx[p] * kTStride);
        double v[10];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double2 w = src[k];
          v[2 * k] = w.x;
          v[2 * k + 1] = w.y;
        }
#pragma unroll
        for (int j = 0; j < 9; ++j) r[j] += v[j];
      }
#pragma unroll
      for (int j = 0; j < 9; ++j)
#pragma unroll
        for (int s = 16; s; s >>= 1) r[j] += __shfl_xor_sync(0xffffffffu, r[j], s);
    } else {
#pragma unroll
      for (int j = 0; j < 9; ++j) r[j] = a.rin[(int64_t)cam * 9 + j];
    }
  }
  double dd = 0.0, xx = 0.0, nonfinite = 0.0, nonzero = 0.0;
  if (cam < cam_end && lane < 9) {
    const int i = lane;
    const int64_t q = (int64_t)cam * 9 + i;
    if (MODE == kCamMerge) {
      a.rout[q] = r[i];
    } else {
      double v[9];
      if (MODE == kCamBt) {
        // b_tilde = b_p - W V^-1 b_l ; t0 = U^-1 (-b_tilde)
#pragma unroll
        for (int j = 0; j < 9; ++j) v[j] = -(a.bp[(int64_t)cam * 9 + j] - r[j]);
        const double bti = a.bp[q] - r[i];
        a.bt[q] = bti;
        nonzero = (bti != 0.0) ? 1.0 : 0.0;
      } else {
#pragma unroll
        for (int j = 0; j < 9; ++j) v[j] = r[j];
      }
      const double* U = a.Uinv + (int64_t)cam * 45;
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) t = fma(U[sym9(i, j)], v[j], t);
      a.tvec[(int64_t)cam * kTStride + i] = t;
      if (MODE == kCamBt) {
        a.xvec[q] = t;
        xx = t * t;
        nonfinite = isfinite(t) ? 0.0 : 1.0;
      } else {
        const double xo = a.xvec[q];
        const double xn = xo + t;
        const double df = xn - xo;  // x_i - x_{i-1} exactly as the reference forms it
        a.xvec[q] = xn;
        dd = df * df;
        xx = xn * xn;
        nonfinite = isfinite(xn) ? 0.0 : 1.0;
      }
    }
  }
  if (MODE == kCamMerge) return;
  // fixed-order reductions: lanes (tree), warps (sequential), blocks (last block)
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    dd += __shfl_down_sync(0xffffffffu, dd, s);
    xx += __shfl_down_sync(0xffffffffu, xx, s);
    nonfinite += __shfl_down_sync(0xffffffffu, nonfinite, s);
    nonzero += __shfl_down_sync(0xffffffffu, nonzero, s);
  }
  if (lane == 0) {
    red[warp][0] = dd;
    red[warp][1] = xx;
    red[warp][2] = nonfinite;
    red[warp][3] = nonzero;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b[4] = {0, 0, 0, 0};
    for (int w = 0; w < 8; ++w)
      for (int k = 0; k < 4; ++k) b[k] += red[w][k];
    for (int k = 0; k < 4; ++k) a.blk[blockIdx.x * 4 + k] = b[k];
    __threadfence();
    const unsigned tk = atomicAdd(&a.st->ticket, 1u);
    last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: fixed-order sum of the block partials
  __shared__ double tot[256][4];
  double s4[4] = {0, 0, 0, 0};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 256)
    for (int k = 0; k < 4; ++k) s4[k] += ((volatile double*)a.blk)[b * 4 + k];
  for (int k = 0; k < 4; ++k) tot[threadIdx.x][k] = s4[k];
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 4; ++k) tot[threadIdx.x][k] += tot[threadIdx.x + s][k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.st->ticket = 0;
    if (SRC == kSrcSlices) {
      for (int k = 0; k < 4; ++k) a.tvec[(int64_t)(a.c0 + k) * kTStride + 9] = tot[0][k];
    } else {
      series_stop<MODE>(a, tot[0][0], tot[0][1], tot[0][2], tot[0][3]);
    }
  }
}

// sliced camera step: the ranks' norm totals (pad doubles of each slice's first
// four t records, all-gathered), summed in rank order -> the stop decision,
// identical on every rank
template <int MODE>
__global__ void k_stop(const CamArgs a) {
  if (threadIdx.x != 0) return;
  if (MODE == kCamTerm && a.st->stopped) return;
  double t4[4] = {0.0, 0.0, 0.0, 0.0};
  for (int rk = 0; rk < a.nranks; ++rk)
    for (int k = 0; k < 4; ++k) t4[k] += a.tvec[((int64_t)rk * a.ls + k) * kTStride + 9];
  series_stop<MODE>(a, t4[0], t4[1], t4[2], t4[3]);
}

// ---------------------------------------------------------------------------
// W^T-type passes with landmark output (apply_wt, back-substitution, long z)
// ---------------------------------------------------------------------------

// (min 3 blocks per SM: lets ptxas keep the twelve plane loads in flight
// together instead of sinking each next to its first use)
template <int OUT, bool F32>
__global__ void __launch_bounds__(kBlockTiles * kTile, 3)
k_wt_tile(const Tile* __restrict__ tiles, int tile0, int tile_end, const int* __restrict__ cam_s,
          const uint8_t* __restrict__ lidx_s, const void* __restrict__ J, const double* __restrict__ tin,
          const double* __restrict__ bl, const double* __restrict__ Vinv, double* __restrict__ out,
          int* __restrict__ nonzero_flag) {
  __shared__ double wbuf_all[kBlockTiles][kTile * 3];
  __shared__ int lstart_all[kBlockTiles][kTile + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ti = tile0 + blockIdx.x * kBlockTiles + w;
  if (ti >= tile_end) return;
  const int64_t o = (int64_t)ti * kTile + lane;
  // all twelve planes in flight first (one coalesced 512-B read per plane per
  // warp; the tile block covers the padding lanes), together with the slot's
  // camera and the tile descriptor; then the camera record
  double2 jr[kJPlanes];
#pragma unroll
  for (int p = 0; p < kJPlanes; ++p) jr[p] = jload<F32>(J, o, p);
  const int cam = cam_s[o];
  const int li_o = lidx_s[o];
  const Tile t = tiles[ti];
  if (t.flags & kTileLong) return;  // handled by k_wt_long
  double* wbuf = wbuf_all[w];
  int* lstart = lstart_all[w];
  // this lane's landmark operands (V^-1, b_l) requested as soon as the tile
  // descriptor is here, so they travel together with the camera records
  // instead of after the landmark sums
  double vi[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, blv[3] = {0.0, 0.0, 0.0};
  if (OUT != kOutWt && lane < t.nlm) {
    const int64_t lm = t.lm0 + lane;
#pragma unroll
    for (int k = 0; k < 6; ++k) vi[k] = Vinv[lm * 6 + k];
    if (OUT == kOutBack) {
#pragma unroll
      for (int k = 0; k < 3; ++k) blv[k] = bl[lm * 3 + k];
    }
  }
  if (lane < t.n) {
    const double2* tv = reinterpret_cast<const double2*>(tin + (int64_t)cam * kTStride);
    double tc[10];
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      const double2 v = __ldg(tv + p);
      tc[2 * p] = v.x;
      tc[2 * p + 1] = v.y;
    }
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      u0 = fma(jr[j].x, tc[j], u0);
      u1 = fma(jr[j].y, tc[j], u1);
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) wbuf[lane * 3 + b] = fma(jr[9 + b].x, u0, jr[9 + b].y * u1);
    const int li = li_o;
    if (lane == 0 || lidx_s[o - 1] != li) lstart[li] = lane;
  }
  if (lane == 0) lstart[t.nlm] = t.n;
  __syncwarp();
  if (lane < t.nlm) {
    const int lm = t.lm0 + lane;
    double y[3] = {0.0, 0.0, 0.0}, z[3];
    for (int r = lstart[lane]; r < lstart[lane + 1]; ++r) {
      y[0] += wbuf[r * 3];
      y[1] += wbuf[r * 3 + 1];
      y[2] += wbuf[r * 3 + 2];
    }
    if (OUT == kOutWt) {
      z[0] = y[0]; z[1] = y[1]; z[2] = y[2];
    } else if (OUT == kOutZ) {
      sym3_mv(vi, y, z);
    } else {
      const double yb[3] = {blv[0] + y[0], blv[1] + y[1], blv[2] + y[2]};
      sym3_mv(vi, yb, z);
      z[0] = -z[0]; z[1] = -z[1]; z[2] = -z[2];
      if (z[0] != 0.0 || z[1] != 0.0 || z[2] != 0.0) atomicOr(nonzero_flag, 1);
    }
    out[lm * 3] = z[0];
    out[lm * 3 + 1] = z[1];
    out[lm * 3 + 2] = z[2];
  }
}

// Landmarks with k > kTile: one warp per landmark, lanes stride its
// observations, fixed-shape butterfly for the landmark sum.
constexpr int kLongWarps = 8;
constexpr int kLongThreads = kLongWarps * 32;

template <int OUT, bool F32>
__global__ void __launch_bounds__(kLongThreads)
k_wt_long(const int* __restrict__ long_lm, int n_long, const int* __restrict__ lm_slot0, const int* __restrict__ lm_k,
          const int* __restrict__ cam_s, const void* __restrict__ J, int ts, const double* __restrict__ tin,
          const double* __restrict__ bl, const double* __restrict__ Vinv, double* __restrict__ out,
          int* __restrict__ nonzero_flag, const SeriesState* __restrict__ st, int check_stop) {
  if (check_stop && st->stopped) return;
  const int w = blockIdx.x * kLongWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n_long) return;
  const int lm = long_lm[w];
  const int o0 = lm_slot0[lm], o1 = o0 + lm_k[lm];
  double y0 = 0.0, y1 = 0.0, y2 = 0.0;
  for (int o = o0 + lane; o < o1; o += 32) {
    const double* tv = tin + (int64_t)cam_s[o] * ts;
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const double2 v = jload<F32>(J, o, j);
      u0 = fma(v.x, tv[j], u0);
      u1 = fma(v.y, tv[j], u1);
    }
    const double2 a = jload<F32>(J, o, 9), b = jload<F32>(J, o, 10), c = jload<F32>(J, o, 11);
    y0 += fma(a.x, u0, a.y * u1);
    y1 += fma(b.x, u0, b.y * u1);
    y2 += fma(c.x, u0, c.y * u1);
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    y0 += __shfl_xor_sync(0xffffffffu, y0, d);
    y1 += __shfl_xor_sync(0xffffffffu, y1, d);
    y2 += __shfl_xor_sync(0xffffffffu, y2, d);
  }
  if (lane == 0) {
    double y[3] = {y0, y1, y2}, z[3];
    if (OUT == kOutWt) {
      z[0] = y[0]; z[1] = y[1]; z[2] = y[2];
    } else if (OUT == kOutZ) {
      sym3_mv(Vinv + (int64_t)lm * 6, y, z);
    } else {
      const double yb[3] = {bl[lm * 3] + y[0], bl[lm * 3 + 1] + y[1], bl[lm * 3 + 2] + y[2]};
      sym3_mv(Vinv + (int64_t)lm * 6, yb, z);
      z[0] = -z[0]; z[1] = -z[1]; z[2] = -z[2];
      if (z[0] != 0.0 || z[1] != 0.0 || z[2] != 0.0) atomicOr(nonzero_flag, 1);
    }
    out[lm * 3] = z[0];
    out[lm * 3 + 1] = z[1];
    out[lm * 3 + 2] = z[2];
  }
}

// elementwise block-diagonal products
__global__ void k_cam_mv(const double* __restrict__ M45, const double* __restrict__ v, int64_t n_cam,
                         double* __restrict__ out, int os = 9) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_cam * 9) return;
  const int64_t c = q / 9;
  const int i = (int)(q - c * 9);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 9; ++j) s = fma(M45[c * 45 + sym9(i, j)], v[c * 9 + j], s);
  out[c * os + i] = s;
}

__global__ void k_restride(const double* __restrict__ in, int is, int64_t n_cam, double* __restrict__ out, int os) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_cam * 9) return;
  const int64_t c = q / 9;
  out[c * os + (q - c * 9)] = in[c * is + (q - c * 9)];
}

__global__ void k_lm_mv(const double* __restrict__ M6, const double* __restrict__ v, int64_t n_lm,
                        double* __restrict__ out) {
  int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (l >= n_lm) return;
  double y[3] = {v[l * 3], v[l * 3 + 1], v[l * 3 + 2]}, z[3];
  sym3_mv(M6 + l * 6, y, z);
  out[l * 3] = z[0];
  out[l * 3 + 1] = z[1];
  out[l * 3 + 2] = z[2];
}

__global__ void k_axpy_sub(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) out[q] = a[q] - b[q];
}

__global__ void k_add_inplace(double* __restrict__ a, const double* __restrict__ b, int64_t n) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) a[q] += b[q];
}

template <int OUT>
// tin: camera vector in 80-B records (kTStride); see wt_input
void launch_wt_tile(Ctx& c, const double* tin, const double* bl, double* out, int* flag, int t0 = 0,
                    int t1 = -1) {
  if (t1 < 0) t1 = c.n_tiles;
  if (t1 <= t0) return;
  const unsigned g = grid_for(t1 - t0, kBlockTiles);
  if (c.precision == 32) {
    k_wt_tile<OUT, true><<<g, kBlockTiles * kTile, 0, c.stream>>>(c.tiles.as<Tile>(), t0, t1, c.cam_s.as<int>(),
                                                                     c.lidx_s.as<uint8_t>(), c.J.p, tin, bl,
                                                                     c.Vinv.as<double>(), out, flag);
  } else {
    k_wt_tile<OUT, false><<<g, kBlockTiles * kTile, 0, c.stream>>>(c.tiles.as<Tile>(), t0, t1, c.cam_s.as<int>(),
                                                                      c.lidx_s.as<uint8_t>(), c.J.p, tin, bl,
                                                                      c.Vinv.as<double>(), out, flag);
  }
  c.launches++;
}

// a 9-stride camera vector copied into 80-B records for k_wt_tile's 16-B loads
int wt_input(Ctx& c, const double* v9, const double** out) {
  PTRY(c.wt_in.alloc(std::max<int64_t>(c.n_cam, 1) * kTStride * 8));
  k_restride<<<grid_for(c.n_cam * 9, 256), 256, 0, c.stream>>>(v9, 9, c.n_cam, c.wt_in.as<double>(), kTStride);
  c.launches++;
  *out = c.wt_in.as<double>();
  return POBA_OK;
}

template <int OUT>
void launch_wt_long(Ctx& c, const double* tin, int ts, const double* bl, double* out, int* flag, bool check_stop) {
  if (!c.n_long) return;
  const unsigned g = grid_for(c.n_long, kLongWarps);
  if (c.precision == 32)
    k_wt_long<OUT, true><<<g, kLongThreads, 0, c.stream>>>(c.long_lm.as<int>(), c.n_long, c.lm_slot0.as<int>(),
                                                           c.lm_k.as<int>(), c.cam_s.as<int>(), c.J.p, ts, tin, bl,
                                                           c.Vinv.as<double>(), out, flag, c.state.as<SeriesState>(),
                                                           check_stop ? 1 : 0);
  else
    k_wt_long<OUT, false><<<g, kLongThreads, 0, c.stream>>>(c.long_lm.as<int>(), c.n_long, c.lm_slot0.as<int>(),
                                                            c.lm_k.as<int>(), c.cam_s.as<int>(), c.J.p, ts, tin, bl,
                                                            c.Vinv.as<double>(), out, flag,
                                                            c.state.as<SeriesState>(), check_stop ? 1 : 0);
  c.launches++;
}

int configure_term(Ctx& c) {
  static thread_local int done_dev = -1;
  int dev = 0;
  PCK(cudaGetDevice(&dev));
  if (done_dev != dev) {
    auto setup = [](const void* f, int smem) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      // all of the SM's unified L1 as shared memory (needed for kTermCtas > 1 to be co-resident)
      return cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    };
#define POBA_TERM_SETUP(CT)                                                                          \
  PCK(setup((const void*)k_term<kModeTerm, false, CT>, TermShape<CT>::kTermSmem));                   \
  PCK(setup((const void*)k_term<kModeBt, false, CT>, TermShape<CT>::kTermSmem));                     \
  PCK(setup((const void*)k_term<kModeW, false, CT>, TermShape<CT>::kTermSmem));                      \
  PCK(setup((const void*)k_term<kModeTerm, true, CT>, TermShape<CT>::kTermSmem));                    \
  PCK(setup((const void*)k_term<kModeBt, true, CT>, TermShape<CT>::kTermSmem));                      \
  PCK(setup((const void*)k_term<kModeW, true, CT>, TermShape<CT>::kTermSmem));
    POBA_TERM_SETUP(false)
    POBA_TERM_SETUP(true)
#undef POBA_TERM_SETUP
    done_dev = dev;
  }
  return POBA_OK;
}

TermArgs term_args(Ctx& c, const double* tin, const double* lvec, bool check_stop) {
  TermArgs a;
  a.tk = c.tilek.as<TileK>();
  a.cta_tiles = c.cta_tiles.as<int2>();
  a.cam_s = c.cam_s.as<int>();
  a.part_cam = c.part_cam.as<int>();
  a.J = c.J.p;
  a.tin = tin;
  a.lvec = lvec;
  a.Vinv = c.Vinv.as<double>();
  a.zlong = c.ltmp.as<double>();
  a.partials = c.partials.as<double>();
  a.st = c.state.as<SeriesState>();
  a.check_stop = check_stop ? 1 : 0;
  a.n_cam = (int)c.n_cam;
  a.n_partials = c.n_partials;
  a.n_lm = (int)c.n_lm_l;
  return a;
}

CamArgs cam_args(Ctx& c, int order, double eps, bool check_stop) {
  CamArgs a;
  a.part_cam_off = c.part_cam_off.as<int>();
  a.part_idx = c.part_idx.as<int>();
  a.partials = c.partials.as<double>();
  a.rin = c.rvec.as<double>();
  a.rout = c.rvec.as<double>();
  a.Uinv = c.Uinv.as<double>();
  a.bp = c.bp.as<double>();
  a.bt = c.bt.as<double>();
  a.tvec = c.tvec.as<double>();
  a.xvec = c.xvec.as<double>();
  a.blk = c.blk_part.as<double>();
  a.st = c.state.as<SeriesState>();
  a.ratios = c.ratios.as<double>();
  a.n_cam = (int)c.n_cam;
  a.order = order;
  a.eps = eps;
  a.check_stop = check_stop ? 1 : 0;
  a.recv = nullptr;
  a.nranks = c.nranks;
  a.ls = (int)c.cam_ls;
  a.c0 = 0;
  a.c1 = (int)c.n_cam;
  return a;
}

template <bool CT>
void launch_term_shape(Ctx& c, int mode, const TermArgs& a) {
  const size_t smem = TermShape<CT>::kTermSmem;
  const unsigned grid = (unsigned)c.n_cta;
  const bool f32 = c.precision == 32;
  if (mode == kModeTerm) {
    if (f32) k_term<kModeTerm, true, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
    else k_term<kModeTerm, false, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
  } else if (mode == kModeBt) {
    if (f32) k_term<kModeBt, true, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
    else k_term<kModeBt, false, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
  } else {
    if (f32) k_term<kModeW, true, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
    else k_term<kModeW, false, CT><<<grid, TermShape<CT>::kWarps * 32, smem, c.stream>>>(a);
  }
}

int launch_term(Ctx& c, int mode, const double* tin, const double* lvec, bool check_stop) {
  PTRY(configure_term(c));
  const TermArgs a = term_args(c, tin, lvec, check_stop);
  if (mode == kModeTerm) launch_wt_long<kOutZ>(c, tin, kTStride, nullptr, c.ltmp.as<double>(), nullptr, check_stop);
  if (c.chunk_t) launch_term_shape<true>(c, mode, a);
  else launch_term_shape<false>(c, mode, a);
  c.launches++;
  PCK(cudaGetLastError());
  return POBA_OK;
}

// camera step after a term kernel.  One GPU: merge the chunk partials and
// finalize in one kernel.  Sharded: merge this rank's partials, then either
// (kCamMerge) the rank-ordered all-reduce of the full vector, or (series
// terms, b_tilde) the SLICED step: exchange slices of the partial vector,
// each rank finalizes only its cameras [c0, c1) (U^-1, x, norms), all-gather
// of the t records (with the norm totals in their pad doubles), and k_stop.
// Same NVLink bytes as an all-reduce; the camera work is 1/R per rank.
int launch_cam(Ctx& c, int mode, int order, double eps, bool check_stop, const CamArgs* override_args = nullptr) {
  const unsigned nb = grid_for(c.n_cam, 8);
  CamArgs a = override_args ? *override_args : cam_args(c, order, eps, check_stop);
  if (c.nranks == 1) {
    if (mode == kCamTerm) k_cam<kCamTerm, kSrcPartials><<<nb, 256, 0, c.stream>>>(a);
    else if (mode == kCamBt) k_cam<kCamBt, kSrcPartials><<<nb, 256, 0, c.stream>>>(a);
    else k_cam<kCamMerge, kSrcPartials><<<nb, 256, 0, c.stream>>>(a);
    c.launches++;
  } else if (mode == kCamMerge) {
    k_cam<kCamMerge, kSrcPartials><<<nb, 256, 0, c.stream>>>(a);
    c.launches++;
    PTRY(allreduce_sum(c, c.rvec.as<double>(), c.n_cam * 9));
  } else {
    {
      // the merge of this rank's partials writes straight into the padded
      // send buffer of the slice exchange (no copy of the camera vector)
      const size_t per = (size_t)c.cam_ls * 9;
      PTRY(c.xch_send.alloc(per * c.nranks * 8));
      PTRY(c.xch_recv.alloc(per * c.nranks * 8));
      double* snd = c.xch_send.as<double>();
      if ((int64_t)per * c.nranks > c.n_cam * 9)
        PCK(cudaMemsetAsync(snd + c.n_cam * 9, 0, (per * c.nranks - c.n_cam * 9) * 8, c.stream));
      CamArgs m = a;
      m.rout = snd;
      k_cam<kCamMerge, kSrcPartials><<<nb, 256, 0, c.stream>>>(m);
      c.launches++;
      PTRY(exchange_slices(c, snd, c.xch_recv.as<double>(), per));
      a.recv = c.xch_recv.as<double>();
      a.nranks = c.nranks;
      a.ls = (int)c.cam_ls;
      a.c0 = (int)std::min<int64_t>(c.n_cam, (int64_t)c.rank * c.cam_ls);
      a.c1 = (int)std::min<int64_t>(c.n_cam, (int64_t)(c.rank + 1) * c.cam_ls);
      const unsigned nbs = std::max(1u, grid_for(a.c1 - a.c0, 8));
      if (mode == kCamTerm) k_cam<kCamTerm, kSrcSlices><<<nbs, 256, 0, c.stream>>>(a);
      else k_cam<kCamBt, kSrcSlices><<<nbs, 256, 0, c.stream>>>(a);
      const size_t rec = (size_t)c.cam_ls * kTStride;
      PTRY(allgather(c, a.tvec + (size_t)c.rank * rec, a.tvec, rec));
      if (mode == kCamTerm) k_stop<kCamTerm><<<1, 32, 0, c.stream>>>(a);
      else k_stop<kCamBt><<<1, 32, 0, c.stream>>>(a);
      c.launches += 2;
    }
  }
  PCK(cudaGetLastError());
  return POBA_OK;
}

int ensure_ratios(Ctx& c, int max_order) {
  if (c.ratios_cap < max_order + 1) {
    PTRY(c.ratios.alloc((size_t)(max_order + 1) * 8));
    c.ratios_cap = max_order + 1;
  }
  return POBA_OK;
}

__global__ void k_fill(double* __restrict__ p, int64_t n, double v) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) p[q] = v;
}

}  // namespace

int damp_device(Ctx& c, double lam, int identity) {
  cudaStream_t s = c.stream;
  int* fl = c.flag.as<int>();
  PCK(cudaMemsetAsync(fl, 0, 4, s));
  k_damp_u<<<grid_for(c.n_cam, 64), 64, 0, s>>>(c.U0.as<double>(), c.Dp.as<double>(), c.n_cam, lam, identity,
                                                c.Ud.as<double>(), c.Uinv.as<double>(), fl);
  if (c.n_lm_l)
    k_damp_v<<<grid_for(c.n_lm_l, 256), 256, 0, s>>>(c.V0.as<double>(), c.Dl.as<double>(), c.n_lm_l, lam, identity,
                                                    c.Vd.as<double>(), c.Vinv.as<double>(), fl);
  c.launches += 2;
  PCK(cudaGetLastError());
  int h = 0;
  PCK(cudaMemcpyAsync(&h, fl, 4, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (c.nranks > 1) {
    double v = (double)h, out = 0;
    PTRY(c.scratch_b.alloc(8));
    PCK(cudaMemcpyAsync(c.scratch_b.p, &v, 8, cudaMemcpyHostToDevice, s));
    PTRY(allreduce_max(c, c.scratch_b.as<double>(), 1));
    PCK(cudaMemcpyAsync(&out, c.scratch_b.p, 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    h = (int)out;
  }
  if (h & 1) return fail(POBA_ENOTSPD, "damped pose blocks are not positive definite, assembly bug or lambda too small");
  if (h & 2) return fail(POBA_ENOTSPD, "damped point blocks are not positive definite, assembly bug or lambda too small");
  c.lam = lam;
  c.identity = identity;
  c.have_damp = true;
  c.have_solution = c.have_delta_l = false;
  return POBA_OK;
}

// entry points for the clustered (PoST) series in clustered.cu
int launch_term_mode(Ctx& c, int mode, const double* tin, const double* lvec, bool check_stop) {
  PTRY(configure_term(c));
  return launch_term(c, mode, tin, lvec, check_stop);
}
int launch_merge(Ctx& c) { return launch_cam(c, kCamMerge, 0, 0.0, false); }

// the launches of one series solve (b_tilde, t0, then max_order terms; every
// kernel checks the device-side stop flag, so the sequence is fixed)
int enqueue_series(Ctx& c, double eps, int max_order, bool forced) {
  cudaStream_t s = c.stream;
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  k_fill<<<grid_for(max_order + 1, 128), 128, 0, s>>>(c.ratios.as<double>(), max_order + 1,
                                                     std::numeric_limits<double>::quiet_NaN());
  c.launches++;
  // order 0: b_tilde and t0
  PTRY(launch_term(c, kModeBt, nullptr, c.bl.as<double>(), false));
  PTRY(launch_cam(c, kCamBt, 0, eps, false));
  PTRY(gather_cam_slices(c, c.bt.as<double>(), 9));
  for (int i = 1; i <= max_order; ++i) {
    PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, true));
    PTRY(launch_cam(c, kCamTerm, i, eps, !forced));
  }
  PTRY(gather_cam_slices(c, c.xvec.as<double>(), 9));
  return POBA_OK;
}

int series_device(Ctx& c, double eps, int max_order, bool forced, int* order_used, int* converged) {
  cudaStream_t s = c.stream;
  PTRY(ensure_ratios(c, max_order));
  PTRY(configure_term(c));
  // The whole solve is one CUDA graph, captured once per (eps, m): on one GPU,
  // and on NCCL-sharded contexts (the per-term exchange / all-gather are
  // captured with the kernels, every rank launches the same graph).  Virtual
  // ranks meet at host barriers inside their collectives, so they enqueue.
  if ((c.nranks > 1 && c.group) || c.graph_off || getenv("POBA_NO_GRAPH")) {
    PTRY(enqueue_series(c, eps, max_order, forced));
  } else {
    SeriesGraph* g = nullptr;
    for (auto& x : c.graphs)
      if (x.eps == eps && x.max_order == max_order && x.forced == forced && x.ratios == c.ratios.p) g = &x;
    if (!g) {
      SeriesGraph ng;
      ng.eps = eps;
      ng.max_order = max_order;
      ng.forced = forced;
      ng.ratios = c.ratios.p;
      const int64_t l0 = c.launches;
      if (c.nranks > 1) {  // collective scratch sized before capture (no allocation inside a graph)
        const size_t per = std::max<size_t>(((size_t)c.n_cam * 9 + c.nranks - 1) / c.nranks, (size_t)c.cam_ls * 9);
        PTRY(c.xch_send.alloc(per * c.nranks * 8));
        PTRY(c.xch_recv.alloc(per * c.nranks * 8));
      }
      PCK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const int st_enq = enqueue_series(c, eps, max_order, forced);
      cudaGraph_t graph = nullptr;
      const cudaError_t e_end = cudaStreamEndCapture(s, &graph);
      cudaError_t e_inst = cudaSuccess;
      if (st_enq == POBA_OK && e_end == cudaSuccess) e_inst = cudaGraphInstantiate(&ng.exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (st_enq != POBA_OK || e_end != cudaSuccess || e_inst != cudaSuccess) {
        c.launches = l0;
        if (c.nranks > 1) {
          // an NCCL build / topology that cannot capture its collectives: the
          // same launches, enqueued (nothing of the failed capture has run)
          cudaGetLastError();
          c.graph_off = true;
          fprintf(stderr, "libpoba: rank %d: series capture failed, enqueueing the sharded series instead\n", c.rank);
          PTRY(enqueue_series(c, eps, max_order, forced));
        } else {
          if (st_enq != POBA_OK) return st_enq;
          PCK(e_end);
          PCK(e_inst);
        }
      } else {
        ng.launches = c.launches - l0;
        c.launches = l0;
        c.graphs.push_back(ng);
        g = &c.graphs.back();
      }
    }
    if (g) {
      PCK(cudaGraphLaunch(g->exec, s));
      c.launches += g->launches;
    }
  }
  SeriesState st;
  PCK(cudaMemcpyAsync(&st, c.state.p, sizeof(st), cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  c.have_solution = false;
  if (st.error == POBA_ENONFINITE)
    return fail(POBA_ENONFINITE, "non-finite series iterate at order " + std::to_string(st.error_order) +
                                     ", assembly is broken");
  if (st.error == POBA_EVANISH)
    return fail(POBA_EVANISH, "vanishing iterate norm with a nonzero right-hand side");
  if (st.any_nonzero == -1) {  // zero rhs: delta_p = 0, order 0
    PCK(cudaMemsetAsync(c.xvec.p, 0, c.n_cam * 9 * 8, s));
    *order_used = 0;
    *converged = 1;
  } else if (max_order == 0) {
    *order_used = 0;
    *converged = 0;
  } else {
    *order_used = st.converged ? st.order_used : max_order;
    *converged = st.converged;
  }
  c.last_order = *order_used;
  c.have_solution = true;
  return POBA_OK;
}

int b_tilde_device(Ctx& c) {
  // b_tilde alone (DampedSystem.b_tilde, blocks.py:256-260) without touching
  // the series state: t0/x0 go to scratch vectors, flags to an aux state.
  cudaStream_t s = c.stream;
  PTRY(c.state_aux.alloc(sizeof(SeriesState)));
  PCK(cudaMemsetAsync(c.state_aux.p, 0, sizeof(SeriesState), s));
  PTRY(launch_term(c, kModeBt, nullptr, c.bl.as<double>(), false));
  CamArgs a = cam_args(c, 0, 1.0, false);
  a.tvec = c.ctmp.as<double>();
  a.xvec = c.ctmp2.as<double>();
  a.st = c.state_aux.as<SeriesState>();
  PTRY(launch_cam(c, kCamBt, 0, 1.0, false, &a));
  PTRY(gather_cam_slices(c, c.bt.as<double>(), 9));
  PCK(cudaStreamSynchronize(s));
  return POBA_OK;
}

int points_accept_device(Ctx& c) {
  k_add_inplace<<<grid_for(c.n_lm_l * 3, 256), 256, 0, c.stream>>>(c.points.as<double>(), c.dl.as<double>(),
                                                                  c.n_lm_l * 3);
  c.launches++;
  PCK(cudaGetLastError());
  PCK(cudaStreamSynchronize(c.stream));
  c.have_delta_l = false;
  return POBA_OK;
}

int series_apply_device(Ctx& c, const double* d_v, int order, double* d_out) {
  // apply_series_inverse (power_series.py:80-91): x = sum_{i<=order} P^i U^-1 v
  cudaStream_t s = c.stream;
  k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.Uinv.as<double>(), d_v, c.n_cam, c.tvec.as<double>(),
                                                     kTStride);
  k_restride<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.tvec.as<double>(), kTStride, c.n_cam, c.xvec.as<double>(), 9);
  c.launches++;
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  c.launches++;
  for (int i = 1; i <= order; ++i) {
    PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
    PTRY(launch_cam(c, kCamTerm, i, 1.0, false));
  }
  PTRY(gather_cam_slices(c, c.xvec.as<double>(), 9));
  PCK(cudaMemcpyAsync(d_out, c.xvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, s));
  PCK(cudaStreamSynchronize(s));
  c.have_solution = false;
  return POBA_OK;
}

int back_substitute_device(Ctx& c, const double* d_dp, int* nonzero, double* h_dl) {
  cudaStream_t s = c.stream;
  int* fl = c.flag.as<int>() + 1;
  PCK(cudaMemsetAsync(fl, 0, 4, s));
  const bool piped = h_dl && xfer_pipelined(c, 3);
  const bool pinned = piped && is_pinned(h_dl);
  if (piped) {
    // long landmarks first, then store prefixes; each completed file piece is
    // permuted and copied out while the next prefix is computed
    launch_wt_long<kOutBack>(c, d_dp, 9, c.bl.as<double>(), c.dl.as<double>(), fl, false);
    const double* tin = nullptr;
    PTRY(wt_input(c, d_dp, &tin));
    PTRY(xfer_begin(c, 3, pinned));
    for (int i = 0; i < kXferPieces; ++i) {
      launch_wt_tile<kOutBack>(c, tin, c.bl.as<double>(), c.dl.as<double>(), fl, c.xf_dn_tile[i],
                               c.xf_dn_tile[i + 1]);
      PTRY(lm_download_piece(c, c.dl.as<double>(), 3, h_dl, i, pinned));
    }
  } else {
    const double* tin = nullptr;
    PTRY(wt_input(c, d_dp, &tin));
    launch_wt_tile<kOutBack>(c, tin, c.bl.as<double>(), c.dl.as<double>(), fl);
    launch_wt_long<kOutBack>(c, d_dp, 9, c.bl.as<double>(), c.dl.as<double>(), fl, false);
  }
  PCK(cudaGetLastError());
  if (piped) PTRY(lm_download_finish(c, h_dl, 3, pinned));
  int h = 0;
  PCK(cudaMemcpyAsync(&h, fl, 4, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (c.nranks > 1) {
    double v = (double)h, out = 0;
    PTRY(c.scratch_b.alloc(8));
    PCK(cudaMemcpyAsync(c.scratch_b.p, &v, 8, cudaMemcpyHostToDevice, s));
    PTRY(allreduce_max(c, c.scratch_b.as<double>(), 1));
    PCK(cudaMemcpyAsync(&out, c.scratch_b.p, 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    h = (int)out;
  }
  *nonzero = h;
  c.have_delta_l = true;
  if (h_dl && !piped) PTRY(lm_download(c, c.dl.as<double>(), 3, h_dl));
  return POBA_OK;
}

int apply_op_device(Ctx& c, int op, const double* d_in, double* d_out) {
  cudaStream_t s = c.stream;
  switch (op) {
    case POBA_OP_W:  // landmark-local input (canonical order) -> camera vector
      PTRY(launch_term(c, kModeW, nullptr, d_in, false));
      PTRY(launch_cam(c, kCamMerge, 0, 0.0, false));
      PCK(cudaMemcpyAsync(d_out, c.rvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, s));
      break;
    case POBA_OP_WT: {
      const double* tin = nullptr;
      PTRY(wt_input(c, d_in, &tin));
      launch_wt_tile<kOutWt>(c, tin, nullptr, d_out, nullptr);
      launch_wt_long<kOutWt>(c, d_in, 9, nullptr, d_out, nullptr, false);
      break;
    }
    case POBA_OP_U_INV:
      k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.Uinv.as<double>(), d_in, c.n_cam, d_out);
      c.launches++;
      break;
    case POBA_OP_U:
      k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.Ud.as<double>(), d_in, c.n_cam, d_out);
      c.launches++;
      break;
    case POBA_OP_V_INV:
      k_lm_mv<<<grid_for(c.n_lm_l, 256), 256, 0, s>>>(c.Vinv.as<double>(), d_in, c.n_lm_l, d_out);
      c.launches++;
      break;
    case POBA_OP_WVW: {  // W V^-1 W^T v with one pass of the fused term kernel
      k_restride<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(d_in, 9, c.n_cam, c.tvec.as<double>(), kTStride);
      c.launches++;
      PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
      PTRY(launch_cam(c, kCamMerge, 0, 0.0, false));
      PCK(cudaMemcpyAsync(d_out, c.rvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, s));
      break;
    }
    case POBA_OP_SCHUR: {
      // S v = U v - W V^-1 W^T v
      PTRY(apply_op_device(c, POBA_OP_WT, d_in, c.ltmp.as<double>()));
      k_lm_mv<<<grid_for(c.n_lm_l, 256), 256, 0, s>>>(c.Vinv.as<double>(), c.ltmp.as<double>(), c.n_lm_l,
                                                      c.ltmp.as<double>());
      c.launches++;
      PTRY(apply_op_device(c, POBA_OP_W, c.ltmp.as<double>(), c.ctmp2.as<double>()));
      k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.Ud.as<double>(), d_in, c.n_cam, c.ctmp.as<double>());
      k_axpy_sub<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.ctmp.as<double>(), c.ctmp2.as<double>(),
                                                            c.n_cam * 9, d_out);
      c.launches += 2;
      break;
    }
    default:
      return fail(POBA_EINVAL, "unknown operator");
  }
  PCK(cudaGetLastError());
  return POBA_OK;
}

// S p = U p - W V^-1 W^T p (apply_schur, blocks.py:252-254) with ONE pass of the
// fused term kernel: p (stride 9) -> 80-B records, term kernel + merge -> W V^-1 W^T p
int schur_product_device(Ctx& c, const double* d_p, double* d_out) {
  cudaStream_t s = c.stream;
  const unsigned g = grid_for(c.n_cam * 9, 256);
  k_restride<<<g, 256, 0, s>>>(d_p, 9, c.n_cam, c.tvec.as<double>(), kTStride);
  c.launches++;
  PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
  PTRY(launch_cam(c, kCamMerge, 0, 0.0, false));
  k_cam_mv<<<g, 256, 0, s>>>(c.Ud.as<double>(), d_p, c.n_cam, c.ctmp.as<double>());
  k_axpy_sub<<<g, 256, 0, s>>>(c.ctmp.as<double>(), c.rvec.as<double>(), c.n_cam * 9, d_out);
  c.launches += 2;
  PCK(cudaGetLastError());
  return POBA_OK;
}

// SPD inverse of 45-packed 9x9 blocks (the damped-U Cholesky path with no damping)
int damp_u_blocks(Ctx& c, const double* M45, double* M45_copy, double* Minv45, const char* what) {
  cudaStream_t s = c.stream;
  int* fl = c.flag.as<int>() + 3;
  PCK(cudaMemsetAsync(fl, 0, 4, s));
  k_damp_u<<<grid_for(c.n_cam, 64), 64, 0, s>>>(M45, c.Dp.as<double>(), c.n_cam, 0.0, 1, M45_copy, Minv45, fl);
  c.launches++;
  PCK(cudaGetLastError());
  int h = 0;
  PTRY(copy_sync(c, &h, fl, 4, cudaMemcpyDeviceToHost));
  if (h & 1) return fail(POBA_ENOTSPD, what);
  return POBA_OK;
}

void launch_cam_mv(Ctx& c, const double* M45, const double* v, double* out) {
  k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, c.stream>>>(M45, v, c.n_cam, out);
  c.launches++;
}

int time_terms_device(Ctx& c, int reps, double* ms_per_term, double* ms_term_kernel, int* launches) {
  cudaStream_t s = c.stream;
  cudaEvent_t e0, e1, e2;
  PCK(cudaEventCreate(&e0));
  PCK(cudaEventCreate(&e1));
  PCK(cudaEventCreate(&e2));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  // warm-up
  PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
  PTRY(launch_cam(c, kCamTerm, 1, 1.0, false));
  const int64_t l0 = c.launches;
  PCK(cudaEventRecord(e0, s));
  for (int r = 0; r < reps; ++r) {
    PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
    PTRY(launch_cam(c, kCamTerm, 1, 1.0, false));
  }
  PCK(cudaEventRecord(e1, s));
  const int64_t l1 = c.launches;
  for (int r = 0; r < reps; ++r) PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
  PCK(cudaEventRecord(e2, s));
  PCK(cudaEventSynchronize(e2));
  float a = 0, b = 0;
  PCK(cudaEventElapsedTime(&a, e0, e1));
  PCK(cudaEventElapsedTime(&b, e1, e2));
  *ms_per_term = a / reps;
  *ms_term_kernel = b / reps;
  *launches = (int)((l1 - l0) / reps);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  c.have_solution = false;
  return POBA_OK;
}

}  // namespace poba
