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
#include <limits>

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
// the fused term kernel (one CTA per chunk of tiles)
// ---------------------------------------------------------------------------

struct TermArgs {
  const Tile* tiles;
  const Chunk* chunks;
  const int* cam_l;
  const uint8_t* perm;
  const uint16_t* seg_start;
  const uint16_t* seg_slot;
  const double2* J;
  int64_t pad;
  const double* tin;    // camera vector (kModeTerm)
  const double* lvec;   // b_l (kModeBt) or landmark input (kModeW)
  const double* Vinv;
  const double* zlong;  // landmark-indexed z of long landmarks (kModeTerm)
  double* partials;
  const SeriesState* st;
  int max_slots;
  int check_stop;
};

template <int MODE>
__global__ void __launch_bounds__(kTile, 2) k_term(const TermArgs a) {
  extern __shared__ double sm[];
  double* acc = sm;
  double* gbuf = acc + a.max_slots * 9;
  double* wbuf = gbuf + kTile * 9;
  double* zbuf = wbuf + kTile * 3;
  uint8_t* pbuf = reinterpret_cast<uint8_t*>(zbuf + kTile * 3);
  uint16_t* sbuf = reinterpret_cast<uint16_t*>(pbuf + kTile);  // [start | slot] x kTile
  const int tid = threadIdx.x;
  if (a.check_stop && a.st->stopped) return;
  const Chunk ch = a.chunks[blockIdx.x];
  for (int q = tid; q < ch.nslot * 9; q += kTile) acc[q] = 0.0;

  // prologue: operands of the first tile
  Tile t = a.tiles[ch.tile0];
  double2 jr[kJPlanes];
  double tc[9];
  uint8_t pr = 0;
  uint16_t s_start = 0, s_slot = 0;
  auto fetch = [&](const Tile& tt) {
    if (tid < tt.n) {
      const int o = tt.obs0 + tid;
#pragma unroll
      for (int p = 0; p < kJPlanes; ++p) jr[p] = __ldcs(&a.J[p * a.pad + o]);  // streamed once per term
      pr = a.perm[o];
      if (MODE == kModeTerm && tt.k <= kTile) {
        const double* tv = a.tin + (int64_t)a.cam_l[o] * 9;
#pragma unroll
        for (int j = 0; j < 9; ++j) tc[j] = tv[j];
      }
    }
    if (tid < tt.nseg) {
      s_start = a.seg_start[tt.seg0 + tid];
      s_slot = a.seg_slot[tt.seg0 + tid];
    }
  };
  fetch(t);

  for (int ti = ch.tile0; ti < ch.tile1; ++ti) {
    const bool valid = tid < t.n;
    const bool is_long = t.k > kTile;
    // phase 1: w_o = J_l^T (J_p t_c)
    if (valid) {
      if (MODE == kModeTerm && !is_long) {
        double u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          u0 = fma(jr[j].x, tc[j], u0);
          u1 = fma(jr[j].y, tc[j], u1);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) wbuf[tid * 3 + b] = fma(jr[9 + b].x, u0, jr[9 + b].y * u1);
      }
    }
    __syncthreads();
    // (pbuf/sbuf are rewritten only after the sync above: the previous tile's
    // phase 4 reads them)
    if (valid) pbuf[tid] = pr;
    if (tid < t.nseg) {
      sbuf[tid] = s_start;
      sbuf[kTile + tid] = s_slot;
    }
    // phase 2: per landmark z_l
    if (tid < t.nlm) {
      const int lm = t.lm0 + tid;
      double y[3], z[3];
      if (MODE == kModeW) {
        z[0] = a.lvec[lm * 3]; z[1] = a.lvec[lm * 3 + 1]; z[2] = a.lvec[lm * 3 + 2];
      } else if (MODE == kModeTerm && is_long) {
        z[0] = a.zlong[lm * 3]; z[1] = a.zlong[lm * 3 + 1]; z[2] = a.zlong[lm * 3 + 2];
      } else {
        if (MODE == kModeBt) {
          y[0] = a.lvec[lm * 3]; y[1] = a.lvec[lm * 3 + 1]; y[2] = a.lvec[lm * 3 + 2];
        } else {
          y[0] = y[1] = y[2] = 0.0;
          const double* w = wbuf + tid * t.k * 3;
          for (int r = 0; r < t.k; ++r) {
            y[0] += w[r * 3];
            y[1] += w[r * 3 + 1];
            y[2] += w[r * 3 + 2];
          }
        }
        sym3_mv(a.Vinv + (int64_t)lm * 6, y, z);
      }
      zbuf[tid * 3] = z[0];
      zbuf[tid * 3 + 1] = z[1];
      zbuf[tid * 3 + 2] = z[2];
    }
    __syncthreads();
    // phase 3: g_o = J_p^T (J_l z_l)
    if (valid) {
      const int j = is_long ? 0 : tid / t.k;
      const double z0 = zbuf[j * 3], z1 = zbuf[j * 3 + 1], z2 = zbuf[j * 3 + 2];
      const double v0 = fma(jr[9].x, z0, fma(jr[10].x, z1, jr[11].x * z2));
      const double v1 = fma(jr[9].y, z0, fma(jr[10].y, z1, jr[11].y * z2));
#pragma unroll
      for (int q = 0; q < 9; ++q) gbuf[tid * 9 + q] = fma(jr[q].x, v0, jr[q].y * v1);
    }
    // prefetch the next tile while this one is reduced
    const int nseg = t.nseg, tn = t.n;
    if (ti + 1 < ch.tile1) {
      t = a.tiles[ti + 1];
      fetch(t);
    }
    __syncthreads();
    // phase 4: camera segments -> slot accumulators, fixed order
    for (int q = tid; q < nseg * 9; q += kTile) {
      const int s = q / 9, comp = q - s * 9;
      const int r0 = sbuf[s], r1 = (s + 1 < nseg) ? sbuf[s + 1] : tn;
      double sum = 0.0;
      for (int r = r0; r < r1; ++r) sum += gbuf[pbuf[r] * 9 + comp];
      acc[sbuf[kTile + s] * 9 + comp] += sum;
    }
    // the next phase-1 sync orders this phase before gbuf/sbuf are rewritten
  }
  __syncthreads();
  double* dst = a.partials + (int64_t)ch.part0 * 9;
  for (int q = tid; q < ch.nslot * 9; q += kTile) dst[q] = acc[q];
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
};

template <int MODE, bool kFromPartials>
__global__ void __launch_bounds__(256) k_cam(const CamArgs a) {
  __shared__ double red[8][4];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cam = blockIdx.x * 8 + warp;
  if (MODE == kCamTerm && a.st->stopped) return;
  double r[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) r[j] = 0.0;
  if (cam < a.n_cam) {
    if (kFromPartials) {
      const int p0 = a.part_cam_off[cam], p1 = a.part_cam_off[cam + 1];
      for (int p = p0 + lane; p < p1; p += 32) {
        const double* src = a.partials + (int64_t)a.part_idx[p] * 9;
#pragma unroll
        for (int j = 0; j < 9; ++j) r[j] += src[j];
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
  if (cam < a.n_cam && lane < 9) {
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
      a.tvec[q] = t;
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
    SeriesState* st = a.st;
    st->ticket = 0;
    const double DD = tot[0][0], XX = tot[0][1], NF = tot[0][2], NZ = tot[0][3];
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
}

// ---------------------------------------------------------------------------
// W^T-type passes with landmark output (apply_wt, back-substitution, long z)
// ---------------------------------------------------------------------------

template <int OUT>
__global__ void __launch_bounds__(kTile)
k_wt_tile(const Tile* __restrict__ tiles, const int* __restrict__ cam_l, const double2* __restrict__ J,
          int64_t pad, const double* __restrict__ tin, const double* __restrict__ bl,
          const double* __restrict__ Vinv, double* __restrict__ out, int* __restrict__ nonzero_flag) {
  __shared__ double wbuf[kTile * 3];
  const Tile t = tiles[blockIdx.x];
  if (t.k > kTile) return;  // handled by k_wt_long
  const int tid = threadIdx.x;
  if (tid < t.n) {
    const int o = t.obs0 + tid;
    const double* tv = tin + (int64_t)cam_l[o] * 9;
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const double2 v = J[j * pad + o];
      u0 = fma(v.x, tv[j], u0);
      u1 = fma(v.y, tv[j], u1);
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double2 v = J[(9 + b) * pad + o];
      wbuf[tid * 3 + b] = fma(v.x, u0, v.y * u1);
    }
  }
  __syncthreads();
  if (tid < t.nlm) {
    const int lm = t.lm0 + tid;
    double y[3] = {0.0, 0.0, 0.0}, z[3];
    const double* w = wbuf + tid * t.k * 3;
    for (int r = 0; r < t.k; ++r) {
      y[0] += w[r * 3];
      y[1] += w[r * 3 + 1];
      y[2] += w[r * 3 + 2];
    }
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

template <int OUT>
__global__ void __launch_bounds__(kTile)
k_wt_long(const int* __restrict__ long_lm, const int* __restrict__ lm_off, const int* __restrict__ cam_l,
          const double2* __restrict__ J, int64_t pad, const double* __restrict__ tin,
          const double* __restrict__ bl, const double* __restrict__ Vinv, double* __restrict__ out,
          int* __restrict__ nonzero_flag, const SeriesState* __restrict__ st, int check_stop) {
  __shared__ double red[kTile][3];
  if (check_stop && st->stopped) return;
  const int lm = long_lm[blockIdx.x];
  const int o0 = lm_off[lm], o1 = lm_off[lm + 1];
  const int tid = threadIdx.x;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0;
  for (int o = o0 + tid; o < o1; o += kTile) {
    const double* tv = tin + (int64_t)cam_l[o] * 9;
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const double2 v = J[j * pad + o];
      u0 = fma(v.x, tv[j], u0);
      u1 = fma(v.y, tv[j], u1);
    }
    const double2 a = J[9 * pad + o], b = J[10 * pad + o], c = J[11 * pad + o];
    y0 += fma(a.x, u0, a.y * u1);
    y1 += fma(b.x, u0, b.y * u1);
    y2 += fma(c.x, u0, c.y * u1);
  }
  red[tid][0] = y0;
  red[tid][1] = y1;
  red[tid][2] = y2;
  __syncthreads();
  for (int s = kTile / 2; s; s >>= 1) {
    if (tid < s)
      for (int k = 0; k < 3; ++k) red[tid][k] += red[tid + s][k];
    __syncthreads();
  }
  if (tid == 0) {
    double y[3] = {red[0][0], red[0][1], red[0][2]}, z[3];
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
                         double* __restrict__ out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_cam * 9) return;
  const int64_t c = q / 9;
  const int i = (int)(q - c * 9);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 9; ++j) s = fma(M45[c * 45 + sym9(i, j)], v[c * 9 + j], s);
  out[q] = s;
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

size_t term_smem(const Ctx& c) {
  return (size_t)c.max_slots * 9 * 8 + kTile * 9 * 8 + kTile * 3 * 8 * 2 + kTile + kTile * 4;
}

int configure_term(Ctx& c) {
  (void)c;
  static thread_local int done_dev = -1;
  int dev = 0;
  PCK(cudaGetDevice(&dev));
  if (done_dev != dev) {
    PCK(cudaFuncSetAttribute(k_term<kModeTerm>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    PCK(cudaFuncSetAttribute(k_term<kModeBt>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    PCK(cudaFuncSetAttribute(k_term<kModeW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    done_dev = dev;
  }
  return POBA_OK;
}

TermArgs term_args(Ctx& c, const double* tin, const double* lvec, bool check_stop) {
  TermArgs a;
  a.tiles = c.tiles.as<Tile>();
  a.chunks = c.chunks.as<Chunk>();
  a.cam_l = c.cam_l.as<int>();
  a.perm = c.perm.as<uint8_t>();
  a.seg_start = c.seg_start.as<uint16_t>();
  a.seg_slot = c.seg_slot.as<uint16_t>();
  a.J = c.J.as<double2>();
  a.pad = c.obs_pad;
  a.tin = tin;
  a.lvec = lvec;
  a.Vinv = c.Vinv.as<double>();
  a.zlong = c.ltmp.as<double>();
  a.partials = c.partials.as<double>();
  a.st = c.state.as<SeriesState>();
  a.max_slots = c.max_slots;
  a.check_stop = check_stop ? 1 : 0;
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
  return a;
}

int launch_term(Ctx& c, int mode, const double* tin, const double* lvec, bool check_stop) {
  PTRY(configure_term(c));
  const TermArgs a = term_args(c, tin, lvec, check_stop);
  const size_t smem = term_smem(c);
  if (mode == kModeTerm) {
    if (c.n_long) {
      k_wt_long<kOutZ><<<c.n_long, kTile, 0, c.stream>>>(
          c.long_lm.as<int>(), c.lm_off.as<int>(), c.cam_l.as<int>(), c.J.as<double2>(), c.obs_pad, tin, nullptr,
          c.Vinv.as<double>(), c.ltmp.as<double>(), nullptr, c.state.as<SeriesState>(), check_stop ? 1 : 0);
      c.launches++;
    }
    k_term<kModeTerm><<<c.n_chunks, kTile, smem, c.stream>>>(a);
  } else if (mode == kModeBt) {
    k_term<kModeBt><<<c.n_chunks, kTile, smem, c.stream>>>(a);
  } else {
    k_term<kModeW><<<c.n_chunks, kTile, smem, c.stream>>>(a);
  }
  c.launches++;
  PCK(cudaGetLastError());
  return POBA_OK;
}

// camera step after a term kernel: merge (+ all-reduce when sharded) + finalize
int launch_cam(Ctx& c, int mode, int order, double eps, bool check_stop, const CamArgs* override_args = nullptr) {
  const unsigned nb = grid_for(c.n_cam, 8);
  CamArgs a = override_args ? *override_args : cam_args(c, order, eps, check_stop);
  if (c.nranks == 1) {
    if (mode == kCamTerm) k_cam<kCamTerm, true><<<nb, 256, 0, c.stream>>>(a);
    else if (mode == kCamBt) k_cam<kCamBt, true><<<nb, 256, 0, c.stream>>>(a);
    else k_cam<kCamMerge, true><<<nb, 256, 0, c.stream>>>(a);
    c.launches++;
  } else {
    k_cam<kCamMerge, true><<<nb, 256, 0, c.stream>>>(a);
    c.launches++;
    PTRY(allreduce_sum(c, c.rvec.as<double>(), c.n_cam * 9));
    if (mode == kCamTerm) {
      k_cam<kCamTerm, false><<<nb, 256, 0, c.stream>>>(a);
      c.launches++;
    } else if (mode == kCamBt) {
      k_cam<kCamBt, false><<<nb, 256, 0, c.stream>>>(a);
      c.launches++;
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
    PNCCL(AllReduce(c.scratch_b.p, c.scratch_b.p, 1, ncclFloat64, ncclMax, c.comm, s));
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

int series_device(Ctx& c, double eps, int max_order, bool forced, int* order_used, int* converged) {
  cudaStream_t s = c.stream;
  PTRY(ensure_ratios(c, max_order));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  k_fill<<<grid_for(max_order + 1, 128), 128, 0, s>>>(c.ratios.as<double>(), max_order + 1,
                                                     std::numeric_limits<double>::quiet_NaN());
  c.launches++;
  // order 0: b_tilde and t0
  PTRY(launch_term(c, kModeBt, nullptr, c.bl.as<double>(), false));
  PTRY(launch_cam(c, kCamBt, 0, eps, false));
  for (int i = 1; i <= max_order; ++i) {
    PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, true));
    PTRY(launch_cam(c, kCamTerm, i, eps, !forced));
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
  k_cam_mv<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.Uinv.as<double>(), d_v, c.n_cam, c.tvec.as<double>());
  PCK(cudaMemcpyAsync(c.xvec.p, c.tvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, s));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  c.launches++;
  for (int i = 1; i <= order; ++i) {
    PTRY(launch_term(c, kModeTerm, c.tvec.as<double>(), nullptr, false));
    PTRY(launch_cam(c, kCamTerm, i, 1.0, false));
  }
  PCK(cudaMemcpyAsync(d_out, c.xvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, s));
  PCK(cudaStreamSynchronize(s));
  c.have_solution = false;
  return POBA_OK;
}

int back_substitute_device(Ctx& c, const double* d_dp, int* nonzero) {
  cudaStream_t s = c.stream;
  int* fl = c.flag.as<int>() + 1;
  PCK(cudaMemsetAsync(fl, 0, 4, s));
  k_wt_tile<kOutBack><<<c.n_tiles, kTile, 0, s>>>(c.tiles.as<Tile>(), c.cam_l.as<int>(), c.J.as<double2>(), c.obs_pad,
                                                  d_dp, c.bl.as<double>(), c.Vinv.as<double>(), c.dl.as<double>(), fl);
  c.launches++;
  if (c.n_long) {
    k_wt_long<kOutBack><<<c.n_long, kTile, 0, s>>>(c.long_lm.as<int>(), c.lm_off.as<int>(), c.cam_l.as<int>(),
                                                   c.J.as<double2>(), c.obs_pad, d_dp, c.bl.as<double>(),
                                                   c.Vinv.as<double>(), c.dl.as<double>(), fl,
                                                   c.state.as<SeriesState>(), 0);
    c.launches++;
  }
  PCK(cudaGetLastError());
  int h = 0;
  PCK(cudaMemcpyAsync(&h, fl, 4, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (c.nranks > 1) {
    double v = (double)h, out = 0;
    PTRY(c.scratch_b.alloc(8));
    PCK(cudaMemcpyAsync(c.scratch_b.p, &v, 8, cudaMemcpyHostToDevice, s));
    PNCCL(AllReduce(c.scratch_b.p, c.scratch_b.p, 1, ncclFloat64, ncclMax, c.comm, s));
    PCK(cudaMemcpyAsync(&out, c.scratch_b.p, 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    h = (int)out;
  }
  *nonzero = h;
  c.have_delta_l = true;
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
    case POBA_OP_WT:
      k_wt_tile<kOutWt><<<c.n_tiles, kTile, 0, s>>>(c.tiles.as<Tile>(), c.cam_l.as<int>(), c.J.as<double2>(),
                                                    c.obs_pad, d_in, nullptr, nullptr, d_out, nullptr);
      c.launches++;
      if (c.n_long) {
        k_wt_long<kOutWt><<<c.n_long, kTile, 0, s>>>(c.long_lm.as<int>(), c.lm_off.as<int>(), c.cam_l.as<int>(),
                                                     c.J.as<double2>(), c.obs_pad, d_in, nullptr, nullptr, d_out,
                                                     nullptr, c.state.as<SeriesState>(), 0);
        c.launches++;
      }
      break;
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
