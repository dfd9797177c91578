// K1-K3 and K8: residual + analytic Jacobian, the landmark-major store, the
// V0/b_l and U0/b_p reductions, Marquardt diagonals, and the cost.
//
// Reference (paths relative to /root/reference/pkg/src/powerba/):
//   camera.evaluate            camera.py:67-135  (projection, residual, J_pose, J_point)
//   camera.rotation_matrices   camera.py:49-51   (scipy from_rotvec().as_matrix())
//   blocks.linearize           blocks.py:293-324 (store rows in canonical order)
//   blocks._finish_linearization blocks.py:375-402 (U0, V0, b_p, b_l, D clamp)
//   blocks.assemble_from_observations blocks.py:333-352
//   lm.residual_cost           lm.py:107-119
//
// All reductions are in fp64 and in a fixed order (no floating-point
// atomics), so every result is bitwise reproducible run to run.
#include "poba_internal.h"

namespace poba {

namespace {

#ifndef POBA_LIN_COOP_PREP
#define POBA_LIN_COOP_PREP 1
#endif
constexpr int kLinRec = 9;  // double2 per staged camera record (8 used; 144-B stride)
constexpr int kLinRecSmem = kBlockTiles * kTile * kLinRec * 16;


constexpr double kMinDepth = 1e-12;   // camera.py:22
constexpr double kClampLo = 1e-6;     // blocks.py:36
constexpr double kClampHi = 1e6;      // blocks.py:37
// 54 fp64 accumulators per lane (~160 registers): small blocks so that three
// fit an SM instead of one
#ifndef POBA_CAM_REDUCE_THREADS
#define POBA_CAM_REDUCE_THREADS 128
#endif
constexpr int kCamReduceThreads = POBA_CAM_REDUCE_THREADS;
// blocks per SM the camera-major reduce is compiled for: 2 keeps all 54
// accumulators + the prefetched operands in registers (252, no spills); 3 and 4
// spill and measured slower (profiles/r02a_linearize_ab.md)
#ifndef POBA_CAM_REDUCE_BLOCKS
#define POBA_CAM_REDUCE_BLOCKS 2
#endif
// tile pass shape: warp-tiles per block x blocks per SM the kernel is compiled for
#ifndef POBA_LIN_TILES
#define POBA_LIN_TILES 8
#endif
#ifndef POBA_LIN_TILE_BLOCKS
#define POBA_LIN_TILE_BLOCKS 2  // 8 x 3 (80 registers, spills) measured slower
#endif
#ifndef POBA_LIN_PIPE_BLOCKS
#define POBA_LIN_PIPE_BLOCKS 3  // blocks of 4 warps per SM the pipelined tile pass is compiled for
#endif
constexpr int kLinTiles = POBA_LIN_TILES;
constexpr int kLinTileSmem = kLinTiles * kTile * kLinRec * 16;

// Rotation matrix of an axis-angle vector through the unit quaternion, the
// same construction scipy uses (from_rotvec -> as_matrix).
__device__ void rotvec_to_matrix(double wx, double wy, double wz, double* R) {
  const double a2 = wx * wx + wy * wy + wz * wz;
  const double angle = sqrt(a2);
  double scale;
  if (angle <= 1e-3) {
    scale = 0.5 - a2 / 48.0 + a2 * a2 / 3840.0;
  } else {
    scale = sin(angle / 2.0) / angle;
  }
  const double x = wx * scale, y = wy * scale, z = wz * scale, w = cos(angle / 2.0);
  const double x2 = x * x, y2 = y * y, z2 = z * z, w2 = w * w;
  const double xy = x * y, zw = z * w, xz = x * z, yw = y * w, yz = y * z, xw = x * w;
  R[0] = x2 - y2 - z2 + w2;
  R[1] = 2.0 * (xy - zw);
  R[2] = 2.0 * (xz + yw);
  R[3] = 2.0 * (xy + zw);
  R[4] = -x2 + y2 - z2 + w2;
  R[5] = 2.0 * (yz - xw);
  R[6] = 2.0 * (xz - yw);
  R[7] = 2.0 * (yz + xw);
  R[8] = -x2 - y2 + z2 + w2;
}

__global__ void k_cam_prep(const double* __restrict__ cams, int64_t n_cam, double* __restrict__ prep) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cam) return;
  const double* q = cams + c * 9;
  double* o = prep + c * 16;
  double R[9];
  rotvec_to_matrix(q[0], q[1], q[2], R);
#pragma unroll
  for (int i = 0; i < 9; ++i) o[i] = R[i];
#pragma unroll
  for (int i = 3; i < 9; ++i) o[i + 6] = q[i];
  o[15] = 0.0;
}

struct ObsModel {
  double r0, r1;
  double jp0[9], jp1[9];  // J_pose rows
  double jl0[3], jl1[3];  // J_point rows
  bool valid;
};

// a camera's prepared record (R, t, f, k1, k2, pad): eight 16-B loads
__device__ __forceinline__ void load_prep(const double* __restrict__ prep, int cam, double* cp) {
  const double2* src = reinterpret_cast<const double2*>(prep + (int64_t)cam * 16);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = __ldg(src + k);
    cp[2 * k] = v.x;
    cp[2 * k + 1] = v.y;
  }
}

// camera.evaluate for one observation (camera.py:85-135)
template <bool kJac>
__device__ __forceinline__ void evaluate_obs(const double* __restrict__ cp, double X0, double X1, double X2,
                                             double2 pix, ObsModel& m) {
  const double* R = cp;
  const double P0 = R[0] * X0 + R[1] * X1 + R[2] * X2 + cp[9];
  const double P1 = R[3] * X0 + R[4] * X1 + R[5] * X2 + cp[10];
  const double P2 = R[6] * X0 + R[7] * X1 + R[8] * X2 + cp[11];
  const double f = cp[12], k1 = cp[13], k2 = cp[14];
  m.valid = fabs(P2) >= kMinDepth;
  const double zs = m.valid ? P2 : 1.0;
  const double p0 = -P0 / zs, p1 = -P1 / zs;
  const double s = p0 * p0 + p1 * p1;
  const double d = 1.0 + s * (k1 + k2 * s);
  const double fd = f * d;
  m.r0 = m.valid ? fd * p0 - pix.x : 0.0;
  m.r1 = m.valid ? fd * p1 - pix.y : 0.0;
  if (!kJac) return;
  if (!m.valid) {
#pragma unroll
    for (int j = 0; j < 9; ++j) m.jp0[j] = m.jp1[j] = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) m.jl0[j] = m.jl1[j] = 0.0;
    return;
  }
  const double iz = 1.0 / zs;
  // dp/dP = [[-iz, 0, P0 iz^2], [0, -iz, P1 iz^2]]
  const double e02 = P0 * iz * iz, e12 = P1 * iz * iz;
  // dproj/dp = f (d I + p g^T), g = (2 k1 + 4 k2 s) p
  const double gs = 2.0 * k1 + 4.0 * k2 * s;
  const double g0 = gs * p0, g1 = gs * p1;
  const double a00 = f * (d + p0 * g0), a01 = f * (p0 * g1);
  const double a10 = f * (p1 * g0), a11 = f * (d + p1 * g1);
  // A = dproj/dp @ dp/dP  (2x3)
  const double A00 = -a00 * iz, A01 = -a01 * iz, A02 = a00 * e02 + a01 * e12;
  const double A10 = -a10 * iz, A11 = -a11 * iz, A12 = a10 * e02 + a11 * e12;
  // J_point = A R
  m.jl0[0] = A00 * R[0] + A01 * R[3] + A02 * R[6];
  m.jl0[1] = A00 * R[1] + A01 * R[4] + A02 * R[7];
  m.jl0[2] = A00 * R[2] + A01 * R[5] + A02 * R[8];
  m.jl1[0] = A10 * R[0] + A11 * R[3] + A12 * R[6];
  m.jl1[1] = A10 * R[1] + A11 * R[4] + A12 * R[7];
  m.jl1[2] = A10 * R[2] + A11 * R[5] + A12 * R[8];
  // rotation (right increment): A (-R [X]x) = -(A R) [X]x
  m.jp0[0] = -(m.jl0[1] * X2 - m.jl0[2] * X1);
  m.jp0[1] = -(m.jl0[2] * X0 - m.jl0[0] * X2);
  m.jp0[2] = -(m.jl0[0] * X1 - m.jl0[1] * X0);
  m.jp1[0] = -(m.jl1[1] * X2 - m.jl1[2] * X1);
  m.jp1[1] = -(m.jl1[2] * X0 - m.jl1[0] * X2);
  m.jp1[2] = -(m.jl1[0] * X1 - m.jl1[1] * X0);
  m.jp0[3] = A00; m.jp0[4] = A01; m.jp0[5] = A02;
  m.jp1[3] = A10; m.jp1[4] = A11; m.jp1[5] = A12;
  m.jp0[6] = d * p0;  m.jp1[6] = d * p1;
  const double fs = f * s;
  m.jp0[7] = fs * p0; m.jp1[7] = fs * p1;
  m.jp0[8] = fs * s * p0; m.jp1[8] = fs * s * p1;
}

// A tile's 32 camera records (128 B each) gathered cooperatively, four records
// per 16-B load instruction, through the warp's shared stage (144-B stride:
// conflict-free 16-B reads by consecutive lanes) -- instead of every lane
// walking its own record with eight uncoalesced loads.
__device__ __forceinline__ void gather_prep(const double* __restrict__ prep, int my_cam, int n, int lane,
                                            double2* __restrict__ pst, double* __restrict__ cp) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int r = 4 * k + (lane >> 3), piece = lane & 7;
    const int cam = __shfl_sync(0xffffffffu, my_cam, r);
    if (r < n) pst[r * 9 + piece] = __ldg(reinterpret_cast<const double2*>(prep + (int64_t)cam * 16) + piece);
  }
  __syncwarp();
  if (lane < n) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 v = pst[lane * 9 + k];
      cp[2 * k] = v.x;
      cp[2 * k + 1] = v.y;
    }
  }
}

// Store rows + per-observation V0/b_l contributions + per-landmark sums; one
// warp per warp-tile, each landmark's observations in camera order (np.add.at's
// sequential fold of blocks.py:394,396 runs over the same observations in the
// same order).
template <bool kExplicit, bool F32>
__global__ void __launch_bounds__(kLinTiles * kTile, POBA_LIN_TILE_BLOCKS)
k_lin_tile(const Tile* __restrict__ tiles, int tile0, int tile_end, const int* __restrict__ cam_s,
           const int* __restrict__ file_s, const double2* __restrict__ pix_s, const uint8_t* __restrict__ lidx_s,
           const double* __restrict__ prep, const double* __restrict__ points, const double* __restrict__ ejp,
           const double* __restrict__ ejl, const double* __restrict__ eres, void* __restrict__ J,
           double2* __restrict__ Rz, double* __restrict__ V0, double* __restrict__ bl, double* __restrict__ Dl,
           unsigned long long* __restrict__ n_invalid) {
  __shared__ double contrib_all[kLinTiles][kTile * 9];
  __shared__ int lstart_all[kLinTiles][kTile + 1];
  // per warp: the tile's 32 camera records, staged for the cooperative gather
  extern __shared__ __align__(16) double2 lin_rec[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ti = tile0 + blockIdx.x * kLinTiles + w;
  if (ti >= tile_end) return;  // warps are independent: no block-wide barrier below
  double* contrib = contrib_all[w];
  int* lstart = lstart_all[w];
  const int64_t o = (int64_t)ti * kTile + lane;
  // per-slot loads first, all independent of the tile descriptor (slot arrays
  // cover the padding too), so their latencies overlap
  const int cam_o = cam_s[o];
  const int li_o = lidx_s[o];
  double2 pix = make_double2(0.0, 0.0);
  if (!kExplicit) pix = __ldcs(pix_s + o);  // streamed once; the slot array covers the padding
  const Tile t = tiles[ti];
  const bool is_long = t.flags & kTileLong;
  bool bad = false;
  double cp[16];  // this observation's camera record (R, t, f, k1, k2, pad)
  double X0 = 0.0, X1 = 0.0, X2 = 0.0;
  if (!kExplicit && lane < t.n) {  // point loads in flight during the camera gather
    const double* X = points + (int64_t)(t.lm0 + (is_long ? 0 : li_o)) * 3;
    X0 = X[0];
    X1 = X[1];
    X2 = X[2];
  }
  if (!kExplicit) {
    const int my_cam = lane < t.n ? cam_o : 0;
#if POBA_LIN_COOP_PREP
    gather_prep(prep, my_cam, t.n, lane, lin_rec + w * kTile * kLinRec, cp);
#else
    if (lane < t.n) load_prep(prep, my_cam, cp);
#endif
  }
  if (lane < t.n) {
    ObsModel m;
    if (kExplicit) {
      const int64_t f = file_s[o];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        m.jp0[j] = ejp[f * 18 + j];
        m.jp1[j] = ejp[f * 18 + 9 + j];
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        m.jl0[j] = ejl[f * 6 + j];
        m.jl1[j] = ejl[f * 6 + 3 + j];
      }
      m.r0 = eres[f * 2];
      m.r1 = eres[f * 2 + 1];
      m.valid = true;
    } else {
      evaluate_obs<true>(cp, X0, X1, X2, pix, m);
      bad = !m.valid;
    }
    // at precision 32 every stored value is rounded to fp32 first and all
    // sums below use the rounded values, as the reference's float32 storage
    // feeds its float64 einsums (blocks.py:316-320, 387-396)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      m.jp0[j] = stored<F32>(m.jp0[j]);
      m.jp1[j] = stored<F32>(m.jp1[j]);
      jstore<F32>(J, o, j, m.jp0[j], m.jp1[j]);  // plane j: coalesced
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      m.jl0[b] = stored<F32>(m.jl0[b]);
      m.jl1[b] = stored<F32>(m.jl1[b]);
      jstore<F32>(J, o, 9 + b, m.jl0[b], m.jl1[b]);
    }
    m.r0 = stored<F32>(m.r0);
    m.r1 = stored<F32>(m.r1);
    Rz[o] = make_double2(m.r0, m.r1);
    double* cc = contrib + lane * 9;
    cc[0] = m.jl0[0] * m.jl0[0] + m.jl1[0] * m.jl1[0];
    cc[1] = m.jl0[0] * m.jl0[1] + m.jl1[0] * m.jl1[1];
    cc[2] = m.jl0[0] * m.jl0[2] + m.jl1[0] * m.jl1[2];
    cc[3] = m.jl0[1] * m.jl0[1] + m.jl1[1] * m.jl1[1];
    cc[4] = m.jl0[1] * m.jl0[2] + m.jl1[1] * m.jl1[2];
    cc[5] = m.jl0[2] * m.jl0[2] + m.jl1[2] * m.jl1[2];
    cc[6] = m.jl0[0] * m.r0 + m.jl1[0] * m.r1;
    cc[7] = m.jl0[1] * m.r0 + m.jl1[1] * m.r1;
    cc[8] = m.jl0[2] * m.r0 + m.jl1[2] * m.r1;
    if (!is_long) {
      const int li = li_o;
      if (lane == 0 || lidx_s[o - 1] != li) lstart[li] = lane;
    }
  }
  if (lane == 0) lstart[t.nlm] = t.n;
  __syncwarp();
  const unsigned nbad = __popc(__ballot_sync(0xffffffffu, bad));
  if (lane == 0 && nbad) atomicAdd(n_invalid, (unsigned long long)nbad);
  __syncwarp();
  if (is_long) return;  // long landmarks are reduced by k_lin_long
  for (int q = lane; q < t.nlm * 9; q += kTile) {
    const int j = q / 9, comp = q - j * 9;
    double acc = 0.0;
    for (int r = lstart[j]; r < lstart[j + 1]; ++r) acc += contrib[r * 9 + comp];
    const int lm = t.lm0 + j;
    if (comp < 6) V0[(int64_t)lm * 6 + comp] = acc; else bl[(int64_t)lm * 3 + comp - 6] = acc;
    if (comp == 0 || comp == 3 || comp == 5) {
      const double c2 = fmin(fmax(acc, kClampLo * kClampLo), kClampHi * kClampHi);
      Dl[(int64_t)lm * 3 + (comp == 0 ? 0 : comp == 3 ? 1 : 2)] = sqrt(c2);
    }
  }
}

// ---------------------------------------------------------------------------
// Software-pipelined tile pass (state path).  Same arithmetic as k_lin_tile,
// but the warps are persistent and keep two tiles of loads in flight behind
// the tile they compute: at tile i a warp issues the per-slot loads (camera,
// landmark index, pixel) and the descriptor of tile i + 2, then -- with tile
// i + 1's of those now landed -- that tile's point loads and its 32 camera
// records (cp.async, 16 B x 8 per lane, into the other half of a two-deep
// shared stage), and only then evaluates tile i.  k_lin_tile's warp waits two
// dependent load waves per tile; this one waits none in steady state.
// ---------------------------------------------------------------------------
constexpr int kPipeWarps = 4;                       // warps per block
constexpr int kPipeRecBytes = kTile * kLinRec * 16;  // one tile's staged camera records (4608 B)
constexpr int kPipeSmem = kPipeWarps * 2 * kPipeRecBytes;

struct LinW1 {  // first load wave of a tile: per-slot values + descriptor
  int cam, li;
  double2 pix;
  Tile t;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <bool F32>
__global__ void __launch_bounds__(kPipeWarps * kTile, POBA_LIN_PIPE_BLOCKS)
k_lin_tile_pipe(const Tile* __restrict__ tiles, int tile0, int tile_end, const int* __restrict__ cam_s,
                const double2* __restrict__ pix_s, const uint8_t* __restrict__ lidx_s,
                const double* __restrict__ prep, const double* __restrict__ points, void* __restrict__ J,
                double2* __restrict__ Rz, double* __restrict__ V0, double* __restrict__ bl, double* __restrict__ Dl,
                unsigned long long* __restrict__ n_invalid) {
  __shared__ double contrib_all[kPipeWarps][kTile * 9];
  __shared__ int lstart_all[kPipeWarps][kTile + 1];
  extern __shared__ __align__(16) double2 pipe_rec[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = gridDim.x * kPipeWarps;
  int ti = tile0 + blockIdx.x * kPipeWarps + w;  // consecutive warps take consecutive tiles
  if (ti >= tile_end) return;                   // warps are independent: no block-wide barrier below
  double* contrib = contrib_all[w];
  int* lstart = lstart_all[w];
  double2* const stage0 = pipe_rec + (w * 2) * kTile * kLinRec;  // two-deep record stage of this warp
  auto stage = [&](int h) { return stage0 + h * kTile * kLinRec; };

  auto wave1 = [&](int tj, LinW1& r) {  // clamped past the end: loads stay in range, the results unused
    const int tt = min(tj, tile_end - 1);
    const int64_t o = (int64_t)tt * kTile + lane;
    r.cam = cam_s[o];
    r.li = lidx_s[o];
    r.pix = __ldcs(pix_s + o);
    r.t = tiles[tt];
  };
  auto wave2 = [&](const LinW1& r, double2* pst, double& X0, double& X1, double& X2) {
    X0 = X1 = X2 = 0.0;
    if (lane < r.t.n) {
      const double* X = points + (int64_t)(r.t.lm0 + ((r.t.flags & kTileLong) ? 0 : r.li)) * 3;
      X0 = X[0];
      X1 = X[1];
      X2 = X[2];
    }
    const int my_cam = lane < r.t.n ? r.cam : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int rr = 4 * k + (lane >> 3), piece = lane & 7;
      const int cam = __shfl_sync(0xffffffffu, my_cam, rr);
      if (rr < r.t.n) cp_async16(pst + rr * 9 + piece, reinterpret_cast<const double2*>(prep + (int64_t)cam * 16) + piece);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  LinW1 a, b, c;
  double XA0, XA1, XA2, XB0 = 0.0, XB1 = 0.0, XB2 = 0.0;
  wave1(ti, a);
  wave1(ti + stride, b);
  wave2(a, stage(0), XA0, XA1, XA2);
  int buf = 0;
  for (; ti < tile_end; ti += stride) {
    wave1(ti + 2 * stride, c);
    const bool has_next = ti + stride < tile_end;
    if (has_next) wave2(b, stage(buf ^ 1), XB0, XB1, XB2);
    else asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count uniform
    asm volatile("cp.async.wait_group 1;" ::: "memory");       // tile i's records have landed
    __syncwarp();
    const Tile t = a.t;
    const int64_t o = (int64_t)ti * kTile + lane;
    const bool is_long = t.flags & kTileLong;
    const int prev_li = __shfl_up_sync(0xffffffffu, a.li, 1);
    bool bad = false;
    if (lane < t.n) {
      double cp[16];
      const double2* pst = stage(buf);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double2 v = pst[lane * 9 + k];
        cp[2 * k] = v.x;
        cp[2 * k + 1] = v.y;
      }
      ObsModel m;
      evaluate_obs<true>(cp, XA0, XA1, XA2, a.pix, m);
      bad = !m.valid;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        m.jp0[j] = stored<F32>(m.jp0[j]);
        m.jp1[j] = stored<F32>(m.jp1[j]);
        jstore<F32>(J, o, j, m.jp0[j], m.jp1[j]);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        m.jl0[q] = stored<F32>(m.jl0[q]);
        m.jl1[q] = stored<F32>(m.jl1[q]);
        jstore<F32>(J, o, 9 + q, m.jl0[q], m.jl1[q]);
      }
      m.r0 = stored<F32>(m.r0);
      m.r1 = stored<F32>(m.r1);
      Rz[o] = make_double2(m.r0, m.r1);
      double* cc = contrib + lane * 9;
      cc[0] = m.jl0[0] * m.jl0[0] + m.jl1[0] * m.jl1[0];
      cc[1] = m.jl0[0] * m.jl0[1] + m.jl1[0] * m.jl1[1];
      cc[2] = m.jl0[0] * m.jl0[2] + m.jl1[0] * m.jl1[2];
      cc[3] = m.jl0[1] * m.jl0[1] + m.jl1[1] * m.jl1[1];
      cc[4] = m.jl0[1] * m.jl0[2] + m.jl1[1] * m.jl1[2];
      cc[5] = m.jl0[2] * m.jl0[2] + m.jl1[2] * m.jl1[2];
      cc[6] = m.jl0[0] * m.r0 + m.jl1[0] * m.r1;
      cc[7] = m.jl0[1] * m.r0 + m.jl1[1] * m.r1;
      cc[8] = m.jl0[2] * m.r0 + m.jl1[2] * m.r1;
      if (!is_long && (lane == 0 || prev_li != a.li)) lstart[a.li] = lane;
    }
    if (lane == 0) lstart[t.nlm] = t.n;
    __syncwarp();
    const unsigned nbad = __popc(__ballot_sync(0xffffffffu, bad));
    if (lane == 0 && nbad) atomicAdd(n_invalid, (unsigned long long)nbad);
    if (!is_long) {  // long landmarks are reduced by k_lin_long
      for (int q = lane; q < t.nlm * 9; q += kTile) {
        const int j = q / 9, comp = q - j * 9;
        double acc = 0.0;
        for (int r = lstart[j]; r < lstart[j + 1]; ++r) acc += contrib[r * 9 + comp];
        const int lm = t.lm0 + j;
        if (comp < 6) V0[(int64_t)lm * 6 + comp] = acc; else bl[(int64_t)lm * 3 + comp - 6] = acc;
        if (comp == 0 || comp == 3 || comp == 5) {
          const double c2 = fmin(fmax(acc, kClampLo * kClampLo), kClampHi * kClampHi);
          Dl[(int64_t)lm * 3 + (comp == 0 ? 0 : comp == 3 ? 1 : 2)] = sqrt(c2);
        }
      }
    }
    __syncwarp();  // contrib / lstart / this stage half are reused by the next tiles
    a = b;
    b = c;
    XA0 = XB0;
    XA1 = XB1;
    XA2 = XB2;
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// V0/b_l of landmarks longer than a tile, straight from the stored rows: one
// warp per landmark, lanes stride its observations (each lane folds its own in
// order), fixed-shape butterfly across lanes
template <bool F32>
__global__ void k_lin_long(const int* __restrict__ long_lm, const int* __restrict__ lm_slot0,
                           const int* __restrict__ lm_k, const void* __restrict__ J,
                           const double2* __restrict__ Rz, int64_t pad, double* __restrict__ V0,
                           double* __restrict__ bl, double* __restrict__ Dl) {
  const int lm = long_lm[blockIdx.x];
  const int o0 = lm_slot0[lm], o1 = o0 + lm_k[lm];
  const int lane = threadIdx.x;  // 32 threads
  double acc[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int o = o0 + lane; o < o1; o += 32) {
    const double2 a = jload<F32>(J, o, 9), b = jload<F32>(J, o, 10), c = jload<F32>(J, o, 11);
    const double2 r = Rz[o];
    acc[0] += a.x * a.x + a.y * a.y;
    acc[1] += a.x * b.x + a.y * b.y;
    acc[2] += a.x * c.x + a.y * c.y;
    acc[3] += b.x * b.x + b.y * b.y;
    acc[4] += b.x * c.x + b.y * c.y;
    acc[5] += c.x * c.x + c.y * c.y;
    acc[6] += a.x * r.x + a.y * r.y;
    acc[7] += b.x * r.x + b.y * r.y;
    acc[8] += c.x * r.x + c.y * r.y;
  }
#pragma unroll
  for (int q = 0; q < 9; ++q)
#pragma unroll
    for (int s = 16; s; s >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], s);
  if (lane == 0) {
#pragma unroll
    for (int comp = 0; comp < 9; ++comp) {
      if (comp < 6) V0[(int64_t)lm * 6 + comp] = acc[comp]; else bl[(int64_t)lm * 3 + comp - 6] = acc[comp];
      if (comp == 0 || comp == 3 || comp == 5) {
        const double c2 = fmin(fmax(acc[comp], kClampLo * kClampLo), kClampHi * kClampHi);
        Dl[(int64_t)lm * 3 + (comp == 0 ? 0 : comp == 3 ? 1 : 2)] = sqrt(c2);
      }
    }
  }
}


// U0 (packed upper 45) and b_p (9) partial sums over chunks of <= kCamChunk
// observations of one camera, walked in camera-major order; fixed
// warp-butterfly reduction.  Each observation's J_p and residual are
// RECOMPUTED here from the camera record (one per warp), the landmark's point
// and the pixel -- the same evaluate_obs (and fp32 rounding at precision 32)
// that produced the stored rows -- instead of being written camera-major by
// the tile pass and read back (160 B per observation each way).
template <bool kExplicit, bool F32>
__global__ void __launch_bounds__(kCamReduceThreads, POBA_CAM_REDUCE_BLOCKS)
k_cam_chunk_reduce(const int* __restrict__ cc_cam_off, const int* __restrict__ cc_cam, const int* __restrict__ cam_start,
                   int n_cc, const double* __restrict__ prep, const double* __restrict__ points,
                   const int* __restrict__ lm_c, const double2* __restrict__ pix_c, const int* __restrict__ file_c,
                   const double* __restrict__ ejp, const double* __restrict__ eres, double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_cc) return;
  const int cam = cc_cam[warp];
  const int p0 = cam_start[cam] + (warp - cc_cam_off[cam]) * kCamChunk;
  const int p1 = min(p0 + kCamChunk, cam_start[cam + 1]);
  double cp[16];
  if (!kExplicit) load_prep(prep, cam, cp);
  double acc[54];
#pragma unroll
  for (int q = 0; q < 54; ++q) acc[q] = 0.0;
  // software pipeline over this lane's observations: the landmark index is
  // loaded two steps ahead and the point + pixel one step ahead, so the two
  // dependent load latencies overlap a whole step of arithmetic
  double nX0 = 0.0, nX1 = 0.0, nX2 = 0.0;
  double2 npx = make_double2(0.0, 0.0);
  int lm_n2 = 0;
  if (!kExplicit) {
    const int pf = p0 + lane;
    if (pf < p1) {
      const int64_t lm = lm_c[pf];
      nX0 = points[lm * 3];
      nX1 = points[lm * 3 + 1];
      nX2 = points[lm * 3 + 2];
      npx = __ldcs(pix_c + pf);
    }
    if (pf + 32 < p1) lm_n2 = lm_c[pf + 32];
  }
  for (int p = p0 + lane; p < p1; p += 32) {
    ObsModel m;
    if (kExplicit) {
      const int64_t f = file_c[p];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        m.jp0[j] = ejp[f * 18 + j];
        m.jp1[j] = ejp[f * 18 + 9 + j];
      }
      m.r0 = eres[f * 2];
      m.r1 = eres[f * 2 + 1];
    } else {
      const double X0 = nX0, X1 = nX1, X2 = nX2;
      const double2 px = npx;
      if (p + 32 < p1) {
        const int64_t lm = lm_n2;
        nX0 = points[lm * 3];
        nX1 = points[lm * 3 + 1];
        nX2 = points[lm * 3 + 2];
        npx = __ldcs(pix_c + p + 32);
      }
      if (p + 64 < p1) lm_n2 = lm_c[p + 64];
      evaluate_obs<true>(cp, X0, X1, X2, px, m);
    }
    double a[9], b[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      a[j] = stored<F32>(m.jp0[j]);
      b[j] = stored<F32>(m.jp1[j]);
    }
    const double r0 = stored<F32>(m.r0), r1 = stored<F32>(m.r1);
    int q = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) acc[q++] += a[i] * a[j] + b[i] * b[j];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[45 + i] += a[i] * r0 + b[i] * r1;
  }
#pragma unroll
  for (int q = 0; q < 54; ++q) {
    double v = acc[q];
#pragma unroll
    for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    acc[q] = v;
  }
  double* dst = out + (int64_t)warp * 54;
#pragma unroll
  for (int q = 0; q < 54; ++q)
    if ((q & 31) == lane) dst[q] = acc[q];
}

// per camera: sum its chunk partials in chunk order -> U0 packed, b_p
__global__ void k_cam_merge54(const int* __restrict__ cc_cam_off, const double* __restrict__ part, int n_cam,
                              double* __restrict__ U0, double* __restrict__ bp) {
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cam >= n_cam) return;
  const int c0 = cc_cam_off[cam], c1 = cc_cam_off[cam + 1];
  for (int q = lane; q < 54; q += 32) {
    double acc = 0.0;
    for (int cc = c0; cc < c1; ++cc) acc += part[(int64_t)cc * 54 + q];
    if (q < 45) U0[(int64_t)cam * 45 + q] = acc; else bp[(int64_t)cam * 9 + q - 45] = acc;
  }
}

__device__ __forceinline__ int diag_index9(int i) { return i * 9 - i * (i - 1) / 2; }

__global__ void k_cam_dp(const double* __restrict__ U0, int64_t n_cam, double* __restrict__ Dp) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_cam * 9) return;
  const int64_t cam = q / 9;
  const int i = (int)(q - cam * 9);
  const double v = U0[cam * 45 + diag_index9(i)];
  Dp[q] = sqrt(fmin(fmax(v, kClampLo * kClampLo), kClampHi * kClampHi));
}

// 0.5 sum ||r||^2: per warp-tile butterfly, per block fixed-order sum, invalid counts
__global__ void __launch_bounds__(kBlockTiles * kTile)
k_cost_tile(const Tile* __restrict__ tiles, int n_tiles, const int* __restrict__ cam_s,
            const double2* __restrict__ pix_s, const uint8_t* __restrict__ lidx_s, const double* __restrict__ prep,
            const double* __restrict__ points, const double* __restrict__ dl, double* __restrict__ block_sum,
            unsigned long long* __restrict__ n_invalid) {
  __shared__ double wsum[kBlockTiles];
  extern __shared__ __align__(16) double2 lin_rec[];  // per warp: the tile's camera records (gather_prep)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ti = blockIdx.x * kBlockTiles + w;
  double v = 0.0;
  bool bad = false;
  if (ti < n_tiles) {
    const int64_t o = (int64_t)ti * kTile + lane;
    // per-slot loads first (the slot arrays cover the padding), then the descriptor's dependants
    const int cam_o = cam_s[o];
    const int li_o = lidx_s[o];
    const double2 pix = __ldcs(pix_s + o);
    const Tile t = tiles[ti];
    // point (and trial increment) loads in flight during the camera gather
    double X0 = 0.0, X1 = 0.0, X2 = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
    if (lane < t.n) {
      const int64_t lm = t.lm0 + ((t.flags & kTileLong) ? 0 : li_o);
      X0 = points[lm * 3];
      X1 = points[lm * 3 + 1];
      X2 = points[lm * 3 + 2];
      if (dl) {
        d0 = dl[lm * 3];
        d1 = dl[lm * 3 + 1];
        d2 = dl[lm * 3 + 2];
      }
    }
    double cp[16];
    gather_prep(prep, lane < t.n ? cam_o : 0, t.n, lane, lin_rec + w * kTile * kLinRec, cp);
    if (lane < t.n) {
      X0 += d0;
      X1 += d1;
      X2 += d2;
      ObsModel m;
      evaluate_obs<false>(cp, X0, X1, X2, pix, m);
      bad = !m.valid;
      v = m.r0 * m.r0 + m.r1 * m.r1;
    }
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  const unsigned nbad = __popc(__ballot_sync(0xffffffffu, bad));
  if (lane == 0) {
    wsum[w] = v;
    if (nbad) atomicAdd(n_invalid, (unsigned long long)nbad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < kBlockTiles; ++k) b += wsum[k];
    block_sum[blockIdx.x] = b;
  }
}

// fixed-order sum of n values by one CTA (strided partial sums, then a tree)
__global__ void k_sum_fixed(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double red[1024];
  const int i = threadIdx.x;
  double acc = 0.0;
  for (int64_t q = i; q < n; q += blockDim.x) acc += v[q];
  red[i] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (i < s) red[i] += red[i + s];
    __syncthreads();
  }
  if (i == 0) out[0] = red[0];
}

}  // namespace

int cameras_prep(Ctx& c, const double* d_cams, double* d_prep) {
  k_cam_prep<<<grid_for(c.n_cam, 128), 128, 0, c.stream>>>(d_cams, c.n_cam, d_prep);
  c.launches++;
  PCK(cudaGetLastError());
  return POBA_OK;
}

int linearize_device(Ctx& c, bool expl, const double* h_jp, const double* h_jl, const double* h_res,
                     const double* h_points) {
  cudaStream_t s = c.stream;
  const int64_t ns = c.n_slots;
  DBuf ejp, ejl, eres;
  if (expl) {
    PTRY(ejp.alloc(c.n_obs * 18 * 8));
    PTRY(ejl.alloc(c.n_obs * 6 * 8));
    PTRY(eres.alloc(c.n_obs * 2 * 8));
    PCK(cudaMemcpyAsync(ejp.p, h_jp, c.n_obs * 18 * 8, cudaMemcpyHostToDevice, s));
    PCK(cudaMemcpyAsync(ejl.p, h_jl, c.n_obs * 6 * 8, cudaMemcpyHostToDevice, s));
    PCK(cudaMemcpyAsync(eres.p, h_res, c.n_obs * 2 * 8, cudaMemcpyHostToDevice, s));
  } else {
    PTRY(cameras_prep(c, c.cams.as<double>(), c.cams_prep.as<double>()));
  }
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(c.flag.as<char>() + 32);
  PCK(cudaMemsetAsync(d_bad, 0, 8, s));
  const bool f32 = c.precision == 32;
  auto lin = [&](auto kern, const double* prep, const double* pts, const double* a, const double* b,
                 const double* r, int t0, int t1) {
    if (t1 <= t0) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kLinTileSmem);
    kern<<<grid_for(t1 - t0, kLinTiles), kLinTiles * kTile, kLinTileSmem, s>>>(
        c.tiles.as<Tile>(), t0, t1, c.cam_s.as<int>(), c.file_s.as<int>(), c.pix_s.as<double2>(),
        c.lidx_s.as<uint8_t>(), prep, pts, a, b, r, c.J.p, c.Rz.as<double2>(), c.V0.as<double>(), c.bl.as<double>(),
        c.Dl.as<double>(), d_bad);
    c.launches++;
  };
  // Tile pass: the software-pipelined kernel (12 warps per SM, two tiles of loads
  // in flight per warp) wins when the camera records come from L2 (C5, 13,700
  // cameras: 3.02 -> 2.72 ms); with ~1,100 cameras the records stay in L1, the
  // load waves are short and the one-tile-per-warp kernel's 16 warps per SM hide
  // the fp64 dependency chain better (C4: 1.15 vs 1.25 ms).  POBA_LIN_PIPE=0/1 forces.
  const bool pipe = getenv("POBA_LIN_PIPE") ? atoi(getenv("POBA_LIN_PIPE")) != 0 : c.n_cam > 4096;
  auto lin_range = [&](int t0, int t1) {
    if (expl) {
      if (f32) lin(k_lin_tile<true, true>, nullptr, nullptr, ejp.as<double>(), ejl.as<double>(), eres.as<double>(), t0, t1);
      else lin(k_lin_tile<true, false>, nullptr, nullptr, ejp.as<double>(), ejl.as<double>(), eres.as<double>(), t0, t1);
    } else if (pipe) {
      if (t1 <= t0) return;
      const int nblk = std::min((t1 - t0 + kPipeWarps - 1) / kPipeWarps, c.n_sm * POBA_LIN_PIPE_BLOCKS);
      auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmem);
        kern<<<nblk, kPipeWarps * kTile, kPipeSmem, s>>>(c.tiles.as<Tile>(), t0, t1, c.cam_s.as<int>(),
                                                        c.pix_s.as<double2>(), c.lidx_s.as<uint8_t>(),
                                                        c.cams_prep.as<double>(), c.points.as<double>(), c.J.p,
                                                        c.Rz.as<double2>(), c.V0.as<double>(), c.bl.as<double>(),
                                                        c.Dl.as<double>(), d_bad);
        c.launches++;
      };
      if (f32) go(k_lin_tile_pipe<true>);
      else go(k_lin_tile_pipe<false>);
    } else {
      if (f32) lin(k_lin_tile<false, true>, c.cams_prep.as<double>(), c.points.as<double>(), nullptr, nullptr, nullptr, t0, t1);
      else lin(k_lin_tile<false, false>, c.cams_prep.as<double>(), c.points.as<double>(), nullptr, nullptr, nullptr, t0, t1);
    }
  };
  if (h_points && !expl) {
    // points arrive in file-order pieces; each piece releases the tiles whose
    // landmarks are complete (the rest of the pass overlaps the copy)
    const bool pinned = is_pinned(h_points);
    PTRY(xfer_begin(c, 3, pinned));
    for (int i = 0; i < kXferPieces; ++i) {
      PTRY(lm_upload_piece(c, h_points, 3, c.points.as<double>(), i, pinned));
      lin_range(c.xf_up_tile[i], c.xf_up_tile[i + 1]);
    }
  } else {
    lin_range(0, c.n_tiles);
  }
  PCK(cudaGetLastError());
  if (c.n_long) {
    if (f32)
      k_lin_long<true><<<c.n_long, 32, 0, s>>>(c.long_lm.as<int>(), c.lm_slot0.as<int>(), c.lm_k.as<int>(), c.J.p,
                                               c.Rz.as<double2>(), ns, c.V0.as<double>(), c.bl.as<double>(),
                                               c.Dl.as<double>());
    else
      k_lin_long<false><<<c.n_long, 32, 0, s>>>(c.long_lm.as<int>(), c.lm_slot0.as<int>(), c.lm_k.as<int>(), c.J.p,
                                                c.Rz.as<double2>(), ns, c.V0.as<double>(), c.bl.as<double>(),
                                                c.Dl.as<double>());
    c.launches++;
  }
  // camera side: U0 / b_p via camera-major chunks, then a fixed-order merge
  if (c.n_cchunks) {
    const unsigned g = grid_for((int64_t)c.n_cchunks * 32, kCamReduceThreads);
    auto reduce = [&](auto kern) {
      kern<<<g, kCamReduceThreads, 0, s>>>(c.cc_cam_off.as<int>(), c.cc_cam.as<int>(), c.cam_start.as<int>(),
                                           c.n_cchunks, c.cams_prep.as<double>(), c.points.as<double>(),
                                           c.lm_c.as<int>(), c.pix_c.as<double2>(), c.file_c.as<int>(),
                                           ejp.as<double>(), eres.as<double>(), c.cc_part.as<double>());
    };
    if (expl) {
      if (f32) reduce(k_cam_chunk_reduce<true, true>);
      else reduce(k_cam_chunk_reduce<true, false>);
    } else {
      if (f32) reduce(k_cam_chunk_reduce<false, true>);
      else reduce(k_cam_chunk_reduce<false, false>);
    }
    c.launches++;
  }
  k_cam_merge54<<<grid_for(c.n_cam * 32, 256), 256, 0, s>>>(c.cc_cam_off.as<int>(), c.cc_part.as<double>(),
                                                            (int)c.n_cam, c.U0.as<double>(), c.bp.as<double>());
  c.launches++;
  PCK(cudaGetLastError());
  if (c.nranks > 1) {
    PTRY(allreduce_sum(c, c.U0.as<double>(), c.n_cam * 45));
    PTRY(allreduce_sum(c, c.bp.as<double>(), c.n_cam * 9));
  }
  k_cam_dp<<<grid_for(c.n_cam * 9, 256), 256, 0, s>>>(c.U0.as<double>(), c.n_cam, c.Dp.as<double>());
  c.launches++;
  unsigned long long bad = 0;
  PCK(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (c.nranks > 1) {
    double b = (double)bad;
    PTRY(c.scratch_b.alloc(8));
    PCK(cudaMemcpyAsync(c.scratch_b.p, &b, 8, cudaMemcpyHostToDevice, s));
    PTRY(allreduce_sum(c, c.scratch_b.as<double>(), 1));
    PCK(cudaMemcpyAsync(&b, c.scratch_b.p, 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    bad = (unsigned long long)b;
  }
  c.n_invalid = (int64_t)bad;
  c.have_lin = true;
  c.have_damp = c.have_solution = c.have_delta_l = false;
  return POBA_OK;
}

int cost_device(Ctx& c, bool trial, double* cost, int64_t* n_invalid) {
  cudaStream_t s = c.stream;
  const unsigned nb = grid_for(c.n_tiles, kBlockTiles);
  PTRY(c.scratch_c.alloc((nb + 8) * 8));
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(c.flag.as<char>() + 40);
  PCK(cudaMemsetAsync(d_bad, 0, 8, s));
  cudaFuncSetAttribute(k_cost_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, kLinRecSmem);
  k_cost_tile<<<nb, kBlockTiles * kTile, kLinRecSmem, s>>>(c.tiles.as<Tile>(), c.n_tiles, c.cam_s.as<int>(),
                                                 c.pix_s.as<double2>(), c.lidx_s.as<uint8_t>(),
                                                 c.trial_prep.as<double>(), c.points.as<double>(),
                                                 trial ? c.dl.as<double>() : nullptr, c.scratch_c.as<double>(), d_bad);
  k_sum_fixed<<<1, 1024, 0, s>>>(c.scratch_c.as<double>(), nb, c.red.as<double>());
  c.launches += 2;
  PCK(cudaGetLastError());
  double sum = 0;
  unsigned long long bad = 0;
  PCK(cudaMemcpyAsync(&sum, c.red.p, 8, cudaMemcpyDeviceToHost, s));
  PCK(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (c.nranks > 1) {
    // per-rank partials gathered and summed in rank order (deterministic)
    std::vector<double> mine = {sum, (double)bad};
    PTRY(c.scratch_b.alloc(2 * 8 * (c.nranks + 1)));
    PCK(cudaMemcpyAsync(c.scratch_b.p, mine.data(), 16, cudaMemcpyHostToDevice, s));
    PTRY(allgather(c, c.scratch_b.as<double>(), c.scratch_b.as<double>() + 2, 2));
    std::vector<double> all(2 * c.nranks);
    PCK(cudaMemcpyAsync(all.data(), c.scratch_b.as<double>() + 2, 16 * c.nranks, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    sum = 0;
    bad = 0;
    for (int r = 0; r < c.nranks; ++r) {
      sum += all[2 * r];
      bad += (unsigned long long)all[2 * r + 1];
    }
  }
  *cost = 0.5 * sum;
  *n_invalid = (int64_t)bad;
  return POBA_OK;
}

}  // namespace poba
