// PoST clustered pose solve (reference clustering.solve_clustered,
// pkg/src/powerba/clustering.py:125-148) without per-cluster sub-problems:
// the caller's store holds one VIRTUAL landmark per (landmark, camera cluster)
// pair, so the reduced system is block diagonal over the clusters and one
// pass of the fused term kernel advances every cluster's series at once.
// Each cluster keeps its own stop test -- (i+1)||x_i - x_{i-1}||_c / ||x_i||_c
// < epsilon over its own cameras, a zero right-hand side stopping it at order
// 0 -- and a stopped cluster's term vector is zeroed, so its iterate freezes
// at its own stopping order exactly as its separate power_series_solve would.
#include <algorithm>
#include <cmath>
#include <vector>

#include "poba_internal.h"

namespace poba {

// from series.cu
int launch_term_mode(Ctx& c, int mode, const double* tin, const double* lvec, bool check_stop);
int launch_merge(Ctx& c);  // partials -> c.rvec (+ all-reduce when sharded)

namespace {

__device__ __forceinline__ int pk9c(int i, int j) { return i * 9 - i * (i - 1) / 2 + (j - i); }
__device__ __forceinline__ int sym9c(int i, int j) { return i <= j ? pk9c(i, j) : pk9c(j, i); }

struct ClState {
  int stopped, order, converged, pad;
};

// per camera: t = U^-1 r (or U^-1(-b_tilde) at order 0), x update unless the
// camera's cluster has stopped; per-camera squared norms for the cluster test
template <bool kBt>
__global__ void k_cam_cl(const double* __restrict__ rvec, const double* __restrict__ Uinv,
                         const double* __restrict__ bp, const int* __restrict__ cl_of_cam,
                         const ClState* __restrict__ cst, int n_cam, double* __restrict__ bt,
                         double* __restrict__ tvec, double* __restrict__ xvec, double* __restrict__ cam_red,
                         const SeriesState* __restrict__ st) {
  const int cam = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cam >= n_cam || st->stopped) return;
  const bool frozen = !kBt && cst[cl_of_cam[cam]].stopped;
  double dd = 0.0, xx = 0.0, nf = 0.0, nz = 0.0;
  if (lane < 9) {
    const int i = lane;
    const int64_t q = (int64_t)cam * 9 + i;
    double v[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const double r = rvec[(int64_t)cam * 9 + j];
      v[j] = kBt ? -(bp[(int64_t)cam * 9 + j] - r) : r;
    }
    double t = 0.0;
    const double* U = Uinv + (int64_t)cam * 45;
#pragma unroll
    for (int j = 0; j < 9; ++j) t = fma(U[sym9c(i, j)], v[j], t);
    if (kBt) {
      const double bti = bp[q] - rvec[q];
      bt[q] = bti;
      nz = bti != 0.0 ? 1.0 : 0.0;
      tvec[(int64_t)cam * kTStride + i] = t;
      xvec[q] = t;
      xx = t * t;
      nf = isfinite(t) ? 0.0 : 1.0;
    } else if (frozen) {
      tvec[(int64_t)cam * kTStride + i] = 0.0;
    } else {
      tvec[(int64_t)cam * kTStride + i] = t;
      const double xo = xvec[q];
      const double xn = xo + t;
      const double df = xn - xo;
      xvec[q] = xn;
      dd = df * df;
      xx = xn * xn;
      nf = isfinite(xn) ? 0.0 : 1.0;
    }
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    dd += __shfl_down_sync(0xffffffffu, dd, s);
    xx += __shfl_down_sync(0xffffffffu, xx, s);
    nf += __shfl_down_sync(0xffffffffu, nf, s);
    nz += __shfl_down_sync(0xffffffffu, nz, s);
  }
  if (lane == 0) {
    cam_red[(int64_t)cam * 4 + 0] = dd;
    cam_red[(int64_t)cam * 4 + 1] = xx;
    cam_red[(int64_t)cam * 4 + 2] = nf;
    cam_red[(int64_t)cam * 4 + 3] = nz;
  }
}

// per cluster (one warp): fixed-order sums over its cameras, then the stop test
template <bool kBt>
__global__ void k_cluster_test(const int* __restrict__ cl_off, const int* __restrict__ cl_cams,
                               const double* __restrict__ cam_red, int n_cl, int order, double eps,
                               ClState* __restrict__ cst, SeriesState* __restrict__ st) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= n_cl || st->stopped) return;
  if (!kBt && cst[c].stopped) return;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = cl_off[c] + lane; k < cl_off[c + 1]; k += 32)
    for (int q = 0; q < 4; ++q) s[q] += cam_red[(int64_t)cl_cams[k] * 4 + q];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int d = 16; d; d >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], d);
  if (lane) return;
  const double DD = s[0], XX = s[1], NF = s[2], NZ = s[3];
  ClState& cs = cst[c];
  if (kBt) {
    cs = ClState{0, 0, 0, 0};
    if (NZ == 0.0) {  // zero right-hand side: (0, 0, True) (power_series.py:64-65)
      cs.stopped = 1;
      cs.converged = 1;
    } else if (NF > 0.0) {
      atomicCAS(&st->error, 0, POBA_ENONFINITE);
    }
  } else {
    if (NF > 0.0) {
      atomicCAS(&st->error, 0, POBA_ENONFINITE);
      st->error_order = order;
      return;
    }
    cs.order = order;
    if (XX == 0.0) {
      atomicCAS(&st->error, 0, POBA_EVANISH);
      return;
    }
    if ((double)(order + 1) * sqrt(DD) / sqrt(XX) < eps) {
      cs.stopped = 1;
      cs.converged = 1;
    }
  }
  if (cs.stopped) {
    const unsigned done = atomicAdd(&st->ticket2, 1u) + 1u;
    if (done == (unsigned)n_cl) st->stopped = 1;
  }
  if (st->error) st->stopped = 1;
}

}  // namespace

int series_clustered_device(Ctx& c, const int64_t* h_cluster_of_cam, int n_clusters, double eps, int max_order,
                            double* h_delta_p, int* order_used, int* converged) {
  cudaStream_t s = c.stream;
  const int n_cam = (int)c.n_cam;
  // cluster CSR (cameras of each cluster in index order)
  std::vector<int> cl(n_cam), off(n_clusters + 1, 0), cams(n_cam);
  for (int q = 0; q < n_cam; ++q) {
    const int64_t k = h_cluster_of_cam[q];
    if (k < 0 || k >= n_clusters) return fail(POBA_EINVAL, "cluster id out of range");
    cl[q] = (int)k;
    off[k + 1]++;
  }
  for (int k = 0; k < n_clusters; ++k) off[k + 1] += off[k];
  {
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (int q = 0; q < n_cam; ++q) cams[pos[cl[q]]++] = q;
  }
  for (int k = 0; k < n_clusters; ++k)
    if (off[k + 1] == off[k]) return fail(POBA_EINVAL, "empty cluster");
  DBuf d_cl, d_off, d_cams, d_cst, d_red;
  PTRY(d_cl.alloc(n_cam * 4));
  PTRY(d_off.alloc((n_clusters + 1) * 4));
  PTRY(d_cams.alloc(n_cam * 4));
  PTRY(d_cst.alloc(std::max(n_clusters, 1) * sizeof(ClState)));
  PTRY(d_red.alloc((size_t)n_cam * 4 * 8));
  PCK(cudaMemcpyAsync(d_cl.p, cl.data(), n_cam * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(d_off.p, off.data(), (n_clusters + 1) * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(d_cams.p, cams.data(), n_cam * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaMemsetAsync(d_cst.p, 0, std::max(n_clusters, 1) * sizeof(ClState), s));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  const unsigned gc = grid_for((int64_t)n_cam * 32, 256), gk = grid_for((int64_t)n_clusters * 32, 256);
  // order 0: b_tilde and t0 per camera, then the per-cluster zero-rhs / finiteness checks
  PTRY(launch_term_mode(c, 1 /* kModeBt */, nullptr, c.bl.as<double>(), false));
  PTRY(launch_merge(c));
  k_cam_cl<true><<<gc, 256, 0, s>>>(c.rvec.as<double>(), c.Uinv.as<double>(), c.bp.as<double>(), d_cl.as<int>(),
                                    d_cst.as<ClState>(), n_cam, c.bt.as<double>(), c.tvec.as<double>(),
                                    c.xvec.as<double>(), d_red.as<double>(), c.state.as<SeriesState>());
  k_cluster_test<true><<<gk, 256, 0, s>>>(d_off.as<int>(), d_cams.as<int>(), d_red.as<double>(), n_clusters, 0, eps,
                                          d_cst.as<ClState>(), c.state.as<SeriesState>());
  c.launches += 2;
  for (int i = 1; i <= max_order; ++i) {
    PTRY(launch_term_mode(c, 0 /* kModeTerm */, c.tvec.as<double>(), nullptr, true));
    PTRY(launch_merge(c));
    k_cam_cl<false><<<gc, 256, 0, s>>>(c.rvec.as<double>(), c.Uinv.as<double>(), c.bp.as<double>(), d_cl.as<int>(),
                                       d_cst.as<ClState>(), n_cam, c.bt.as<double>(), c.tvec.as<double>(),
                                       c.xvec.as<double>(), d_red.as<double>(), c.state.as<SeriesState>());
    k_cluster_test<false><<<gk, 256, 0, s>>>(d_off.as<int>(), d_cams.as<int>(), d_red.as<double>(), n_clusters, i,
                                             eps, d_cst.as<ClState>(), c.state.as<SeriesState>());
    c.launches += 2;
  }
  PCK(cudaGetLastError());
  SeriesState st;
  std::vector<ClState> hc(n_clusters);
  PCK(cudaMemcpyAsync(&st, c.state.p, sizeof(st), cudaMemcpyDeviceToHost, s));
  PCK(cudaMemcpyAsync(hc.data(), d_cst.p, n_clusters * sizeof(ClState), cudaMemcpyDeviceToHost, s));
  if (h_delta_p) PCK(cudaMemcpyAsync(h_delta_p, c.xvec.p, (size_t)n_cam * 9 * 8, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (st.error == POBA_ENONFINITE)
    return fail(POBA_ENONFINITE, "non-finite series iterate at order " + std::to_string(st.error_order) +
                                     ", assembly is broken");
  if (st.error == POBA_EVANISH) return fail(POBA_EVANISH, "vanishing iterate norm with a nonzero right-hand side");
  int ord = 0, conv = 1;
  for (const ClState& x : hc) {
    // a cluster that ran out of terms reports max_order (power_series.py:77)
    const int o = x.stopped ? x.order : max_order;
    ord = std::max(ord, o);
    conv &= x.converged;
  }
  *order_used = ord;
  *converged = conv;
  c.have_solution = true;
  c.last_order = ord;
  return POBA_OK;
}

}  // namespace poba
