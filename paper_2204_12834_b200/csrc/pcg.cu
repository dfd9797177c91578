// PCG baselines on the same device operators (reference solvers.py:30-118):
// the exact 9x9 Schur diagonal blocks and their inverses (schur_diagonal_blocks /
// make_schur_jacobi_preconditioner, solvers.py:71-95), and preconditioned CG on
// S dx_p = -b_tilde (pcg, solvers.py:30-64) with either the Schur-Jacobi or the
// order-m power-series preconditioner (pcg_power_series_preconditioner,
// solvers.py:105-118).  One Schur product S p = U p - W V^-1 W^T p is one pass
// of the fused term kernel; dot products are fixed-order block reductions; the
// CG scalars go to the host once per dot (the reference's control flow).
#include <cmath>
#include <vector>

#include "poba_internal.h"

namespace poba {

// from series.cu
int schur_product_device(Ctx& c, const double* d_p, double* d_out);
int damp_u_blocks(Ctx& c, const double* M45, double* M45_copy, double* Minv45, const char* what);
int series_apply_device(Ctx& c, const double* d_v, int order, double* d_out);
int b_tilde_device(Ctx& c);
void launch_cam_mv(Ctx& c, const double* M45, const double* v, double* out);

namespace {

// per camera-major chunk (<= kCamChunk observations of one camera):
// sum of W_o V_l^-1 W_o^T, W_o = J_p^T J_l (9x3), packed upper 45
template <bool F32>
__global__ void __launch_bounds__(128)
k_schur_diag_chunk(const int* __restrict__ cc_cam_off, const int* __restrict__ cc_cam, const int* __restrict__ cam_start,
                   const int* __restrict__ cperm, const void* __restrict__ J, const Tile* __restrict__ tiles,
                   const uint8_t* __restrict__ lidx_s, const double* __restrict__ Vinv, int n_cam, int n_cc,
                   double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_cc) return;
  const int cam = cc_cam[warp];
  const int p0 = cam_start[cam] + (warp - cc_cam_off[cam]) * kCamChunk;
  const int p1 = min(p0 + kCamChunk, cam_start[cam + 1]);
  double acc[45];
#pragma unroll
  for (int q = 0; q < 45; ++q) acc[q] = 0.0;
  for (int p = p0 + lane; p < p1; p += 32) {
    const int o = cperm[p];
    const Tile t = tiles[o >> 5];
    const int lm = t.lm0 + ((t.flags & kTileLong) ? 0 : lidx_s[o]);
    const double* V = Vinv + (int64_t)lm * 6;
    const double v00 = V[0], v01 = V[1], v02 = V[2], v11 = V[3], v12 = V[4], v22 = V[5];
    const double2 l0 = jload<F32>(J, o, 9), l1 = jload<F32>(J, o, 10), l2 = jload<F32>(J, o, 11);
    double w[9][3], tm[9][3];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double2 a = jload<F32>(J, o, i);
      w[i][0] = fma(a.x, l0.x, a.y * l0.y);
      w[i][1] = fma(a.x, l1.x, a.y * l1.y);
      w[i][2] = fma(a.x, l2.x, a.y * l2.y);
      tm[i][0] = w[i][0] * v00 + w[i][1] * v01 + w[i][2] * v02;
      tm[i][1] = w[i][0] * v01 + w[i][1] * v11 + w[i][2] * v12;
      tm[i][2] = w[i][0] * v02 + w[i][1] * v12 + w[i][2] * v22;
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int k = i; k < 9; ++k) acc[q++] += tm[i][0] * w[k][0] + tm[i][1] * w[k][1] + tm[i][2] * w[k][2];
  }
#pragma unroll
  for (int q = 0; q < 45; ++q) {
    double v = acc[q];
#pragma unroll
    for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    acc[q] = v;
  }
  double* dst = out + (int64_t)warp * 54;
#pragma unroll
  for (int q = 0; q < 45; ++q)
    if ((q & 31) == lane) dst[q] = acc[q];
}

// per camera: sum of its chunk partials (chunk order)
__global__ void k_schur_diag_merge(const int* __restrict__ cc_cam_off, const double* __restrict__ part, int n_cam,
                                   double* __restrict__ sum45) {
  const int cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cam >= n_cam) return;
  const int c0 = cc_cam_off[cam], c1 = cc_cam_off[cam + 1];
  for (int q = lane; q < 45; q += 32) {
    double acc = 0.0;
    for (int cc = c0; cc < c1; ++cc) acc += part[(int64_t)cc * 54 + q];
    sum45[(int64_t)cam * 45 + q] = acc;
  }
}

__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}

// fixed-order dot product: one block, 1024 threads, strided partial sums then a tree
constexpr int kDotThreads = 1024;
__global__ void __launch_bounds__(kDotThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                     int64_t n, double* __restrict__ out) {
  __shared__ double red[kDotThreads];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kDotThreads) s = fma(a[i], b[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kDotThreads / 2; w; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// out = -a, flag if any entry is nonzero
__global__ void k_neg(const double* __restrict__ a, int64_t n, double* __restrict__ out, int* __restrict__ nonzero) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = a[i];
  out[i] = -v;
  if (v != 0.0) *nonzero = 1;
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double alpha, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = y[i] + alpha * x[i];
}

__global__ void k_xpby(double* __restrict__ p, const double* __restrict__ z, double beta, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = z[i] + beta * p[i];
}

}  // namespace

// M = U - sum_o W_o V^-1 W_o^T per camera, and its inverse (c.Minv)
int schur_diag_device(Ctx& c, double* d_out45 /* nullable */) {
  cudaStream_t s = c.stream;
  const int64_t n_cam = c.n_cam;
  PTRY(c.Mbuf.alloc(n_cam * 45 * 8));
  PTRY(c.Minv.alloc(n_cam * 45 * 8));
  PTRY(c.scratch_c.alloc(n_cam * 45 * 8));
  if (c.n_cchunks) {
    const int threads = 128;
    const unsigned g = grid_for((int64_t)c.n_cchunks * 32, threads);
    if (c.precision == 32)
      k_schur_diag_chunk<true><<<g, threads, 0, s>>>(c.cc_cam_off.as<int>(), c.cc_cam.as<int>(), c.cam_start.as<int>(), c.cperm.as<int>(),
                                                     c.J.p, c.tiles.as<Tile>(), c.lidx_s.as<uint8_t>(),
                                                     c.Vinv.as<double>(), (int)n_cam, c.n_cchunks,
                                                     c.cc_part.as<double>());
    else
      k_schur_diag_chunk<false><<<g, threads, 0, s>>>(c.cc_cam_off.as<int>(), c.cc_cam.as<int>(), c.cam_start.as<int>(),
                                                      c.cperm.as<int>(), c.J.p, c.tiles.as<Tile>(),
                                                      c.lidx_s.as<uint8_t>(), c.Vinv.as<double>(), (int)n_cam,
                                                      c.n_cchunks, c.cc_part.as<double>());
    c.launches++;
  }
  k_schur_diag_merge<<<grid_for(n_cam * 32, 256), 256, 0, s>>>(c.cc_cam_off.as<int>(), c.cc_part.as<double>(),
                                                              (int)n_cam, c.scratch_c.as<double>());
  c.launches++;
  PCK(cudaGetLastError());
  if (c.nranks > 1) PTRY(allreduce_sum(c, c.scratch_c.as<double>(), n_cam * 45));
  k_sub<<<grid_for(n_cam * 45, 256), 256, 0, s>>>(c.Ud.as<double>(), c.scratch_c.as<double>(), n_cam * 45,
                                                  c.Mbuf.as<double>());
  c.launches++;
  PTRY(damp_u_blocks(c, c.Mbuf.as<double>(), c.scratch_c.as<double>(), c.Minv.as<double>(),
                     "Schur diagonal blocks are not positive definite"));
  if (d_out45) PCK(cudaMemcpyAsync(d_out45, c.Mbuf.p, n_cam * 45 * 8, cudaMemcpyDeviceToDevice, s));
  PCK(cudaStreamSynchronize(s));
  return POBA_OK;
}

namespace {

int dot_host(Ctx& c, const double* a, const double* b, int64_t n, double* out) {
  PTRY(c.red.alloc(64 * 8));
  k_dot<<<1, kDotThreads, 0, c.stream>>>(a, b, n, c.red.as<double>());
  c.launches++;
  PCK(cudaGetLastError());
  return copy_sync(c, out, c.red.p, 8, cudaMemcpyDeviceToHost);
}

int precondition(Ctx& c, int precond, int order, const double* r, double* z) {
  if (precond == POBA_PRECOND_SCHUR_JACOBI) {
    launch_cam_mv(c, c.Minv.as<double>(), r, z);
    PCK(cudaGetLastError());
    return POBA_OK;
  }
  return series_apply_device(c, r, order, z);
}

}  // namespace

int pcg_device(Ctx& c, int precond, int order, double tol, int max_iter, bool resume, double* h_delta_p,
               int* iterations, double* final_rel, int* converged, double* rel_history) {
  cudaStream_t s = c.stream;
  const int64_t n = c.n_cam * 9;
  const unsigned g = grid_for(n, 256);
  PTRY(c.pcg_vec.alloc(5 * n * 8));
  double* x = c.pcg_vec.as<double>();
  double* r = x + n;
  double* z = r + n;
  double* p = z + n;
  double* sp = p + n;
  PcgState& st = c.pcg;
  int done_here = 0;
  if (!resume || !st.active) {
    if (precond == POBA_PRECOND_SCHUR_JACOBI) PTRY(schur_diag_device(c, nullptr));
    PTRY(b_tilde_device(c));
    PCK(cudaMemsetAsync(x, 0, n * 8, s));
    PTRY(c.flag.alloc(64));
    int* nz = c.flag.as<int>() + 2;
    PCK(cudaMemsetAsync(nz, 0, 4, s));
    k_neg<<<g, 256, 0, s>>>(c.bt.as<double>(), n, r, nz);  // rhs = -b_tilde
    c.launches++;
    int h_nz = 0;
    PTRY(copy_sync(c, &h_nz, nz, 4, cudaMemcpyDeviceToHost));
    st = PcgState{};
    st.precond = precond;
    st.order = order;
    if (!h_nz) {  // zero right-hand side (solvers.py:41-43)
      st.active = false;
      *iterations = 0;
      *final_rel = 0.0;
      *converged = 1;
      if (h_delta_p) PTRY(copy_sync(c, h_delta_p, x, n * 8, cudaMemcpyDeviceToHost));
      return POBA_OK;
    }
    PTRY(precondition(c, precond, order, r, z));
    PTRY(dot_host(c, r, z, n, &st.rz));
    if (!(st.rz > 0)) return fail(POBA_ENOTSPD, "preconditioner is not positive definite");
    st.rz0 = st.rz;
    PCK(cudaMemcpyAsync(p, z, n * 8, cudaMemcpyDeviceToDevice, s));
    st.rel = 1.0;
    st.it = 0;
    st.active = true;
  } else if (st.precond != precond || st.order != order) {
    return fail(POBA_EINVAL, "resumed PCG with a different preconditioner");
  }
  bool conv = false;
  for (int k = 0; k < max_iter; ++k) {
    ++st.it;
    PTRY(schur_product_device(c, p, sp));
    double psp = 0.0;
    PTRY(dot_host(c, p, sp, n, &psp));
    if (!(psp > 0)) {
      st.active = false;
      return fail(POBA_ENOTSPD, "reduced system is not positive definite");
    }
    const double alpha = st.rz / psp;
    k_axpy<<<g, 256, 0, s>>>(x, p, alpha, n);
    k_axpy<<<g, 256, 0, s>>>(r, sp, -alpha, n);
    c.launches += 2;
    PTRY(precondition(c, precond, order, r, z));
    double rz_new = 0.0;
    PTRY(dot_host(c, r, z, n, &rz_new));
    st.rel = std::sqrt(std::max(rz_new, 0.0) / st.rz0);
    if (rel_history) rel_history[done_here] = st.rel;
    ++done_here;
    if (st.rel < tol) {
      conv = true;
      st.active = false;
      break;
    }
    k_xpby<<<g, 256, 0, s>>>(p, z, rz_new / st.rz, n);
    c.launches++;
    st.rz = rz_new;
  }
  PCK(cudaGetLastError());
  *iterations = st.it;
  *final_rel = st.rel;
  *converged = conv ? 1 : 0;
  if (h_delta_p) PTRY(copy_sync(c, h_delta_p, x, n * 8, cudaMemcpyDeviceToHost));
  return POBA_OK;
}

}  // namespace poba
