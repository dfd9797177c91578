// Spectral radius of the series iteration matrix on the device.
//
// Reference (paths relative to /root/reference/pkg/src/powerba/):
//   _u_inv_sqrt_blocks        spectral.py:46-51
//   estimate_spectral_radius  spectral.py:54-86
//
// rho(P), P = U^-1 W V^-1 W^T, is the dominant eigenvalue of the similar
// symmetric M = U^-1/2 (W V^-1 W^T) U^-1/2.  U^-1/2 is formed per camera by a
// cyclic Jacobi eigendecomposition of the damped 9x9 block (one thread per
// camera); every power-iteration step is then M v (two block-diagonal products
// around one pass of the fused term kernel), a fixed-order two-value reduction
// (v.w, w.w), one 16-B read to the host for the convergence test, and the
// normalisation v <- w / |w| -- the iterate never leaves the device.
#include <cmath>

#include "poba_internal.h"

namespace poba {

void launch_cam_mv(Ctx& c, const double* M45, const double* v, double* out);
int schur_product_device(Ctx& c, const double* d_p, double* d_out);

namespace {

__device__ __forceinline__ int pk9s(int i, int j) {  // packed upper-triangle index, any order
  if (i > j) {
    const int t = i;
    i = j;
    j = t;
  }
  return i * 9 - i * (i - 1) / 2 + (j - i);
}

// U^-1/2 of each damped block (packed 45) by cyclic Jacobi rotations;
// flag |= 1 if a block is not positive definite
__global__ void k_inv_sqrt9(const double* __restrict__ U45, int64_t n_cam, double* __restrict__ out45,
                            int* __restrict__ flag) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cam) return;
  double A[9][9], Q[9][9];
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) {
      A[i][j] = U45[c * 45 + pk9s(i, j)];
      Q[i][j] = (i == j) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < 9; ++i) {
      diag += A[i][i] * A[i][i];
      for (int j = i + 1; j < 9; ++j) off += A[i][j] * A[i][j];
    }
    if (off <= 1e-34 * diag) break;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 9; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 9; ++k) {  // A <- J^T A J
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = cs * akp - sn * akq;
          A[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 9; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = cs * apk - sn * aqk;
          A[q][k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < 9; ++k) {  // Q <- Q J
          const double qkp = Q[k][p], qkq = Q[k][q];
          Q[k][p] = cs * qkp - sn * qkq;
          Q[k][q] = sn * qkp + cs * qkq;
        }
      }
  }
  double s[9];
  for (int k = 0; k < 9; ++k) {
    if (!(A[k][k] > 0.0)) atomicOr(flag, 1);
    s[k] = 1.0 / sqrt(A[k][k]);
  }
  for (int i = 0; i < 9; ++i)
    for (int j = i; j < 9; ++j) {
      double v = 0.0;
      for (int k = 0; k < 9; ++k) v += Q[i][k] * s[k] * Q[j][k];
      out45[c * 45 + pk9s(i, j)] = v;
    }
}

// out = (v.w, w.w), one block, fixed order (strided thread sums, then a tree)
__global__ void __launch_bounds__(1024) k_dot2(const double* __restrict__ v, const double* __restrict__ w, int64_t n,
                                               double* __restrict__ out) {
  __shared__ double red[2][1024];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    a = fma(v[i], w[i], a);
    b = fma(w[i], w[i], b);
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if ((int)threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = red[0][0];
    out[1] = red[1][0];
  }
}

__global__ void k_div(const double* __restrict__ w, double d, int64_t n, double* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = w[i] / d;
}

__global__ void k_unit(double* e, int64_t n, int64_t j) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) e[i] = (i == j) ? 1.0 : 0.0;
}

}  // namespace

// Dense matrix of a camera-space operator (S, W V^-1 W^T, U, U^-1), built on
// the device one basis vector at a time (one fused pass per column for S and
// W V^-1 W^T) and copied to the host once, column-major (out[j * dim + i] =
// (Op e_j)_i).  Oracle-scale systems only (the dense solvers, the spectral
// check): dim <= limit.
int materialize_device(Ctx& c, int op, int64_t limit, double* h_out) {
  const int64_t dim = c.n_cam * 9;
  if (dim > limit) return fail(POBA_EINVAL, "dense operator refused: " + std::to_string(dim) +
                                                " pose parameters exceeds limit " + std::to_string(limit));
  if (op != POBA_OP_SCHUR && op != POBA_OP_WVW && op != POBA_OP_U && op != POBA_OP_U_INV)
    return fail(POBA_EINVAL, "only camera-space operators can be materialized");
  DBuf M, e;
  PTRY(M.alloc((size_t)dim * dim * 8));
  PTRY(e.alloc(dim * 8));
  for (int64_t j = 0; j < dim; ++j) {
    k_unit<<<grid_for(dim, 256), 256, 0, c.stream>>>(e.as<double>(), dim, j);
    c.launches++;
    double* col = M.as<double>() + j * dim;
    if (op == POBA_OP_SCHUR) PTRY(schur_product_device(c, e.as<double>(), col));
    else PTRY(apply_op_device(c, op, e.as<double>(), col));
  }
  PCK(cudaGetLastError());
  return copy_sync(c, h_out, M.p, (size_t)dim * dim * 8, cudaMemcpyDeviceToHost);
}

int spectral_radius_device(Ctx& c, const double* h_v0, double tol, int max_iter, double* rho, int* iterations,
                           int* converged) {
  cudaStream_t s = c.stream;
  const int64_t n = c.n_cam * 9;
  DBuf uis, v, y, z, w, dots;
  PTRY(uis.alloc(c.n_cam * 45 * 8));
  PTRY(v.alloc(n * 8));
  PTRY(y.alloc(n * 8));
  PTRY(z.alloc(n * 8));
  PTRY(w.alloc(n * 8));
  PTRY(dots.alloc(16));
  int* fl = c.flag.as<int>() + 3;
  PCK(cudaMemsetAsync(fl, 0, 4, s));
  k_inv_sqrt9<<<grid_for(c.n_cam, 64), 64, 0, s>>>(c.Ud.as<double>(), c.n_cam, uis.as<double>(), fl);
  c.launches++;
  PCK(cudaGetLastError());
  int h = 0;
  PTRY(copy_sync(c, &h, fl, 4, cudaMemcpyDeviceToHost));
  if (h) return fail(POBA_EINVAL, "damped pose blocks must be positive definite");
  PTRY(copy_sync(c, v.p, h_v0, n * 8, cudaMemcpyHostToDevice));
  double est = 0.0;
  for (int it = 1; it <= max_iter; ++it) {
    launch_cam_mv(c, uis.as<double>(), v.as<double>(), y.as<double>());
    PTRY(apply_op_device(c, POBA_OP_WVW, y.as<double>(), z.as<double>()));
    launch_cam_mv(c, uis.as<double>(), z.as<double>(), w.as<double>());
    k_dot2<<<1, 1024, 0, s>>>(v.as<double>(), w.as<double>(), n, dots.as<double>());
    c.launches++;
    PCK(cudaGetLastError());
    double d2[2];
    PTRY(copy_sync(c, d2, dots.p, 16, cudaMemcpyDeviceToHost));
    const double nw = std::sqrt(d2[1]);
    if (nw == 0.0) {
      *rho = 0.0;
      *iterations = it;
      *converged = 1;
      return POBA_OK;
    }
    const double next = d2[0];
    k_div<<<grid_for(n, 256), 256, 0, s>>>(w.as<double>(), nw, n, v.as<double>());
    c.launches++;
    if (std::fabs(next - est) <= tol * std::fmax(std::fabs(next), 1e-300)) {
      *rho = next;
      *iterations = it;
      *converged = 1;
      return POBA_OK;
    }
    est = next;
  }
  *rho = est;
  *iterations = max_iter;
  *converged = 0;
  return POBA_OK;
}

}  // namespace poba
