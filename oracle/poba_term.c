/* Oracle (TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or
 * shipped): a plain-C restatement of the reference's two landmark-block
 * operator passes, for parity checks at configuration scale (C4/C5, 10-29M
 * observations) where the numpy restatement in poba_oracle.py would take
 * minutes per series.  Only tests/ and bench.py's CPU baseline load it.
 *
 * Reference (pkg/src/powerba/blocks.py):
 *   apply_wt  blocks.py:226-236   (W^T v)_l = sum_{o in l} J_l,o^T (J_p,o v_c(o))
 *   apply_w   blocks.py:214-224   (W v)_c   = sum_{o in c} J_p,o^T (J_l,o v_l(o))
 * over the canonical store (blocks.py:318-320): row o holds the 2x13 block
 * [J_p (9) | J_l (3) | r] of observation o in (k, landmark, camera) order,
 * every contraction accumulated in fp64 (blocks.py:45-47).
 *
 * Summation order.  W^T: each landmark's observations are contiguous in the
 * canonical order and are summed in that order, as the reference's per-group
 * einsum does.  W: observations are cut into T contiguous ranges (T = the
 * thread count argument); range t accumulates into its own camera table in
 * storage order, and the tables are added in range order -- deterministic for
 * a given T, and within a few ulps of the reference's sequential np.add.at
 * (the parity bar is 1e-9 relative).  Pinned against poba_oracle.py (itself
 * pinned to the reference's golden outputs) by tests/test_oracle_golden.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ROW 26 /* 2 x 13 doubles per observation */

/* out (3 n_pt) = W^T v (9 n_cam) */
int oracle_apply_wt(int64_t n_obs, const double* store, const int64_t* cam_sorted, const int64_t* pt_sorted,
                    int64_t n_pt, const double* v, double* out, int threads) {
  memset(out, 0, (size_t)n_pt * 3 * sizeof(double));
  /* landmark runs: maximal ranges of equal pt_sorted */
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t o = 0; o < n_obs; ++o) {
    if (o > 0 && pt_sorted[o - 1] == pt_sorted[o]) continue; /* not a run head */
    const int64_t l = pt_sorted[o];
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int64_t q = o; q < n_obs && pt_sorted[q] == l; ++q) {
      const double* b = store + q * ROW;
      const double* vc = v + cam_sorted[q] * 9;
      double u[2];
      for (int a = 0; a < 2; ++a) {
        double s = 0.0;
        for (int j = 0; j < 9; ++j) s += b[a * 13 + j] * vc[j];
        u[a] = s;
      }
      double w[3];
      for (int i = 0; i < 3; ++i) w[i] = b[9 + i] * u[0] + b[13 + 9 + i] * u[1];
      acc0 += w[0];
      acc1 += w[1];
      acc2 += w[2];
    }
    out[l * 3 + 0] = acc0;
    out[l * 3 + 1] = acc1;
    out[l * 3 + 2] = acc2;
  }
  return 0;
}

/* out (9 n_cam) = W v (3 n_pt) */
int oracle_apply_w(int64_t n_obs, const double* store, const int64_t* cam_sorted, const int64_t* pt_sorted,
                   int64_t n_cam, const double* v, double* out, int threads) {
  if (threads < 1) threads = 1;
  double* part = (double*)calloc((size_t)threads * n_cam * 9, sizeof(double));
  if (!part) return 1;
#pragma omp parallel for schedule(static, 1) num_threads(threads)
  for (int t = 0; t < threads; ++t) {
    const int64_t o0 = n_obs * t / threads, o1 = n_obs * (t + 1) / threads;
    double* acc = part + (size_t)t * n_cam * 9;
    for (int64_t o = o0; o < o1; ++o) {
      const double* b = store + o * ROW;
      const double* vl = v + pt_sorted[o] * 3;
      double u[2];
      for (int a = 0; a < 2; ++a) u[a] = b[a * 13 + 9] * vl[0] + b[a * 13 + 10] * vl[1] + b[a * 13 + 11] * vl[2];
      double* g = acc + cam_sorted[o] * 9;
      for (int j = 0; j < 9; ++j) g[j] += b[j] * u[0] + b[13 + j] * u[1];
    }
  }
  memset(out, 0, (size_t)n_cam * 9 * sizeof(double));
  for (int t = 0; t < threads; ++t) {
    const double* acc = part + (size_t)t * n_cam * 9;
    for (int64_t i = 0; i < n_cam * 9; ++i) out[i] += acc[i];
  }
  free(part);
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
