/*
 * libpoba -- B200-native (sm_100a, fp64) power-series Schur solve for bundle
 * adjustment, the hot path of Power Bundle Adjustment (arXiv 2204.12834).
 *
 * Plain C ABI: opaque context, plain pointers and sizes, no torch types.  The
 * Python host layer (paper_2204_12834_b200/_lib.py) binds it with ctypes.  The
 * reference is a pure-Python package; each entry point below replaces the
 * reference function cited beside it (paths relative to
 * /root/reference/pkg/src/powerba/), and INTEGRATION.md shows the ctypes
 * binding a powerba maintainer would add.
 *
 * Every function returns a status code (POBA_OK = 0).  On failure
 * poba_last_error() returns a thread-local message; the Python layer maps
 * POBA_EINVAL / POBA_ENOTSPD / POBA_ENONFINITE / POBA_EVANISH to ValueError
 * with the reference's own messages.
 *
 * Arrays: observation arrays are in the caller's (file) order, cameras are
 * (n_cam, 9) row-major BAL order [rotvec, t, f, k1, k2], points (n_pt, 3),
 * pixels (n_obs, 2), pose vectors 9*n_cam, landmark vectors 3*n_pt -- exactly
 * the reference's BalProblem layout (bal_io.py:55-78).  Inputs are copied at
 * call time and never aliased after return.
 */
#ifndef POBA_H
#define POBA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POBA_OK 0
#define POBA_EINVAL 1     /* invalid argument / problem structure         */
#define POBA_ENOTSPD 2    /* damped pose or point block not SPD           */
#define POBA_ENONFINITE 3 /* non-finite series iterate (order in message) */
#define POBA_ECUDA 4      /* CUDA runtime error                            */
#define POBA_ENCCL 5      /* NCCL error                                    */
#define POBA_EVANISH 6    /* vanishing iterate norm with nonzero rhs       */
#define POBA_EPARSE 7     /* malformed BAL text (message as BalParseError) */

typedef struct poba_ctx poba_ctx;

/* thread-local message of the last failing call on this thread */
const char* poba_last_error(void);
int poba_version(void);

/* ---- context ------------------------------------------------------------
 * One context per process and GPU.  poba_create_sharded() joins an NCCL
 * communicator of nranks processes (one per GPU); landmarks and their
 * observations are partitioned across ranks, cameras are replicated, and
 * every series term ends in one all-reduce of the 9*n_cam camera vector.   */
int poba_create(int device, poba_ctx** out);
int poba_nccl_unique_id(void* out_128_bytes);
int poba_create_sharded(int device, int rank, int nranks, const void* nccl_id_128_bytes,
                        poba_ctx** out);
int poba_destroy(poba_ctx* ctx);
/* In-process virtual ranks on one device (testing the sharded path with fewer
 * GPUs than ranks): a group of nranks (<= 8) contexts, each driven by its own
 * host thread, whose collectives meet at a host barrier and reduce every
 * rank's buffer in rank order -- the same partition, store and replicated
 * camera-side decisions as poba_create_sharded, with the exchange done
 * without NCCL.  The group must outlive its contexts.                      */
int poba_local_group_create(int nranks, void** group);
int poba_local_group_destroy(void* group);
int poba_create_local(int device, int rank, int nranks, void* group, poba_ctx** out);

/* ---- K0: observation store structure -------------------------------------
 * Replaces blocks._sorted_observation_order (blocks.py:362-372) and
 * blocks._build_groups (blocks.py:405-417): canonical (k, landmark, camera)
 * order by a stable device radix sort, landmark-aligned tiles, the chunked
 * camera-slot map used by the deterministic camera reductions, and (sharded)
 * this rank's landmark range.  pixels may be NULL (explicit-Jacobian use).   */
int poba_set_problem(poba_ctx* ctx, int64_t n_cam, int64_t n_pt, int64_t n_obs,
                     const int64_t* cam_idx, const int64_t* pt_idx, const double* pixels);
/* Block-storage precision (PoBA-32 / PoBA-64, blocks.py:42-47 `precision`):
 * 32 keeps the Jacobian rows and residuals rounded to fp32 (half the bytes per
 * series term) while every sum stays fp64, as the reference's float32 storage
 * with float64 einsums.  Invalidates the linearization; default 64.          */
int poba_set_precision(poba_ctx* ctx, int bits);
/* info[0..15]: n_groups, n_tiles, n_chunks, n_partials, obs_lo, obs_hi, lm_lo,
 * lm_hi, max_slots, n_long, device_bytes, k_max, n_cam, n_pt, n_obs, rank   */
int poba_problem_info(poba_ctx* ctx, int64_t* info);
/* Camera-side layout the store build chose for the fused term kernel (no
 * reference counterpart; a measurement aid): *table = 1 when the chunk's term
 * records are kept in a per-CTA shared-memory table (camera working set of a
 * CTA range fits: C1-C4), 0 when every tile gathers its records (C5).        */
int poba_term_layout(poba_ctx* ctx, int* table);
/* order / cam_sorted / pt_sorted (n_obs each): bit-exact with the reference */
int poba_get_ordering(poba_ctx* ctx, int64_t* order, int64_t* cam_sorted, int64_t* pt_sorted);
/* k-groups (k ascending): group k, first canonical observation, #landmarks */
int poba_get_groups(poba_ctx* ctx, int64_t cap, int64_t* n_groups, int64_t* group_k,
                    int64_t* group_start, int64_t* group_n);

/* ---- K1-K3: linearization -------------------------------------------------
 * blocks.linearize (blocks.py:293-324) + _finish_linearization (375-402):
 * residual + analytic Jacobians (camera.evaluate, camera.py:67-135), the
 * landmark-major store, V0/b_l per landmark, U0/b_p per camera (deterministic
 * segmented reductions, no atomics), Marquardt diagonals D_p/D_l.
 * points == NULL uses the device-resident points (poba_set_points).        */
int poba_linearize(poba_ctx* ctx, const double* cam_params, const double* points,
                   int64_t* n_invalid);
/* blocks.assemble_from_observations (blocks.py:333-352): explicit per-observation
 * j_pose (n_obs,2,9), j_point (n_obs,2,3), residuals (n_obs,2) in file order.  */
int poba_linearize_explicit(poba_ctx* ctx, const double* j_pose, const double* j_point,
                            const double* residuals);

/* ---- K2-K4: damping ---------------------------------------------------------
 * DampedSystem.__init__ (blocks.py:164-192) with _spd_block_inverse (277-285):
 * U = U0 + lam diag(D_p^2), V = V0 + lam diag(D_l^2) (identity != 0: D = 1),
 * batched 9x9 / 3x3 Cholesky inverses.                                       */
int poba_damp(poba_ctx* ctx, double lam, int identity);

/* ---- K4-K6: power-series solve ---------------------------------------------
 * power_series_solve (power_series.py:53-77): b_tilde = b_p - W V^-1 b_l
 * (blocks.py:256-260), t0 = U^-1(-b_tilde), t_i = U^-1 W V^-1 W^T t_{i-1},
 * x_i = x_{i-1} + t_i, stop when (i+1)||x_i - x_{i-1}||/||x_i|| < epsilon
 * (power_series.py:29-42) -- evaluated on the device, the whole loop enqueued
 * (CUDA graph) without host round trips.  ratios (nullable, max_order+1
 * doubles) receives the stop ratio per order (NaN where not evaluated).      */
int poba_series_solve(poba_ctx* ctx, double epsilon, int max_order, double* delta_p,
                      int* order_used, int* converged, double* ratios);
/* apply_series_inverse (power_series.py:80-91): fixed order, no stop test.  */
int poba_series_apply(poba_ctx* ctx, const double* v, int order, double* out);

/* ---- K7: back-substitution (power_series.py:94-100) -------------------------
 * dx_l = -V^-1 (b_l + W^T dx_p); delta_p NULL = the last series solution.
 * delta_l (nullable) is scattered to point-index order (3*n_pt; sharded: only
 * this rank's landmarks are written).  nonzero: 1 if dx_p or dx_l != 0.      */
int poba_back_substitute(poba_ctx* ctx, const double* delta_p, double* delta_l, int* nonzero);

/* ---- PCG baselines on the same operators (solvers.py:30-118) --------------
 * poba_schur_diagonal: the exact 9x9 diagonal blocks of S = U - W V^-1 W^T of
 * the damped system (schur_diagonal_blocks, solvers.py:71-85), written as
 * n_cam full row-major 9x9 blocks (nullable: only prepare the inverses).
 * poba_pcg: preconditioned CG on S dx_p = -b_tilde (pcg, solvers.py:30-64)
 * with the Schur-Jacobi preconditioner (pcg_schur_jacobi, solvers.py:98-102)
 * or the order-`order` power-series preconditioner
 * (pcg_power_series_preconditioner, solvers.py:105-118).  Stops when
 * sqrt(r^T M^-1 r / r0^T M^-1 r0) < tol or after max_iter iterations.
 * resume != 0 continues the previous solve for up to max_iter more
 * iterations (the Python layer uses it to honour a per-iteration callback).
 * rel_history (nullable, max_iter entries) receives the relative residual of
 * each iteration of this call.  The solution also becomes the device-side
 * delta_p used by poba_back_substitute(ctx, NULL, ...).
 * POBA_ENOTSPD: "Schur diagonal blocks are not positive definite",
 * "preconditioner is not positive definite", "reduced system is not positive
 * definite" (the reference's asserts).                                      */
#define POBA_PRECOND_SCHUR_JACOBI 1
#define POBA_PRECOND_SERIES 2
int poba_schur_diagonal(poba_ctx* ctx, double* blocks_81);
int poba_pcg(poba_ctx* ctx, int precond, int order, double tol, int max_iter, int resume, double* delta_p,
             int* iterations, double* final_rel, int* converged, double* rel_history);

/* ---- K8: cost (lm.residual_cost, lm.py:107-119) ------------------------------
 * 0.5 sum ||r||^2 and the invalid count.  points NULL: device points, plus
 * the last back-substituted delta_l when trial != 0 (lm.apply_update,
 * lm.py:132-144, points part).                                               */
int poba_cost(poba_ctx* ctx, const double* cam_params, const double* points, int trial,
              double* cost, int64_t* n_invalid);

/* ---- device-resident landmark state ------------------------------------------ */
int poba_set_points(poba_ctx* ctx, const double* points);
int poba_accept_points(poba_ctx* ctx); /* points += last delta_l (lm.py:140) */
int poba_get_points(poba_ctx* ctx, double* points);
/* every rank's rows (sharded contexts; collective: all ranks call it) -- the
   state lm.run returns (lm.py:228-232, BaState) */
int poba_get_points_all(poba_ctx* ctx, double* points);

/* ---- operator passes (DampedSystem.apply_*, blocks.py:214-254) --------------- */
#define POBA_OP_W 0      /* (3 n_pt) -> (9 n_cam)   */
#define POBA_OP_WT 1     /* (9 n_cam) -> (3 n_pt)   */
#define POBA_OP_U_INV 2  /* (9 n_cam) -> (9 n_cam)  */
#define POBA_OP_V_INV 3  /* (3 n_pt) -> (3 n_pt)    */
#define POBA_OP_U 4      /* (9 n_cam) -> (9 n_cam)  */
#define POBA_OP_SCHUR 5  /* (9 n_cam) -> (9 n_cam)  */
#define POBA_OP_WVW 6    /* (9 n_cam) -> (9 n_cam): W V^-1 W^T, one fused pass (spectral.py power iteration) */
int poba_apply(poba_ctx* ctx, int op, const double* in, double* out);

/* ---- read-back of assembled quantities (parity tests, attributes) ----------- */
#define POBA_READ_U0 0      /* n_cam x 9 x 9 */
#define POBA_READ_V0 1      /* n_pt x 3 x 3  */
#define POBA_READ_B_P 2     /* 9 n_cam       */
#define POBA_READ_B_L 3     /* 3 n_pt        */
#define POBA_READ_D_P 4     /* n_cam x 9     */
#define POBA_READ_D_L 5     /* n_pt x 3      */
#define POBA_READ_U 6       /* n_cam x 9 x 9 (damped) */
#define POBA_READ_V 7       /* n_pt x 3 x 3  */
#define POBA_READ_U_INV 8   /* n_cam x 9 x 9 */
#define POBA_READ_V_INV 9   /* n_pt x 3 x 3  */
#define POBA_READ_B_TILDE 10 /* 9 n_cam      */
#define POBA_READ_STORAGE 11 /* n_obs x 2 x 13, canonical order (local obs) */
int poba_read(poba_ctx* ctx, int what, double* dst);

/* ---- instrumentation ------------------------------------------------------------
 * Time `reps` forced series terms (no stop test) with CUDA events on the
 * library stream; ms_per_term receives the mean.  launches: kernel launches
 * per term.  Used by bench.py for the roofline figure.                       */
/* Spectral radius of P = U^-1 W V^-1 W^T by power iteration on the similar
   symmetric U^-1/2 W V^-1 W^T U^-1/2, from the unit start vector v0 (9 n_cam),
   stop when |rho_i - rho_{i-1}| <= tol |rho_i| (spectral.py:54-86,
   estimate_spectral_radius); U^-1/2 per camera on the device; one fused term
   pass per step. */
int poba_spectral_radius(poba_ctx* ctx, const double* v0, double tol, int max_iter, double* rho,
                         int* iterations, int* converged);
/* Dense (9 n_cam)^2 matrix of a camera-space operator (POBA_OP_SCHUR, _WVW, _U,
   _U_INV), column-major: out[j*dim + i] = (Op e_j)_i; refused (status 1) above
   `limit` pose parameters.  Replaces the host basis-vector loops of
   materialize_schur (solvers.py:124-133) and spectral._dense_operator. */
int poba_materialize(poba_ctx* ctx, int op, int64_t limit, double* out);
int poba_time_terms(poba_ctx* ctx, int reps, double* ms_per_term, double* ms_term_kernel,
                    int* launches);
/* kernel launches issued by the library since creation (all entry points)  */
int64_t poba_launch_count(poba_ctx* ctx);
/* the cudaStream_t every kernel of this context runs on (for external events) */
int poba_stream(poba_ctx* ctx, void** stream);
/* landmark bounds [lm_bounds[r], lm_bounds[r+1]) of each rank's shard, as
 * poba_create_sharded contexts choose them (host-only, callable without a GPU) */
int poba_shard_bounds(int64_t n_pt, const int64_t* k_per_point, int nranks, int64_t* lm_bounds);

/* ---- PoST clustered solve (clustering.py:49-148) ------------------------------
 * poba_cluster_cameras: host-only greedy covisibility clustering
 * (cluster_cameras): assignment[n_cam], cluster count, cut observations.
 * The clustered pose solve runs on a context whose store holds one virtual
 * landmark per (landmark, cluster) pair: poba_set_dl installs the global
 * landmark damping diagonal (restrict_system keeps it), and
 * poba_series_solve_clustered runs every cluster's truncated series at once
 * with per-cluster stop tests (solve_clustered): order_used = max, converged
 * = all.                                                                      */
int poba_cluster_cameras(int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_idx, const int64_t* pt_idx,
                         int64_t max_cluster_size, int64_t* assignment, int64_t* n_clusters,
                         int64_t* cut_observations);
int poba_set_dl(poba_ctx* ctx, const double* d_l);
int poba_series_solve_clustered(poba_ctx* ctx, const int64_t* cluster_of_cam, int n_clusters, double epsilon,
                                int max_order, double* delta_p, int* order_used, int* converged);

/* ---- native BAL ingest (bal_io.parse_bal / _parse_lines, bal_io.py:180-260) --
 * Parses BAL text from a path (text-mode line endings) or from an in-memory
 * buffer (lines end at '\n'), with the reference's token grammar (Python int()
 * / float()), validation order, pruning of unreferenced cameras and points, and
 * line-numbered messages (POBA_EPARSE).  Host only; no GPU needed.
 * info: n_cam, n_pt, n_obs (after pruning), n_pruned_cameras, n_pruned_points.  */
typedef struct poba_bal poba_bal;
int poba_bal_parse(const char* path, const char* text, int64_t text_len, poba_bal** out);
int poba_bal_info(const poba_bal* bal, int64_t* info5);
int poba_bal_copy(const poba_bal* bal, double* cams, double* points, int64_t* cam_idx, int64_t* pt_idx,
                  double* pixels);
int poba_bal_free(poba_bal* bal);

#ifdef __cplusplus
}
#endif
#endif /* POBA_H */
