// Internal definitions shared by the libpoba translation units.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/poba.h"

namespace poba {

// ---- fixed geometry of the landmark-tile kernels --------------------------------
constexpr int kTile = 256;        // observations per tile == threads per CTA
constexpr int kSlotCap = 1536;    // max distinct cameras per chunk (smem accumulators)
constexpr int kCamChunk = 128;    // observations per camera-major reduction chunk
constexpr int kJPlanes = 12;      // double2 planes: 9 x (Jp[0][j],Jp[1][j]) + 3 x (Jl[0][b],Jl[1][b])

// Error plumbing ---------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define PCK(call)                                                                     \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return ::poba::fail(POBA_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
// NCCL is resolved at run time (dlopen) and only for sharded contexts, so the
// library never pins a libnccl.so.2 into a process that also loads PyTorch's.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
const NcclApi* nccl_api();  // nullptr (error set) when libnccl cannot be loaded

#define PNCCL(call)                                                                   \
  do {                                                                                \
    const ::poba::NcclApi* api_ = ::poba::nccl_api();                                 \
    if (!api_) return POBA_ENCCL;                                                     \
    ncclResult_t r_ = api_->call;                                                     \
    if (r_ != ncclSuccess)                                                            \
      return ::poba::fail(POBA_ENCCL, std::string(#call) + ": " + api_->GetErrorString(r_)); \
  } while (0)
#define PTRY(call)            \
  do {                        \
    int s_ = (call);          \
    if (s_ != POBA_OK) return s_; \
  } while (0)

// A device buffer that frees itself.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  int alloc(size_t n) {  // (re)allocate, contents undefined
    if (n <= bytes && p) return POBA_OK;
    release();
    if (n == 0) n = 16;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess)
      return fail(POBA_ECUDA, std::string("cudaMalloc ") + std::to_string(n) + " B: " + cudaGetErrorString(e));
    bytes = n;
    return POBA_OK;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Device-side flags of the running series solve.
struct SeriesState {
  int stopped;       // 1 once the stop test fired / zero rhs / error
  int order_used;
  int converged;
  int error;         // 0, POBA_ENONFINITE or POBA_EVANISH
  int error_order;
  int any_nonzero;   // back-substitution: dx_p or dx_l non-zero
  unsigned ticket;   // last-block-done counter
  unsigned ticket2;
};

// Per-tile descriptor (landmark-aligned, all landmarks of one tile share k).
struct Tile {
  int obs0;    // first local observation
  int n;       // observations in tile
  int k;       // track length of its landmarks (k > kTile: one sub-range of a long landmark)
  int lm0;     // first local landmark
  int nlm;     // landmarks in tile (1 for long sub-tiles)
  int seg0;    // first segment of the tile in the segment arrays
  int nseg;    // number of (camera) segments
  int chunk;   // owning chunk
};

struct Chunk {
  int tile0, tile1;  // tile range
  int part0;         // first partial (slot 0)
  int nslot;         // distinct cameras (slots)
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  int n_sm = 148;
  int64_t launches = 0;

  // global sizes
  int64_t n_cam = 0, n_pt = 0, n_obs = 0;
  bool have_problem = false, have_lin = false, have_damp = false, have_solution = false,
       have_delta_l = false, have_points = false, have_pixels = false;
  int k_max = 0;

  // global ordering (kept for export; K0)
  DBuf order;        // int64 [n_obs] canonical -> file index
  DBuf cam_file;     // int32 [n_obs] file-order camera index
  DBuf pt_file;      // int32 [n_obs] file-order point index
  std::vector<int64_t> grp_k, grp_start, grp_n;  // k-groups (host)

  // local shard
  int64_t obs_lo = 0, obs_hi = 0, lm_lo = 0, lm_hi = 0;
  int64_t n_obs_l = 0, n_lm_l = 0, obs_pad = 0;
  DBuf cam_l;        // int32 [n_obs_l] camera of each local observation (canonical order)
  DBuf pix_l;        // double2 [n_obs_l] pixels, canonical order
  DBuf file_l;       // int32 [n_obs_l] file index of each local observation
  DBuf lm_pt;        // int32 [n_lm_l] point id of each local landmark
  DBuf lm_off;       // int32 [n_lm_l+1] local obs offset
  DBuf pt_to_lm;     // int32 [n_pt] local landmark of a point, -1 if not local

  // tiles / chunks / camera-slot map
  int n_tiles = 0, n_chunks = 0, n_partials = 0, max_slots = 0, n_long = 0, n_segs = 0;
  DBuf tiles;        // Tile [n_tiles]
  DBuf chunks;       // Chunk [n_chunks]
  DBuf perm;         // uint8 [n_obs_l] tile-local position sorted by camera
  DBuf seg_start;    // uint16 [n_segs]
  DBuf seg_slot;     // uint16 [n_segs]
  DBuf part_cam_off; // int32 [n_cam+1] camera -> range in part_idx
  DBuf part_idx;     // int32 [n_partials] partial indices per camera, chunk order
  DBuf long_lm;      // int32 [n_long] local landmark ids with k > kTile
  DBuf long_zb;      // double [n_long*3] per long landmark z (V^-1 y)
  std::vector<int> long_host;  // host copy of long landmarks
  // camera-major reduction chunks over cperm
  int n_cchunks = 0;
  DBuf cperm;        // int32 [n_obs_l] local obs sorted by (camera, obs)
  DBuf cc_start;     // int32 [n_cchunks]
  DBuf cc_cam_off;   // int32 [n_cam+1] camera -> cchunk range

  // store (K1)
  DBuf J;            // double2 [kJPlanes][obs_pad]
  DBuf Rz;           // double2 [obs_pad] residuals

  // camera arrays
  DBuf cams;         // double [n_cam*9] current linearization cameras
  DBuf cams_prep;    // double [n_cam*16] R (9), t (3), f, k1, k2, pad
  DBuf cams_trial;   // double [n_cam*9]
  DBuf trial_prep;   // double [n_cam*16]
  DBuf U0;           // double [n_cam*45] packed upper
  DBuf bp;           // double [n_cam*9]
  DBuf Dp;           // double [n_cam*9]
  DBuf Uinv;         // double [n_cam*45]
  DBuf Ud;           // double [n_cam*45] damped U
  DBuf bt;           // double [n_cam*9] b_tilde
  DBuf tvec;         // double [n_cam*9] current term
  DBuf xvec;         // double [n_cam*9] partial sum
  DBuf rvec;         // double [n_cam*9] reduced camera vector (pre U^-1)
  DBuf cc_part;      // double [n_cchunks*54]
  DBuf partials;     // double [n_partials*9]
  DBuf blk_part;     // double [blocks*4] per-block reduction partials
  DBuf state;        // SeriesState
  DBuf state_aux;    // SeriesState for side computations (b_tilde read-back)
  DBuf ratios;       // double [max_order+1]
  int ratios_cap = 0;

  // landmark arrays (local, canonical landmark order)
  DBuf points;       // double [n_lm_l*3]
  DBuf V0;           // double [n_lm_l*6] packed
  DBuf bl;           // double [n_lm_l*3]
  DBuf Dl;           // double [n_lm_l*3]
  DBuf Vinv;         // double [n_lm_l*6]
  DBuf Vd;           // double [n_lm_l*6] damped V
  DBuf dl;           // double [n_lm_l*3] last delta_l
  DBuf ltmp;         // double [n_lm_l*3] scratch
  DBuf ctmp;         // double [n_cam*9] scratch
  DBuf ctmp2;        // double [n_cam*9]
  DBuf flag;         // int [4]
  DBuf red;          // double scratch for reductions
  DBuf cub_tmp;      // CUB temp storage

  double lam = 0;
  int identity = 0;
  int64_t n_invalid = 0;
  int last_order = 0;

  // host staging
  DBuf scratch_a, scratch_b, scratch_c, scratch_d;
};

// ---- host-side orchestration entry points (defined per translation unit) ------
int build_structure(Ctx& c, const int64_t* cam_idx, const int64_t* pt_idx, const double* pixels);
int linearize_device(Ctx& c, bool explicit_jac, const double* jp, const double* jl, const double* res);
int damp_device(Ctx& c, double lam, int identity);
int series_device(Ctx& c, double eps, int max_order, bool forced, int* order_used, int* converged);
int series_apply_device(Ctx& c, const double* d_v, int order, double* d_out);
int back_substitute_device(Ctx& c, const double* d_delta_p, int* nonzero);
int cost_device(Ctx& c, bool trial, double* cost, int64_t* n_invalid);
int apply_op_device(Ctx& c, int op, const double* d_in, double* d_out);
int cameras_prep(Ctx& c, const double* d_cams, double* d_prep);
int allreduce_sum(Ctx& c, double* d_buf, size_t n);
int time_terms_device(Ctx& c, int reps, double* ms_per_term, double* ms_term_kernel, int* launches);
int b_tilde_device(Ctx& c);
int points_accept_device(Ctx& c);
int points_scatter_to_host(Ctx& c, const double* d_lm3, double* host_pt3);
int points_gather_from_host(Ctx& c, const double* host_pt3, double* d_lm3);

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace poba
