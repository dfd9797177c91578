// Internal definitions shared by the libpoba translation units.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cassert>
#include <cstdint>
#include <string>
#include <vector>

// Device-side bounds checks (index < bound on every gathered / scattered
// table): compiled in with -DPOBA_DEVICE_CHECKS for the checked build the GPU
// tests run against (tools/build_variant.sh checked -DPOBA_DEVICE_CHECKS);
// compute-sanitizer is not available on the GPU pool.
#ifdef POBA_DEVICE_CHECKS
#define POBA_DCHECK(cond) assert(cond)
#else
#define POBA_DCHECK(cond) ((void)0)
#endif

#include "../../include/poba.h"

namespace poba {

// ---- fixed geometry ------------------------------------------------------------
// The device store is landmark-major in "slot space": warp-tile t owns slots
// [t*kTile, t*kTile + n_t); a warp-tile packs whole landmarks (index order, each
// landmark's observations sorted by camera) up to kTile observations and kTileLm
// landmarks; a landmark with k > kTile spans consecutive full sub-tiles.  Each
// warp-tile is one contiguous block: a 128-B metadata array (one 32-bit word
// per slot: chunk slot of the camera, landmark index in the tile, first and
// last lane of the landmark's run) followed by 12 planes of 32 column pairs --
// plane p holds column pair p of every slot's 2x12 Jacobian row (J_p: 9 pairs,
// J_l: 3 pairs), i.e. the reference's 2x13 block row without the residual
// column (residuals live in their own array; the series never reads them).
// A warp reads plane p with 32 consecutive 16-B accesses (coalesced in global
// memory, conflict-free in shared memory), and the tile's copy ends at plane
// 11's last valid slot.
constexpr int kTile = 32;         // observation slots per warp-tile (one warp)
constexpr int kTileLm = 16;       // landmarks per warp-tile (bounds the staged V^-1 slice)
constexpr int kMetaBytes = kTile * 4;                 // per-tile metadata words
constexpr int kTileBlock = kMetaBytes + 12 * kTile * 16;  // 6272 B per warp-tile (fp64 planes)
constexpr int kTileBlockF32 = kMetaBytes + 12 * kTile * 8;  // 3200 B (fp32 planes, PoBA-32)
constexpr int kBlockTiles = 8;    // warp-tiles per CTA in the streaming kernels (256 threads)
#ifndef POBA_CAM_CHUNK
#define POBA_CAM_CHUNK 1024
#endif
constexpr int kCamChunk = POBA_CAM_CHUNK;  // observations per camera-major reduction chunk
constexpr int kJPlanes = 12;      // Jacobian column pairs per row
#ifndef POBA_TERM_WARPS
#define POBA_TERM_WARPS 12
#endif
constexpr int kTermWarps = POBA_TERM_WARPS;  // warps per CTA of the term kernel
#ifndef POBA_TERM_CTAS
#define POBA_TERM_CTAS 1
#endif
// co-resident term-kernel CTAs per SM, each with its own tile range, accumulator table and apply-turn
// ring.  1 is the measured optimum (profiles/r02a_term_cta_shapes.md: 2 x 6 warps and 3 x 4 warps are
// 4-9% slower on C5 and double / triple the chunk partials).
constexpr int kTermCtas = POBA_TERM_CTAS;
constexpr int kPackWindow = 64;   // landmark lookahead of the tile packer
constexpr int kTStride = 10;      // doubles per camera record of the term vector / partials (80 B, 16-B aligned)
// Term-kernel shared memory: per warp one bulk-copy stage (the tile block, the
// tile descriptor, the V^-1 slice of its <= kTileLm landmarks) and the gathered
// camera records of its tile; per CTA the chunk accumulator table (one 80-B
// record per camera slot of the chunk), the stage barriers and the turn word.
constexpr int kStDesc = kTileBlock;                              // 32-B tile descriptor
constexpr int kStVinv = kStDesc + 32;                            // V^-1 slice
constexpr int kStageBytes = kStVinv + kTileLm * 48;              // 7072
constexpr int kTRecBytes = kTStride * 8;                         // 80
// Two layouts of the camera side, chosen per context when the store is built
// (Ctx::chunk_t):
//   gather (CT = false)  every warp gathers the 32 term records of its next
//                        tile from L2 into a per-warp table; the accumulator
//                        table gets all the remaining shared memory (1440 slots)
//   table  (CT = true)   the term records of the chunk's cameras sit in a
//                        second per-CTA table next to the accumulator table,
//                        loaded once per chunk by all warps and read by slot
//                        (no per-tile gather); 896 slots, so chunks are
//                        smaller -- chosen when a CTA range's camera working
//                        set still fits (C1-C4), not on C5
// one CTA: the 227-KB per-CTA limit; several: an equal share of the SM's 228 KB less the 1 KB reserved per CTA
constexpr int kTermSmemMax = kTermCtas == 1 ? 227 * 1024 : (228 * 1024) / kTermCtas - 1024;
#ifndef POBA_TERM_WARPS_TABLE
#define POBA_TERM_WARPS_TABLE 12  // 13 / 14 warps fit its 145 registers but measured 12% slower on C4 and C3 (smaller table, 128-register build)
#endif
template <bool CT>
struct TermShape {
  static constexpr int kWarps = CT ? POBA_TERM_WARPS_TABLE : kTermWarps;        // warps per CTA
  static constexpr int kCtl = kWarps * 16 + 16;                                 // full + empty stage barriers + pad
  static constexpr int kWarpSmem = kStageBytes + (CT ? 0 : kTile * kTRecBytes);  // stage (+ per-warp record table)
  static constexpr int kSlotBytes = CT ? 2 * kTRecBytes : kTRecBytes;           // accumulator (+ term record)
  static constexpr int kAccSlots = ((kTermSmemMax - kWarps * kWarpSmem - kCtl) / kSlotBytes) / 32 * 32;
  static constexpr int kTermSmem = kWarps * kWarpSmem + kCtl + kAccSlots * kSlotBytes;
  static_assert(kTermSmem <= kTermSmemMax, "term kernel shared memory over budget");
  static_assert(kAccSlots < 2048, "chunk slots must fit the 11-bit metadata field");
  static_assert(kWarpSmem % 16 == 0 && kCtl % 16 == 0, "bulk-copy destinations and the tables must be 16-B aligned");
  static_assert(kWarps >= 2 && kWarps <= 14, "the apply turn uses named barriers 1..kWarps (ring of >= 2), the chunk barrier 15");
};
static_assert(kStageBytes % 16 == 0, "bulk-copy destinations must be 16-B aligned");
// the table layout is taken when it needs at most this many times the gather layout's chunk partials
constexpr double kChunkTMaxGrowth = 3.0;  // C4: 2.1x the partials, kernel -6%; C5 x 0.3: 8x, kernel 2x slower
constexpr int kSlotSlack = 2;   // extra slots per bank colour class in the slot numbering (store.cu)
constexpr int kSlotPasses = 2;  // local-search passes of the slot colouring
constexpr int kLaneRounds = 2;  // rounds of within-run lane ordering + re-colouring (store.cu)

// PoBA-32 (blocks.py:42-47): block storage may be fp32 (planes of float2);
// every value read from it is widened to fp64 and all arithmetic and
// reductions stay fp64.

// metadata word of a slot: chunk slot (bits 0-10), landmark index in the tile
// (11-15; 0 for a long landmark's sub-tile), first (16-20) and last (21-25)
// lane of the landmark's run, apply lane (26-30: the lane whose camera
// contribution this lane adds to the accumulator table, 31: this lane applies;
// carried in the slot word's upper bits, see store.cu)
__host__ __device__ __forceinline__ uint32_t pack_meta(int slot, int li, int first, int last) {
  return (uint32_t)slot | ((uint32_t)li << 11) | ((uint32_t)first << 16) | ((uint32_t)last << 21);
}
__host__ __device__ __forceinline__ int meta_slot(uint32_t m) { return (int)(m & 0x7ffu); }
__host__ __device__ __forceinline__ int meta_li(uint32_t m) { return (int)((m >> 11) & 0x1fu); }
__host__ __device__ __forceinline__ int meta_first(uint32_t m) { return (int)((m >> 16) & 0x1fu); }
__host__ __device__ __forceinline__ int meta_last(uint32_t m) { return (int)((m >> 21) & 0x1fu); }
__host__ __device__ __forceinline__ int meta_apply_src(uint32_t m) { return (int)((m >> 26) & 0x1fu); }
__host__ __device__ __forceinline__ bool meta_apply_on(uint32_t m) { return (m >> 31) != 0u; }
template <bool F32>
constexpr int tile_block_bytes() { return F32 ? kTileBlockF32 : kTileBlock; }
// bytes of a tile's bulk copy: metadata + planes up to plane 11's last valid
// slot (fp32: an even slot count, bulk copies move multiples of 16 B)
template <bool F32>
__host__ __device__ __forceinline__ uint32_t tile_copy_bytes(int n) {
  return F32 ? (uint32_t)(kMetaBytes + (11 * kTile + ((n + 1) & ~1)) * 8)
             : (uint32_t)(kMetaBytes + (11 * kTile + n) * 16);
}

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
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
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
  int any_nonzero;   // -1: zero right-hand side shortcut
  unsigned ticket;   // last-block-done counter
  unsigned ticket2;
};

// Per-tile descriptor.
struct Tile {
  int obs0;    // first local observation (prefix count over tiles; slots are tile*kTile)
  int n;       // observations in tile
  int lm0;     // first local landmark
  int nlm;     // landmarks in tile (1 for a sub-tile of a long landmark)
  int chunk;   // owning chunk
  int flags;   // kTileLong | kTileDupCam | kTileChunkLast
};
constexpr int kTileLong = 1;      // sub-tile of a landmark with k > kTile
constexpr int kTileDupCam = 2;    // some camera appears twice in the tile
constexpr int kTileChunkLast = 4; // last tile of its chunk: write the partials after applying it
constexpr int kTileScanShift = 8; // bits 8-10: segmented-scan steps, ceil(log2(longest landmark run))

// Compact per-tile descriptor streamed into the term kernel's stage (32 B).
struct TileK {
  int n, lm0, nlm, flags;
  int part0, nslot;  // the owning chunk's partials
  int nx_n, nx_lm0;  // copy sizes of the same warp's next tile (n | nlm << 8), 0 if none
};

// A chunk: contiguous tiles of one CTA whose distinct cameras fit kAccSlots.
struct Chunk {
  int tile0, tile1;  // tile range
  int part0;         // first partial (slot 0)
  int nslot;         // distinct cameras (slots)
};

// An instantiated CUDA graph of one complete series solve (b_tilde + m terms,
// device-side stop test), replayed while the problem's buffers stay put.
struct SeriesGraph {
  cudaGraphExec_t exec = nullptr;
  double eps = 0;
  int max_order = 0;
  bool forced = false;
  const void* ratios = nullptr;
  int64_t launches = 0;
};

// pipelined landmark transfers: file-order pieces, used when a single-GPU
// context moves at least kXferMinBytes of landmark rows
constexpr int kXferPieces = 8;
constexpr size_t kXferMinBytes = 16u << 20;

// host-side state of a (resumable) device PCG solve
struct PcgState {
  bool active = false;
  int precond = 0, order = 0, it = 0;
  double rz = 0, rz0 = 0, rel = 0;
};

// in-process group of virtual ranks sharing one device (api.cu): stands in
// for the NCCL communicator when fewer GPUs than ranks are available
constexpr int kMaxLocalRanks = 8;
struct LocalGroup;

struct Ctx {
  int device = 0;
  int precision = 64;  // block storage: 64 (double2 rows) or 32 (float2 rows)
  cudaStream_t stream = nullptr;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  LocalGroup* group = nullptr;  // set instead of comm for in-process virtual ranks
  DBuf coll_tmp;                // local-group collective result scratch
  DBuf xch_send, xch_recv;      // rank-ordered all-reduce: padded slices out / in
  int64_t cam_ls = 0;           // sharded: cameras per rank slice of the camera step (>= 4)
  int n_sm = 148;
  bool chunk_t = false;         // term-kernel camera-side layout of this store (TermShape<chunk_t>)
  bool graph_off = false;       // sharded NCCL context whose series capture failed once: enqueue from then on
  int64_t launches = 0;

  // global sizes
  int64_t n_cam = 0, n_pt = 0, n_obs = 0;
  bool have_problem = false, have_lin = false, have_damp = false, have_solution = false,
       have_delta_l = false, have_points = false, have_pixels = false;
  int k_max = 0;

  // global ordering (export only; K0), built lazily
  DBuf cam_file;     // int32 [n_obs] file-order camera index
  DBuf pt_file;      // int32 [n_obs] file-order point index
  DBuf kpt;          // int32 [n_pt] track length
  DBuf order;        // int32 [n_obs] canonical -> file index (lazy)
  bool have_order = false;
  std::vector<int64_t> grp_k, grp_start, grp_n;  // k-groups (host, lazy)

  // local shard: points [lm_lo, lm_hi), its observations, tiles
  int64_t lm_lo = 0, lm_hi = 0, n_lm_l = 0, n_obs_l = 0;
  int64_t n_slots = 0;  // n_tiles * kTile
  int n_tiles = 0, n_chunks = 0, n_partials = 0, max_slots = 0, n_long = 0, n_cta = 0;
  DBuf tiles;        // Tile [n_tiles]
  DBuf tilek;        // TileK [n_tiles]
  DBuf chunks;       // Chunk [n_chunks]
  DBuf cta_tiles;    // int2 [n_cta] tile range of each CTA of the term kernel
  DBuf cam_s;        // int32 [n_slots] camera of each slot
  DBuf file_s;       // int32 [n_slots] file index of each slot (-1 padding)
  DBuf pix_s;        // double2 [n_slots] pixels
  DBuf lidx_s;       // uint8 [n_slots] landmark index within its tile
  DBuf lm_slot0;     // int32 [n_lm_l] first slot of each local landmark
  DBuf lm_k;         // int32 [n_lm_l]
  DBuf lm_perm;      // int32 [n_lm_l] store landmark j -> file-local landmark (lm_lo + lm_perm[j])
  std::vector<int> lm_order_host;
  DBuf lm_stage;     // double staging for landmark uploads/downloads (file order)
  void* host_stage = nullptr;  // pinned host staging for large pageable copies
  size_t host_stage_bytes = 0;
  // pipelined landmark transfers (kXferPieces + 1 cuts each): piece i holds
  // file-local landmarks [xf_file[i], xf_file[i+1]); after it arrives, store
  // landmarks [0, xf_up_lm[i+1]) and tiles [0, xf_up_tile[i+1]) can be formed;
  // store landmarks [0, xf_dn_lm[i+1]) (tiles [0, xf_dn_tile[i+1])) hold every
  // landmark of file pieces 0..i
  std::vector<int64_t> xf_file, xf_up_lm, xf_dn_lm;
  std::vector<int> xf_up_tile, xf_dn_tile;
  DBuf lm_inv;       // int32 [n_lm_l] file-local landmark -> store landmark
  cudaStream_t xfer = nullptr;
  cudaEvent_t xfer_ev[2 * kXferPieces + 1] = {};
  DBuf part_cam_off; // int32 [n_cam+1] camera -> range in part_idx
  DBuf part_idx;     // int32 [n_partials] partial indices per camera, chunk order
  DBuf part_cam;     // int32 [n_partials] camera of each partial (-1: hole of the slot numbering)
  DBuf long_lm;      // int32 [n_long] local landmarks with k > kTile
  std::vector<int> long_host;
  std::vector<Chunk> chunks_host;
  // camera-major reduction chunks
  int n_cchunks = 0;
  DBuf cperm;        // int32 [n_obs_l] slots sorted by (camera, slot)
  DBuf lm_c;         // int32 [n_obs_l] store landmark of each camera-major position (U0 / b_p pass)
  DBuf pix_c;        // double2 [n_obs_l] its pixel
  DBuf file_c;       // int32 [n_obs_l] its file index (explicit-Jacobian systems)
  DBuf cam_start;    // int32 [n_cam+1] camera -> first position in cperm
  DBuf cc_cam_off;   // int32 [n_cam+1] camera -> cchunk range
  DBuf cc_cam;       // int32 [n_cchunks] cchunk -> camera

  // store (K1), slot space
  DBuf J;            // [n_tiles] tile blocks (metadata + 12 planes): double2 planes, or float2 at precision 32
  DBuf slot_s;       // int32 [n_slots] chunk slot of each observation's camera (metadata source)
  DBuf Rz;           // double2 [n_slots] residuals

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
  DBuf tvec;         // double [n_cam*kTStride] current term (80-B records)
  DBuf xvec;         // double [n_cam*9] partial sum
  DBuf rvec;         // double [n_cam*9] reduced camera vector (pre U^-1)
  DBuf cc_part;      // double [n_cchunks*54]
  DBuf partials;     // double [n_partials*kTStride]
  DBuf blk_part;     // double [blocks*4] per-block reduction partials
  DBuf state;        // SeriesState
  DBuf state_aux;    // SeriesState for side computations (b_tilde read-back)
  DBuf ratios;       // double [max_order+1]
  int ratios_cap = 0;

  // landmark arrays (local, point order)
  DBuf points;       // double [n_lm_l*3]
  DBuf V0;           // double [n_lm_l*6] packed
  DBuf bl;           // double [n_lm_l*3]
  DBuf Dl;           // double [n_lm_l*3]
  DBuf Vinv;         // double [n_lm_l*6]
  DBuf Vd;           // double [n_lm_l*6] damped V
  DBuf dl;           // double [n_lm_l*3] last delta_l
  DBuf ltmp;         // double [n_lm_l*3] scratch / z of long landmarks
  DBuf ctmp;         // double [n_cam*kTStride] scratch
  DBuf ctmp2;        // double [n_cam*kTStride]
  DBuf wt_in;        // double [n_cam*kTStride] camera input of the W^T tile pass
  DBuf flag;         // int [16]
  DBuf red;          // double scratch for reductions
  DBuf cub_tmp;      // CUB temp storage

  double lam = 0;
  int identity = 0;
  int64_t n_invalid = 0;
  int last_order = 0;

  DBuf scratch_a, scratch_b, scratch_c;
  DBuf Mbuf;         // double [n_cam*45] Schur diagonal blocks (PCG)
  DBuf Minv;         // double [n_cam*45] their inverses
  DBuf pcg_vec;      // double [5*9*n_cam] x, r, z, p, S p
  PcgState pcg;
  std::vector<SeriesGraph> graphs;
  void drop_graphs() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  ~Ctx() {
    drop_graphs();
    for (auto& e : xfer_ev)
      if (e) cudaEventDestroy(e);
    if (xfer) cudaStreamDestroy(xfer);
    if (host_stage) cudaFreeHost(host_stage);
  }
};

// ---- host-only planning (no GPU needed) ------------------------------------------
struct TilePlan {
  std::vector<int64_t> lm_first;       // first observation of each landmark (store order)
  std::vector<Tile> tiles;             // global warp-tiles
  std::vector<char> cut_ok;            // may a shard boundary sit before this tile?
  std::vector<int> lm_tile, lm_off_in_tile;
};
void plan_tiles(const int* k_per_point, int64_t n_pt, TilePlan& plan);
void pack_landmarks(const int* k, int64_t n, int window, std::vector<Tile>& tiles, std::vector<int>& order);
size_t shard_cut(const TilePlan& plan, int64_t n_obs, int r, int nranks);

// ---- host-side orchestration entry points ---------------------------------------
int build_structure(Ctx& c, const int64_t* cam_idx, const int64_t* pt_idx, const double* pixels);
int build_canonical_order(Ctx& c);
// h_points: upload the points (host, file order) pipelined with the Jacobian pass
int linearize_device(Ctx& c, bool explicit_jac, const double* jp, const double* jl, const double* res,
                     const double* h_points = nullptr);
int damp_device(Ctx& c, double lam, int identity);
int series_device(Ctx& c, double eps, int max_order, bool forced, int* order_used, int* converged);
int series_apply_device(Ctx& c, const double* d_v, int order, double* d_out);
// h_delta_l: also download delta_l (host, file order), pipelined with the pass when possible
int back_substitute_device(Ctx& c, const double* d_delta_p, int* nonzero, double* h_delta_l = nullptr);
// landmark transfers (api.cu)
bool is_pinned(const void* p);
int lm_upload(Ctx& c, const double* host_full, int width, double* d_local);
int lm_download(Ctx& c, const double* d_local, int width, double* host_full);
bool xfer_pipelined(const Ctx& c, int width);
int xfer_begin(Ctx& c, int width, bool pinned);
int lm_upload_piece(Ctx& c, const double* host_full, int width, double* d_local, int i, bool pinned);
int lm_download_piece(Ctx& c, const double* d_local, int width, double* host_full, int i, bool pinned);
int lm_download_finish(Ctx& c, double* host_full, int width, bool pinned);
int cost_device(Ctx& c, bool trial, double* cost, int64_t* n_invalid);
int apply_op_device(Ctx& c, int op, const double* d_in, double* d_out);
int materialize_device(Ctx& c, int op, int64_t limit, double* h_out);
int spectral_radius_device(Ctx& c, const double* h_v0, double tol, int max_iter, double* rho, int* iterations,
                           int* converged);
int cameras_prep(Ctx& c, const double* d_cams, double* d_prep);
// collectives over the context's ranks (NCCL communicator or local group);
// no-ops at nranks == 1.  Sums are fp64; allgather concatenates in rank order.
int allreduce_sum(Ctx& c, double* d_buf, size_t n);
int allreduce_max(Ctx& c, double* d_buf, size_t n);
int allgather(Ctx& c, const double* d_src, double* d_dst, size_t n);
// all-to-all of equal slices (slice j of d_dst <- rank j's slice [rank] of d_src)
int exchange_slices(Ctx& c, const double* d_src, double* d_dst, size_t per);
// rank-ordered, run-to-run bitwise deterministic sum (allreduce_sum forwards here)
int allreduce_ordered(Ctx& c, double* d_buf, size_t n);
// sharded: all-gather a per-camera vector whose rank slices were updated locally
int gather_cam_slices(Ctx& c, double* d_vec, int width);
int time_terms_device(Ctx& c, int reps, double* ms_per_term, double* ms_term_kernel, int* launches);
int set_precision_device(Ctx& c, int bits);
int series_clustered_device(Ctx& c, const int64_t* h_cluster_of_cam, int n_clusters, double eps, int max_order,
                            double* h_delta_p, int* order_used, int* converged);
int b_tilde_device(Ctx& c);
int schur_diag_device(Ctx& c, double* d_out45);
int pcg_device(Ctx& c, int precond, int order, double tol, int max_iter, bool resume, double* h_delta_p,
               int* iterations, double* final_rel, int* converged, double* rel_history);
int points_accept_device(Ctx& c);

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// Synchronous copies ON THE CONTEXT STREAM.  (Plain cudaMemcpy runs on the
// legacy default stream, which does not order with the context's non-blocking
// stream: a read-back could overtake the kernel producing the data.)
inline int copy_sync(Ctx& c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return fail(POBA_ECUDA, std::string("copy_sync: ") + cudaGetErrorString(e));
  return POBA_OK;
}

// ---- device helpers shared by the tile kernels -----------------------------------
#ifdef __CUDACC__
// Jacobian column pair p (0..11) of slot o, widened to fp64 (tile block layout)
template <bool F32>
__device__ __forceinline__ int64_t jindex(int64_t o, int p) {  // element index past the tile's metadata
  return (o >> 5) * (tile_block_bytes<F32>() / (F32 ? 8 : 16)) + kMetaBytes / (F32 ? 8 : 16) + p * kTile + (o & 31);
}
template <bool F32>
__device__ __forceinline__ double2 jload(const void* __restrict__ J, int64_t o, int p) {
  if (F32) {
    const float2 v = reinterpret_cast<const float2*>(J)[jindex<true>(o, p)];
    return make_double2((double)v.x, (double)v.y);
  }
  return reinterpret_cast<const double2*>(J)[jindex<false>(o, p)];
}
template <bool F32>
__device__ __forceinline__ void jstore(void* __restrict__ J, int64_t o, int p, double a, double b) {
  if (F32) reinterpret_cast<float2*>(J)[jindex<true>(o, p)] = make_float2((float)a, (float)b);
  else reinterpret_cast<double2*>(J)[jindex<false>(o, p)] = make_double2(a, b);
}
template <bool F32>
__device__ __forceinline__ uint32_t* meta_ptr(void* J, int64_t o) {
  return reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(J) + (o >> 5) * tile_block_bytes<F32>()) + (o & 31);
}
// the value fp32 storage keeps (round to nearest, as numpy's astype(float32))
template <bool F32>
__device__ __forceinline__ double stored(double v) {
  return F32 ? (double)__double2float_rn(v) : v;
}

// landmark starts inside a tile from the per-slot landmark index (lstart has nlm+1 entries)
__device__ __forceinline__ void tile_landmark_starts(const uint8_t* __restrict__ lidx_tile, int n, int nlm,
                                                     int* lstart) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int l = lidx_tile[i];
    if (i == 0 || lidx_tile[i - 1] != l) lstart[l] = i;
  }
  if (threadIdx.x == 0) lstart[nlm] = n;
}
#endif

}  // namespace poba
