// K0 -- observation store structure.
//
// Replaces the reference's canonical ordering and grouping
// (/root/reference/pkg/src/powerba/blocks.py:362-372 _sorted_observation_order,
//  blocks.py:405-417 _build_groups, blocks.py:83-87 per-landmark offsets):
//   * canonical order = stable radix sort of the packed key (k[pt], pt, cam),
//     identical to np.lexsort((cam, pt, k[pt])) -- ties (duplicate pairs, only
//     possible through assemble_from_observations) keep file order, as lexsort;
//   * landmark-aligned tiles of <= 256 observations (one k per tile, so a tile
//     is a slice of one k-group view (n, k, 2, 13));
//   * chunks = contiguous tile ranges, one per persistent CTA of the series
//     kernel, with a chunk-local camera "slot" map: the series kernel reduces
//     per-observation camera contributions into shared-memory slot
//     accumulators in a fixed order (deterministic, no fp64 atomics);
//   * the camera-major permutation used by the U0/b_p reduction;
//   * (sharded) this rank's contiguous landmark range.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>

#include "poba_internal.h"

namespace poba {

namespace {

__global__ void k_convert_idx(const int64_t* __restrict__ cam64, const int64_t* __restrict__ pt64,
                              int64_t n, int64_t n_cam, int64_t n_pt, int* __restrict__ cam32,
                              int* __restrict__ pt32, int* __restrict__ kpt, int* __restrict__ kcam,
                              int* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c = cam64[i], p = pt64[i];
  if (c < 0 || c >= n_cam || p < 0 || p >= n_pt) {
    atomicOr(flag, 1);
    return;
  }
  cam32[i] = (int)c;
  pt32[i] = (int)p;
  atomicAdd(&kpt[p], 1);
  atomicAdd(&kcam[c], 1);
}

__global__ void k_minmax(const int* __restrict__ a, int64_t n, int* __restrict__ out /*min,max*/) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int v_min = INT32_MAX, v_max = INT32_MIN;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int v = a[i];
    v_min = min(v_min, v);
    v_max = max(v_max, v);
  }
  for (int o = 16; o; o >>= 1) {
    v_min = min(v_min, __shfl_xor_sync(0xffffffffu, v_min, o));
    v_max = max(v_max, __shfl_xor_sync(0xffffffffu, v_max, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out[0], v_min);
    atomicMax(&out[1], v_max);
  }
}

__global__ void k_obs_keys(const int* __restrict__ cam, const int* __restrict__ pt,
                           const int* __restrict__ kpt, int64_t n, int bc, int bp,
                           uint64_t* __restrict__ key, int* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = pt[i];
  key[i] = ((uint64_t)kpt[p] << (bp + bc)) | ((uint64_t)p << bc) | (uint64_t)cam[i];
  val[i] = (int)i;
}

__global__ void k_lm_keys(const int* __restrict__ kpt, int64_t n_pt, int bp, uint64_t* __restrict__ key) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_pt) return;
  key[p] = ((uint64_t)kpt[p] << bp) | (uint64_t)p;
}

__global__ void k_lm_split(const uint64_t* __restrict__ key, int64_t n_pt, int bp,
                           int* __restrict__ lm_pt, int* __restrict__ lm_k) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_pt) return;
  uint64_t k = key[j];
  lm_pt[j] = (int)(k & ((1ull << bp) - 1));
  lm_k[j] = (int)(k >> bp);
}

// local observation arrays for the shard [obs_lo, obs_lo + n)
__global__ void k_local_obs(const int* __restrict__ order, const int* __restrict__ cam_file,
                            const double2* __restrict__ pix_file, int64_t obs_lo, int64_t n,
                            int* __restrict__ cam_l, int* __restrict__ file_l, double2* __restrict__ pix_l) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f = order[obs_lo + i];
  file_l[i] = f;
  cam_l[i] = cam_file[f];
  if (pix_file) pix_l[i] = pix_file[f];
}

__global__ void k_pt_to_lm(const int* __restrict__ lm_pt, int64_t n_lm, int* __restrict__ pt_to_lm) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n_lm) pt_to_lm[lm_pt[j]] = (int)j;
}

// key (chunk, cam) per local observation, via the tile table
__global__ void k_chunk_cam_keys(const Tile* __restrict__ tiles, const int* __restrict__ cam_l, int bc,
                                 uint64_t* __restrict__ key) {
  const Tile t = tiles[blockIdx.x];
  for (int i = threadIdx.x; i < t.n; i += blockDim.x)
    key[t.obs0 + i] = ((uint64_t)t.chunk << bc) | (uint64_t)cam_l[t.obs0 + i];
}

__global__ void k_unique_flags(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// compact unique keys; pos = exclusive scan of flags
__global__ void k_unique_compact(const uint64_t* __restrict__ key, const int* __restrict__ flag,
                                 const int* __restrict__ pos, int64_t n, uint64_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[pos[i]] = key[i];
}

// first unique entry of each chunk
__global__ void k_chunk_first(const uint64_t* __restrict__ ukey, int n_u, int bc, int* __restrict__ first) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  int ch = (int)(ukey[i] >> bc);
  if (i == 0 || (int)(ukey[i - 1] >> bc) != ch) first[ch] = i;
}

// (cam, chunk) keys of the unique pairs, value = partial index
__global__ void k_part_keys(const uint64_t* __restrict__ ukey, int n_u, int bc, int bch,
                            uint64_t* __restrict__ key, int* __restrict__ val, int* __restrict__ cam_cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_u) return;
  uint64_t u = ukey[i];
  int cam = (int)(u & ((1ull << bc) - 1));
  int ch = (int)(u >> bc);
  key[i] = ((uint64_t)cam << bch) | (uint64_t)ch;
  val[i] = i;
  atomicAdd(&cam_cnt[cam], 1);
}

// key (tile, cam, tile-local position) per local observation
__global__ void k_tile_cam_keys(const Tile* __restrict__ tiles, const int* __restrict__ cam_l, int bc,
                                uint64_t* __restrict__ key) {
  const int ti = blockIdx.x;
  const Tile t = tiles[ti];
  for (int i = threadIdx.x; i < t.n; i += blockDim.x)
    key[t.obs0 + i] = ((uint64_t)ti << (bc + 8)) | ((uint64_t)cam_l[t.obs0 + i] << 8) | (uint64_t)i;
}

__global__ void k_seg_flags(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ flag) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  flag[q] = (q == 0 || (key[q] >> 8) != (key[q - 1] >> 8)) ? 1 : 0;
}

__device__ __forceinline__ int lower_bound_cam(const uint64_t* __restrict__ ukey, int lo, int hi,
                                               uint64_t target) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (ukey[mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_segments(const uint64_t* __restrict__ key, const int* __restrict__ flag,
                           const int* __restrict__ segpos, Tile* __restrict__ tiles,
                           const Chunk* __restrict__ chunks, const uint64_t* __restrict__ ukey, int bc,
                           uint8_t* __restrict__ perm, uint16_t* __restrict__ seg_start,
                           uint16_t* __restrict__ seg_slot) {
  const int ti = blockIdx.x;
  Tile t = tiles[ti];
  const Chunk ch = chunks[t.chunk];
  for (int r = threadIdx.x; r < t.n; r += blockDim.x) {
    int64_t q = t.obs0 + r;
    uint64_t k = key[q];
    perm[q] = (uint8_t)(k & 0xff);
    if (flag[q]) {
      int cam = (int)((k >> 8) & ((1ull << bc) - 1));
      uint64_t target = ((uint64_t)t.chunk << bc) | (uint64_t)cam;
      int u = lower_bound_cam(ukey, ch.part0, ch.part0 + ch.nslot, target);
      int s = segpos[q];
      seg_start[s] = (uint16_t)r;
      seg_slot[s] = (uint16_t)(u - ch.part0);
    }
  }
  if (threadIdx.x == 0) {
    int s0 = segpos[t.obs0];
    int s1 = segpos[t.obs0 + t.n - 1] + flag[t.obs0 + t.n - 1];
    tiles[ti].seg0 = s0;
    tiles[ti].nseg = s1 - s0;
  }
}

__global__ void k_cam_obs_keys(const int* __restrict__ cam_l, int64_t n, uint64_t* __restrict__ key) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) key[i] = ((uint64_t)cam_l[i] << 32) | (uint64_t)i;
}

__global__ void k_low32(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)(key[i] & 0xffffffffu);
}

__global__ void k_cam_degree(const int* __restrict__ cam_l, int64_t n, int* __restrict__ deg) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&deg[cam_l[i]], 1);
}

__global__ void k_cc_counts(const int* __restrict__ deg, int64_t n_cam, int* __restrict__ cnt) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n_cam) cnt[c] = (deg[c] + kCamChunk - 1) / kCamChunk;
}

int bitlen(uint64_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// CUB helpers with a growing temp buffer
template <class F>
int cub_call(Ctx& c, F&& f) {
  size_t need = 0;
  PCK(f((void*)nullptr, need));
  PTRY(c.cub_tmp.alloc(need));
  size_t have = c.cub_tmp.bytes;
  PCK(f(c.cub_tmp.p, have));
  return POBA_OK;
}

int sort_keys(Ctx& c, uint64_t* keys_in, uint64_t* keys_out, int64_t n, int end_bit) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(tmp, bytes, keys_in, keys_out, (int)n, 0, end_bit, c.stream);
  });
}

int sort_pairs(Ctx& c, uint64_t* k_in, uint64_t* k_out, int* v_in, int* v_out, int64_t n, int end_bit) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceRadixSort::SortPairs(tmp, bytes, k_in, k_out, v_in, v_out, (int)n, 0, end_bit,
                                           c.stream);
  });
}

int excl_sum(Ctx& c, int* in, int* out, int64_t n) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, c.stream);
  });
}

}  // namespace

int build_structure(Ctx& c, const int64_t* h_cam, const int64_t* h_pt, const double* h_pix) {
  const int64_t n = c.n_obs, n_cam = c.n_cam, n_pt = c.n_pt;
  const int B = 256;
  cudaStream_t s = c.stream;
  if (n >= (1ll << 31) - 1 || n_pt >= (1ll << 31) - 1 || n_cam >= (1ll << 24))
    return fail(POBA_EINVAL, "problem too large for 32-bit observation indexing");

  // --- upload + validate indices, histograms --------------------------------------
  DBuf cam64, pt64, kpt, kcam, flag;
  PTRY(cam64.alloc(n * 8));
  PTRY(pt64.alloc(n * 8));
  PCK(cudaMemcpyAsync(cam64.p, h_cam, n * 8, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(pt64.p, h_pt, n * 8, cudaMemcpyHostToDevice, s));
  PTRY(c.cam_file.alloc(n * 4));
  PTRY(c.pt_file.alloc(n * 4));
  PTRY(kpt.alloc(n_pt * 4));
  PTRY(kcam.alloc(n_cam * 4));
  PTRY(flag.alloc(16));
  PCK(cudaMemsetAsync(kpt.p, 0, n_pt * 4, s));
  PCK(cudaMemsetAsync(kcam.p, 0, n_cam * 4, s));
  int hflag[4] = {0, INT32_MAX, INT32_MIN, 0};
  PCK(cudaMemcpyAsync(flag.p, hflag, 16, cudaMemcpyHostToDevice, s));
  k_convert_idx<<<grid_for(n, B), B, 0, s>>>(cam64.as<int64_t>(), pt64.as<int64_t>(), n, n_cam, n_pt,
                                            c.cam_file.as<int>(), c.pt_file.as<int>(), kpt.as<int>(),
                                            kcam.as<int>(), flag.as<int>());
  k_minmax<<<std::min<unsigned>(grid_for(n_pt, B), 1024), B, 0, s>>>(kpt.as<int>(), n_pt, flag.as<int>() + 1);
  c.launches += 2;
  PCK(cudaMemcpyAsync(hflag, flag.p, 16, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  cam64.release();
  pt64.release();
  if (hflag[0]) return fail(POBA_EINVAL, "camera or point index out of range");
  if (hflag[1] == 0) return fail(POBA_EINVAL, "every point must be observed at least once");
  c.k_max = hflag[2];
  {
    int mm[2] = {INT32_MAX, INT32_MIN};
    PCK(cudaMemcpyAsync(flag.p, mm, 8, cudaMemcpyHostToDevice, s));
    k_minmax<<<std::min<unsigned>(grid_for(n_cam, B), 1024), B, 0, s>>>(kcam.as<int>(), n_cam, flag.as<int>());
    c.launches++;
    PCK(cudaMemcpyAsync(mm, flag.p, 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    if (mm[0] == 0) return fail(POBA_EINVAL, "every camera must have at least one observation");
  }

  // --- canonical order: stable sort of (k, pt, cam) --------------------------------
  const int bc = std::max(1, bitlen((uint64_t)(n_cam - 1)));
  const int bp = std::max(1, bitlen((uint64_t)(n_pt - 1)));
  const int bk = bitlen((uint64_t)c.k_max);
  if (bk + bp + bc > 64) return fail(POBA_EINVAL, "ordering key exceeds 64 bits");
  {
    DBuf ka, kb, va, vb;
    PTRY(ka.alloc(n * 8));
    PTRY(kb.alloc(n * 8));
    PTRY(va.alloc(n * 4));
    PTRY(vb.alloc(n * 4));
    k_obs_keys<<<grid_for(n, B), B, 0, s>>>(c.cam_file.as<int>(), c.pt_file.as<int>(), kpt.as<int>(), n,
                                           bc, bp, ka.as<uint64_t>(), va.as<int>());
    c.launches++;
    PTRY(sort_pairs(c, ka.as<uint64_t>(), kb.as<uint64_t>(), va.as<int>(), vb.as<int>(), n, bk + bp + bc));
    PTRY(c.order.alloc(n * 4));
    PCK(cudaMemcpyAsync(c.order.p, vb.p, n * 4, cudaMemcpyDeviceToDevice, s));
  }

  // --- canonical landmark order: sort points by (k, pt) -----------------------------
  std::vector<int> h_lm_pt(n_pt), h_lm_k(n_pt);
  DBuf g_lm_pt, g_lm_k;
  PTRY(g_lm_pt.alloc(n_pt * 4));
  PTRY(g_lm_k.alloc(n_pt * 4));
  {
    DBuf ka, kb;
    PTRY(ka.alloc(n_pt * 8));
    PTRY(kb.alloc(n_pt * 8));
    k_lm_keys<<<grid_for(n_pt, B), B, 0, s>>>(kpt.as<int>(), n_pt, bp, ka.as<uint64_t>());
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), n_pt, bk + bp));
    k_lm_split<<<grid_for(n_pt, B), B, 0, s>>>(kb.as<uint64_t>(), n_pt, bp, g_lm_pt.as<int>(), g_lm_k.as<int>());
    c.launches += 2;
    PCK(cudaMemcpyAsync(h_lm_pt.data(), g_lm_pt.p, n_pt * 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaMemcpyAsync(h_lm_k.data(), g_lm_k.p, n_pt * 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
  }
  std::vector<int64_t> h_lm_off(n_pt + 1);
  h_lm_off[0] = 0;
  for (int64_t j = 0; j < n_pt; ++j) h_lm_off[j + 1] = h_lm_off[j] + h_lm_k[j];

  // --- k-groups (blocks.py:405-417) ---------------------------------------------------
  c.grp_k.clear();
  c.grp_start.clear();
  c.grp_n.clear();
  std::vector<int64_t> grp_lm0;
  for (int64_t j = 0; j < n_pt;) {
    int64_t e = j;
    while (e < n_pt && h_lm_k[e] == h_lm_k[j]) ++e;
    c.grp_k.push_back(h_lm_k[j]);
    c.grp_start.push_back(h_lm_off[j]);
    c.grp_n.push_back(e - j);
    grp_lm0.push_back(j);
    j = e;
  }

  // --- tiles (global) -----------------------------------------------------------------
  std::vector<Tile> gt;
  std::vector<char> cut_ok;  // may a shard boundary sit before this tile?
  gt.reserve(n / kTile + c.grp_k.size() + 16);
  for (size_t g = 0; g < c.grp_k.size(); ++g) {
    const int k = (int)c.grp_k[g];
    const int64_t lm0 = grp_lm0[g], ng = c.grp_n[g];
    if (k <= kTile) {
      const int per = kTile / k;
      for (int64_t a = 0; a < ng; a += per) {
        Tile t{};
        t.lm0 = (int)(lm0 + a);
        t.nlm = (int)std::min<int64_t>(per, ng - a);
        t.k = k;
        t.obs0 = (int)h_lm_off[lm0 + a];
        t.n = t.nlm * k;
        gt.push_back(t);
        cut_ok.push_back(1);
      }
    } else {
      for (int64_t a = 0; a < ng; ++a) {
        for (int sub = 0; sub < k; sub += kTile) {
          Tile t{};
          t.lm0 = (int)(lm0 + a);
          t.nlm = 1;
          t.k = k;
          t.obs0 = (int)(h_lm_off[lm0 + a] + sub);
          t.n = std::min(kTile, k - sub);
          gt.push_back(t);
          cut_ok.push_back(sub == 0);
        }
      }
    }
  }

  // --- shard: contiguous tile range balanced by observations ---------------------------
  size_t t_lo = 0, t_hi = gt.size();
  if (c.nranks > 1) {
    auto cut_at = [&](int r) -> size_t {
      if (r <= 0) return 0;
      if (r >= c.nranks) return gt.size();
      const int64_t target = (n * r) / c.nranks;
      size_t lo = 0, hi = gt.size();
      while (lo < hi) {  // first tile with obs0 >= target
        size_t mid = (lo + hi) / 2;
        if (gt[mid].obs0 < target) lo = mid + 1; else hi = mid;
      }
      while (lo < gt.size() && !cut_ok[lo]) ++lo;
      return lo;
    };
    t_lo = cut_at(c.rank);
    t_hi = cut_at(c.rank + 1);
  }
  if (t_hi <= t_lo) return fail(POBA_EINVAL, "shard received no landmarks (too many ranks)");
  c.obs_lo = gt[t_lo].obs0;
  c.obs_hi = (t_hi < gt.size()) ? gt[t_hi].obs0 : n;
  c.lm_lo = gt[t_lo].lm0;
  c.lm_hi = (t_hi < gt.size()) ? gt[t_hi].lm0 : n_pt;
  c.n_obs_l = c.obs_hi - c.obs_lo;
  c.n_lm_l = c.lm_hi - c.lm_lo;
  c.obs_pad = (c.n_obs_l + 63) / 64 * 64;
  std::vector<Tile> tiles(gt.begin() + t_lo, gt.begin() + t_hi);
  std::vector<int> long_host;
  for (auto& t : tiles) {
    t.obs0 -= (int)c.obs_lo;
    t.lm0 -= (int)c.lm_lo;
    if (t.k > kTile && (long_host.empty() || long_host.back() != t.lm0)) long_host.push_back(t.lm0);
  }
  c.n_tiles = (int)tiles.size();
  c.long_host = long_host;
  c.n_long = (int)long_host.size();

  // --- local observation / landmark arrays ------------------------------------------------
  const int64_t nl = c.n_obs_l;
  PTRY(c.cam_l.alloc(nl * 4));
  PTRY(c.file_l.alloc(nl * 4));
  PTRY(c.pix_l.alloc(nl * 16));
  {
    DBuf pix_file;
    if (h_pix) {
      PTRY(pix_file.alloc(n * 16));
      PCK(cudaMemcpyAsync(pix_file.p, h_pix, n * 16, cudaMemcpyHostToDevice, s));
    }
    k_local_obs<<<grid_for(nl, B), B, 0, s>>>(c.order.as<int>(), c.cam_file.as<int>(),
                                             h_pix ? pix_file.as<double2>() : nullptr, c.obs_lo, nl,
                                             c.cam_l.as<int>(), c.file_l.as<int>(), c.pix_l.as<double2>());
    c.launches++;
    PCK(cudaStreamSynchronize(s));
  }
  c.have_pixels = h_pix != nullptr;
  PTRY(c.lm_pt.alloc(c.n_lm_l * 4));
  PTRY(c.lm_off.alloc((c.n_lm_l + 1) * 4));
  PCK(cudaMemcpyAsync(c.lm_pt.p, h_lm_pt.data() + c.lm_lo, c.n_lm_l * 4, cudaMemcpyHostToDevice, s));
  {
    std::vector<int> off(c.n_lm_l + 1);
    for (int64_t j = 0; j <= c.n_lm_l; ++j) off[j] = (int)(h_lm_off[c.lm_lo + j] - c.obs_lo);
    PCK(cudaMemcpyAsync(c.lm_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, s));
    PCK(cudaStreamSynchronize(s));
  }
  PTRY(c.pt_to_lm.alloc(n_pt * 4));
  PCK(cudaMemsetAsync(c.pt_to_lm.p, 0xff, n_pt * 4, s));
  k_pt_to_lm<<<grid_for(c.n_lm_l, B), B, 0, s>>>(c.lm_pt.as<int>(), c.n_lm_l, c.pt_to_lm.as<int>());
  c.launches++;
  if (c.n_long) {
    PTRY(c.long_lm.alloc(c.n_long * 4));
    PTRY(c.long_zb.alloc(c.n_long * 3 * 8));
    PCK(cudaMemcpyAsync(c.long_lm.p, long_host.data(), c.n_long * 4, cudaMemcpyHostToDevice, s));
  }

  // --- chunks + camera slots ------------------------------------------------------------------
  // one chunk per resident CTA of the series kernel (2 per SM); a chunk whose
  // distinct cameras exceed kSlotCap is split until it fits.
  std::vector<Chunk> chunks;
  {
    const int target = std::max(1, std::min(c.n_tiles, 2 * c.n_sm));
    std::vector<int64_t> cum(c.n_tiles + 1, 0);
    for (int i = 0; i < c.n_tiles; ++i) cum[i + 1] = cum[i] + tiles[i].n;
    int prev = 0;
    for (int q = 1; q <= target; ++q) {
      int64_t want = (nl * q) / target;
      int e = (int)(std::lower_bound(cum.begin(), cum.end(), want) - cum.begin());
      e = std::min(std::max(e, prev + 1), c.n_tiles);
      if (q == target) e = c.n_tiles;
      if (e > prev) chunks.push_back(Chunk{prev, e, 0, 0});
      prev = e;
      if (prev >= c.n_tiles) break;
    }
  }
  const int bch_tiles = std::max(1, bitlen((uint64_t)c.n_tiles));
  DBuf d_tiles_buf;
  DBuf ka, kb, ukey, fl, pos;
  PTRY(ka.alloc(nl * 8));
  PTRY(kb.alloc(nl * 8));
  PTRY(ukey.alloc(nl * 8));
  PTRY(fl.alloc((nl + 1) * 4));
  PTRY(pos.alloc((nl + 1) * 4));
  int n_u = 0;
  std::vector<int> first;
  for (int iter = 0;; ++iter) {
    for (size_t q = 0; q < chunks.size(); ++q)
      for (int t = chunks[q].tile0; t < chunks[q].tile1; ++t) tiles[t].chunk = (int)q;
    PTRY(c.tiles.alloc(tiles.size() * sizeof(Tile)));
    PCK(cudaMemcpyAsync(c.tiles.p, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice, s));
    const int bchunk = std::max(1, bitlen((uint64_t)chunks.size()));
    if (bchunk + bc > 64) return fail(POBA_EINVAL, "chunk key exceeds 64 bits");
    k_chunk_cam_keys<<<c.n_tiles, B, 0, s>>>(c.tiles.as<Tile>(), c.cam_l.as<int>(), bc, ka.as<uint64_t>());
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), nl, bchunk + bc));
    k_unique_flags<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), nl, fl.as<int>());
    PCK(cudaMemsetAsync(fl.as<int>() + nl, 0, 4, s));
    PTRY(excl_sum(c, fl.as<int>(), pos.as<int>(), nl + 1));
    k_unique_compact<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), fl.as<int>(), pos.as<int>(), nl,
                                                  ukey.as<uint64_t>());
    c.launches += 3;
    PCK(cudaMemcpyAsync(&n_u, pos.as<int>() + nl, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    DBuf dfirst;
    PTRY(dfirst.alloc(chunks.size() * 4));
    k_chunk_first<<<grid_for(n_u, B), B, 0, s>>>(ukey.as<uint64_t>(), n_u, bc, dfirst.as<int>());
    c.launches++;
    first.assign(chunks.size() + 1, 0);
    PCK(cudaMemcpyAsync(first.data(), dfirst.p, chunks.size() * 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    first[chunks.size()] = n_u;
    bool split = false;
    std::vector<Chunk> next;
    for (size_t q = 0; q < chunks.size(); ++q) {
      chunks[q].part0 = first[q];
      chunks[q].nslot = first[q + 1] - first[q];
      if (chunks[q].nslot > kSlotCap && chunks[q].tile1 - chunks[q].tile0 > 1) {
        int mid = (chunks[q].tile0 + chunks[q].tile1) / 2;
        next.push_back(Chunk{chunks[q].tile0, mid, 0, 0});
        next.push_back(Chunk{mid, chunks[q].tile1, 0, 0});
        split = true;
      } else {
        next.push_back(chunks[q]);
      }
    }
    if (!split) break;
    chunks.swap(next);
    if (iter > 40) return fail(POBA_EINVAL, "cannot split chunks under the camera-slot cap");
  }
  c.n_chunks = (int)chunks.size();
  c.n_partials = n_u;
  c.max_slots = 0;
  for (auto& q : chunks) c.max_slots = std::max(c.max_slots, q.nslot);
  if (c.max_slots > kSlotCap) return fail(POBA_EINVAL, "a single tile touches more cameras than the slot cap");
  PTRY(c.chunks.alloc(chunks.size() * sizeof(Chunk)));
  PCK(cudaMemcpyAsync(c.chunks.p, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice, s));

  // camera -> partials (chunk order)
  {
    DBuf k1, k2, v1, v2, cnt;
    PTRY(k1.alloc(n_u * 8));
    PTRY(k2.alloc(n_u * 8));
    PTRY(v1.alloc(n_u * 4));
    PTRY(v2.alloc(n_u * 4));
    PTRY(cnt.alloc((n_cam + 1) * 4));
    PCK(cudaMemsetAsync(cnt.p, 0, (n_cam + 1) * 4, s));
    const int bchunk = std::max(1, bitlen((uint64_t)chunks.size()));
    k_part_keys<<<grid_for(n_u, B), B, 0, s>>>(ukey.as<uint64_t>(), n_u, bc, bchunk, k1.as<uint64_t>(),
                                              v1.as<int>(), cnt.as<int>());
    c.launches++;
    PTRY(sort_pairs(c, k1.as<uint64_t>(), k2.as<uint64_t>(), v1.as<int>(), v2.as<int>(), n_u, bc + bchunk));
    PTRY(c.part_idx.alloc(n_u * 4));
    PCK(cudaMemcpyAsync(c.part_idx.p, v2.p, n_u * 4, cudaMemcpyDeviceToDevice, s));
    PTRY(c.part_cam_off.alloc((n_cam + 1) * 4));
    PTRY(excl_sum(c, cnt.as<int>(), c.part_cam_off.as<int>(), n_cam + 1));
  }

  // per-tile camera segments + tile-local permutation
  {
    if (bch_tiles + bc + 8 > 64) return fail(POBA_EINVAL, "tile key exceeds 64 bits");
    k_tile_cam_keys<<<c.n_tiles, B, 0, s>>>(c.tiles.as<Tile>(), c.cam_l.as<int>(), bc, ka.as<uint64_t>());
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), nl, bch_tiles + bc + 8));
    k_seg_flags<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), nl, fl.as<int>());
    PCK(cudaMemsetAsync(fl.as<int>() + nl, 0, 4, s));
    PTRY(excl_sum(c, fl.as<int>(), pos.as<int>(), nl + 1));
    c.launches += 2;
    int nseg = 0;
    PCK(cudaMemcpyAsync(&nseg, pos.as<int>() + nl, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    c.n_segs = nseg;
    PTRY(c.perm.alloc(nl));
    PTRY(c.seg_start.alloc(std::max(nseg, 1) * 2));
    PTRY(c.seg_slot.alloc(std::max(nseg, 1) * 2));
    k_segments<<<c.n_tiles, B, 0, s>>>(kb.as<uint64_t>(), fl.as<int>(), pos.as<int>(), c.tiles.as<Tile>(),
                                       c.chunks.as<Chunk>(), ukey.as<uint64_t>(), bc, c.perm.as<uint8_t>(),
                                       c.seg_start.as<uint16_t>(), c.seg_slot.as<uint16_t>());
    c.launches++;
  }

  // camera-major permutation and chunks for the U0 / b_p reduction
  {
    k_cam_obs_keys<<<grid_for(nl, B), B, 0, s>>>(c.cam_l.as<int>(), nl, ka.as<uint64_t>());
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), nl, 32 + bc));
    PTRY(c.cperm.alloc(nl * 4));
    k_low32<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), nl, c.cperm.as<int>());
    DBuf deg, ccnt;
    PTRY(deg.alloc((n_cam + 1) * 4));
    PTRY(ccnt.alloc((n_cam + 1) * 4));
    PCK(cudaMemsetAsync(deg.p, 0, (n_cam + 1) * 4, s));
    k_cam_degree<<<grid_for(nl, B), B, 0, s>>>(c.cam_l.as<int>(), nl, deg.as<int>());
    k_cc_counts<<<grid_for(n_cam, B), B, 0, s>>>(deg.as<int>(), n_cam, ccnt.as<int>());
    PCK(cudaMemsetAsync(ccnt.as<int>() + n_cam, 0, 4, s));
    c.launches += 4;
    PTRY(c.cc_start.alloc((n_cam + 1) * 4));  // camera -> first observation in cperm
    PTRY(excl_sum(c, deg.as<int>(), c.cc_start.as<int>(), n_cam + 1));
    PTRY(c.cc_cam_off.alloc((n_cam + 1) * 4));
    PTRY(excl_sum(c, ccnt.as<int>(), c.cc_cam_off.as<int>(), n_cam + 1));
    int ncc = 0;
    PCK(cudaMemcpyAsync(&ncc, c.cc_cam_off.as<int>() + n_cam, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    c.n_cchunks = ncc;
  }

  // --- per-context work buffers ---------------------------------------------------------------
  PTRY(c.J.alloc((size_t)kJPlanes * c.obs_pad * 16));
  PTRY(c.Rz.alloc((size_t)c.obs_pad * 16));
  PCK(cudaMemsetAsync(c.J.p, 0, (size_t)kJPlanes * c.obs_pad * 16, s));
  PCK(cudaMemsetAsync(c.Rz.p, 0, (size_t)c.obs_pad * 16, s));
  const int64_t nc = n_cam, nlm = c.n_lm_l;
  for (DBuf* b : {&c.cams, &c.cams_trial, &c.bp, &c.Dp, &c.bt, &c.tvec, &c.xvec, &c.rvec, &c.ctmp, &c.ctmp2})
    PTRY(b->alloc(nc * 9 * 8));
  for (DBuf* b : {&c.cams_prep, &c.trial_prep}) PTRY(b->alloc(nc * 16 * 8));
  for (DBuf* b : {&c.U0, &c.Uinv, &c.Ud}) PTRY(b->alloc(nc * 45 * 8));
  for (DBuf* b : {&c.points, &c.bl, &c.Dl, &c.dl, &c.ltmp}) PTRY(b->alloc(std::max<int64_t>(nlm, 1) * 3 * 8));
  for (DBuf* b : {&c.V0, &c.Vinv, &c.Vd}) PTRY(b->alloc(std::max<int64_t>(nlm, 1) * 6 * 8));
  PTRY(c.cc_part.alloc(std::max(c.n_cchunks, 1) * 54 * 8));
  PTRY(c.partials.alloc(std::max(c.n_partials, 1) * 9 * 8));
  PTRY(c.state.alloc(sizeof(SeriesState)));
  PTRY(c.blk_part.alloc(4096 * 4 * 8));
  PTRY(c.flag.alloc(64));
  PTRY(c.red.alloc(64 * 8));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  PCK(cudaStreamSynchronize(s));
  c.have_problem = true;
  c.have_lin = c.have_damp = c.have_solution = c.have_delta_l = c.have_points = false;
  return POBA_OK;
}

}  // namespace poba
