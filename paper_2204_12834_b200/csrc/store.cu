// K0 -- observation store structure.
//
// Two orders exist for the observations:
//   * the reference's CANONICAL order, (k of landmark, landmark, camera), which
//     np.lexsort((cam, pt, k[pt])) produces in blocks._sorted_observation_order
//     (/root/reference/pkg/src/powerba/blocks.py:362-372) and which defines
//     the k-groups of blocks._build_groups (blocks.py:405-417).  libpoba
//     reproduces it bit-exactly with a stable device radix sort of the packed
//     key (k, pt, cam) and exports it (order / cam_sorted / pt_sorted / groups);
//   * the STORE order the kernels stream: each rank's landmarks packed into
//     warp-tiles of <= 32 observation slots and <= kTileLm landmarks, in index
//     order with a bounded lookahead (pack_landmarks), each landmark's
//     observations sorted by camera (the reference's within-block order); the
//     device numbers landmarks in this packed order.  Dropping the k-grouping
//     keeps spatially adjacent landmarks (and the cameras that see them)
//     together.  The store order changes only fp64 summation order, never
//     which terms are summed.
// On top of the tiles it builds the term kernel's work plan (one contiguous tile
// range per SM, cut into chunks whose distinct cameras fit the shared-memory
// accumulator table; each observation's chunk slot and landmark run in the
// row metadata), the camera -> partial CSR, and the camera-major permutation
// used by U0/b_p.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "poba_internal.h"

namespace poba {

namespace {

constexpr uint64_t kSentinel = ~0ull;

__global__ void k_convert_idx(const int64_t* __restrict__ cam64, const int64_t* __restrict__ pt64, int64_t n,
                              int64_t n_cam, int64_t n_pt, int* __restrict__ cam32, int* __restrict__ pt32,
                              int* __restrict__ kpt, int* __restrict__ kcam, int* __restrict__ flag) {
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

// canonical key (k, pt, cam) + file index
__global__ void k_canon_keys(const int* __restrict__ cam, const int* __restrict__ pt, const int* __restrict__ kpt,
                             int64_t n, int bc, int bp, uint64_t* __restrict__ key, int* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = pt[i];
  key[i] = ((uint64_t)kpt[p] << (bp + bc)) | ((uint64_t)p << bc) | (uint64_t)cam[i];
  val[i] = (int)i;
}

// store key (pt, cam) + file index
__global__ void k_store_keys(const int* __restrict__ cam, const int* __restrict__ pt, int64_t n, int bc,
                             uint64_t* __restrict__ key, int* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = ((uint64_t)pt[i] << bc) | (uint64_t)cam[i];
  val[i] = (int)i;
}

__global__ void k_lm_keys(const int* __restrict__ kpt, int64_t n_pt, int bp, uint64_t* __restrict__ key) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_pt) return;
  key[p] = ((uint64_t)kpt[p] << bp) | (uint64_t)p;
}

// place the local observations into their slots
__global__ void k_fill_slots(const uint64_t* __restrict__ key, const int* __restrict__ val, int64_t q0,
                             int64_t nq, int bc, int64_t lm_lo, const int* __restrict__ lm_first_l,
                             const int* __restrict__ lm_slot0, const uint8_t* __restrict__ lm_tidx,
                             const double2* __restrict__ pix, int* __restrict__ cam_s, int* __restrict__ file_s,
                             double2* __restrict__ pix_s, uint8_t* __restrict__ lidx_s) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const uint64_t k = key[q0 + q];
  const int f = val[q0 + q];
  const int l = (int)((int64_t)(k >> bc) - lm_lo);
  const int c = (int)(k & ((1ull << bc) - 1));
  const int r = (int)q - lm_first_l[l];
  const int s = lm_slot0[l] + r;
  cam_s[s] = c;
  file_s[s] = f;
  if (pix) pix_s[s] = pix[f];
  lidx_s[s] = lm_tidx[l];
}

// slot arrays after the within-run lane reordering: new slot s <- old slot perm[s]
__global__ void k_permute_slots(const int* __restrict__ perm, int64_t ns, const int* __restrict__ cam_in,
                                const int* __restrict__ file_in, const double2* __restrict__ pix_in,
                                int* __restrict__ cam_out, int* __restrict__ file_out, double2* __restrict__ pix_out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= ns) return;
  const int64_t o = perm[q];
  cam_out[q] = cam_in[o];
  file_out[q] = file_in[o];
  pix_out[q] = pix_in[o];
}

__global__ void k_fill_i32(int* __restrict__ a, int64_t n, int v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

// metadata word of every slot (the first 128 B of each tile block); one warp per tile
template <bool F32>
__global__ void k_pack_meta(const Tile* __restrict__ tiles, const int* __restrict__ slot_s,
                            const uint8_t* __restrict__ lidx_s, void* __restrict__ J) {
  const Tile t = tiles[blockIdx.x];
  const int lane = threadIdx.x;
  const int64_t s = (int64_t)blockIdx.x * kTile + lane;
  const bool valid = lane < t.n;
  const int li = valid ? lidx_s[s] : -1;
  const int prev = __shfl_up_sync(0xffffffffu, li, 1);
  const bool head = valid && (lane == 0 || prev != li);
  const unsigned heads = __ballot_sync(0xffffffffu, head) | (t.n < 32 ? (1u << t.n) : 0u);
  const unsigned above = heads & ~((2u << lane) - 1u);
  const int last = (above ? __ffs(above) - 1 : t.n) - 1;
  const int first = 31 - __clz(heads & ((2u << lane) - 1u));
  // slot_s carries the apply lane in bits 26-31 (every lane, padding included)
  *meta_ptr<F32>(J, s) = valid ? pack_meta(slot_s[s], li, first, last) : ((uint32_t)slot_s[s] & 0xfc000000u);
}

__global__ void k_cam_slot_keys(const Tile* __restrict__ tiles, const int* __restrict__ cam_s,
                                uint64_t* __restrict__ key) {
  const Tile t = tiles[blockIdx.x];
  const int64_t s0 = (int64_t)blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile; i += blockDim.x)
    key[s0 + i] = i < t.n ? (((uint64_t)cam_s[s0 + i] << 32) | (uint64_t)(s0 + i)) : kSentinel;
}

__global__ void k_low32(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)(key[i] & 0xffffffffu);
}

// the U0 / b_p pass walks observations camera-major and recomputes each one's
// J_p and residual: its landmark (store index), pixel and file index, in that order
__global__ void k_cam_major_gather(const int* __restrict__ cperm, int64_t n, const Tile* __restrict__ tiles,
                                   const uint8_t* __restrict__ lidx_s, const double2* __restrict__ pix_s,
                                   const int* __restrict__ file_s, int* __restrict__ lm_c, double2* __restrict__ pix_c,
                                   int* __restrict__ file_c) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int slot = cperm[p];
  const Tile t = tiles[slot >> 5];
  lm_c[p] = t.lm0 + ((t.flags & kTileLong) ? 0 : lidx_s[slot]);
  if (pix_c) pix_c[p] = pix_s[slot];
  file_c[p] = file_s[slot];
}


__global__ void k_cam_degree(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ deg) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&deg[(int)(key[i] >> 32)], 1);
}

// camera of every camera-major reduction chunk (replaces a per-warp binary search)
__global__ void k_cc_cam(const int* __restrict__ cc_cam_off, int64_t n_cam, int* __restrict__ cc_cam) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cam) return;
  for (int k = cc_cam_off[c]; k < cc_cam_off[c + 1]; ++k) cc_cam[k] = (int)c;
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

template <class F>
int cub_call(Ctx& c, F&& f) {
  size_t need = 0;
  PCK(f((void*)nullptr, need));
  PTRY(c.cub_tmp.alloc(need));
  size_t have = c.cub_tmp.bytes;
  PCK(f(c.cub_tmp.p, have));
  return POBA_OK;
}

int sort_keys(Ctx& c, uint64_t* in, uint64_t* out, int64_t n, int end_bit) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(tmp, bytes, in, out, (int)n, 0, end_bit, c.stream);
  });
}

int sort_pairs(Ctx& c, uint64_t* k_in, uint64_t* k_out, int* v_in, int* v_out, int64_t n, int end_bit) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceRadixSort::SortPairs(tmp, bytes, k_in, k_out, v_in, v_out, (int)n, 0, end_bit, c.stream);
  });
}

int excl_sum(Ctx& c, int* in, int* out, int64_t n) {
  return cub_call(c, [&](void* tmp, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, c.stream);
  });
}

}  // namespace

// Host-only: greedy packing of landmarks (index order) into warp-tiles.
void plan_tiles(const int* k_per_point, int64_t n_pt, TilePlan& plan) {
  plan.lm_first.assign(n_pt + 1, 0);
  for (int64_t j = 0; j < n_pt; ++j) plan.lm_first[j + 1] = plan.lm_first[j] + k_per_point[j];
  plan.tiles.clear();
  plan.cut_ok.clear();
  plan.lm_tile.assign(n_pt, 0);
  plan.lm_off_in_tile.assign(n_pt, 0);
  plan.tiles.reserve(plan.lm_first[n_pt] / kTile * 11 / 10 + 16);
  Tile cur{};
  bool open = false;
  auto close = [&]() {
    if (open) {
      plan.tiles.push_back(cur);
      plan.cut_ok.push_back(1);
      open = false;
    }
  };
  for (int64_t j = 0; j < n_pt; ++j) {
    const int k = k_per_point[j];
    if (k > kTile) {
      close();
      plan.lm_tile[j] = (int)plan.tiles.size();
      plan.lm_off_in_tile[j] = 0;
      for (int sub = 0; sub < k; sub += kTile) {
        Tile t{};
        t.obs0 = (int)(plan.lm_first[j] + sub);
        t.n = std::min(kTile, k - sub);
        t.lm0 = (int)j;
        t.nlm = 1;
        t.flags = kTileLong;
        plan.tiles.push_back(t);
        plan.cut_ok.push_back(sub == 0);
      }
      continue;
    }
    if (open && (cur.n + k > kTile || cur.nlm >= kTileLm)) close();
    if (!open) {
      cur = Tile{};
      cur.obs0 = (int)plan.lm_first[j];
      cur.lm0 = (int)j;
      open = true;
    }
    plan.lm_tile[j] = (int)plan.tiles.size();
    plan.lm_off_in_tile[j] = cur.n;
    cur.n += k;
    cur.nlm += 1;
  }
  close();
}

// First tile of rank r's contiguous shard: balanced by observations, cut only
// where a tile starts a new landmark (a long landmark never straddles ranks).
size_t shard_cut(const TilePlan& plan, int64_t n_obs, int r, int nranks) {
  const auto& gt = plan.tiles;
  if (r <= 0) return 0;
  if (r >= nranks) return gt.size();
  const int64_t target = (n_obs * r) / nranks;
  size_t lo = 0, hi = gt.size();
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (gt[mid].obs0 < target) lo = mid + 1; else hi = mid;
  }
  while (lo < gt.size() && !plan.cut_ok[lo]) ++lo;
  return lo;
}

// Host-only: pack one rank's landmarks (file-local 0..n-1) into warp-tiles with a
// bounded lookahead.  Landmarks are taken in index order (spatial locality);
// when the next one does not fit the open tile, the largest landmarks of the
// next `window` that still fit are pulled forward first.  Returns the tiles
// (lm0 in the new STORE numbering) and order[j] = file-local landmark at store
// position j.  Long landmarks (k > kTile) span consecutive full sub-tiles.
void pack_landmarks(const int* k, int64_t n, int window, std::vector<Tile>& tiles, std::vector<int>& order) {
  tiles.clear();
  order.clear();
  order.reserve(n);
  std::vector<char> used(n, 0);
  int64_t obs = 0;
  Tile cur{};
  bool open = false;
  auto place = [&](int64_t l) {
    if (!open) {
      cur = Tile{};
      cur.obs0 = (int)obs;
      cur.lm0 = (int)order.size();
      open = true;
    }
    order.push_back((int)l);
    used[l] = 1;
    cur.n += k[l];
    cur.nlm += 1;
    obs += k[l];
  };
  auto close = [&]() {
    if (open) tiles.push_back(cur);
    open = false;
  };
  auto fill = [&](int64_t from) {  // best fit from the lookahead window
    if (!open) return;
    const int64_t to = std::min<int64_t>(n, from + window);
    while (cur.n < kTile && cur.nlm < kTileLm) {
      int64_t best = -1;
      for (int64_t l = from; l < to; ++l)
        if (!used[l] && k[l] <= kTile - cur.n && (best < 0 || k[l] > k[best])) best = l;
      if (best < 0) break;
      place(best);
    }
  };
  for (int64_t l = 0; l < n; ++l) {
    if (used[l]) continue;
    const int kk = k[l];
    if (kk > kTile) {
      fill(l + 1);
      close();
      const int j = (int)order.size();
      order.push_back((int)l);
      used[l] = 1;
      for (int sub = 0; sub < kk; sub += kTile) {
        Tile t{};
        t.obs0 = (int)(obs + sub);
        t.n = std::min(kTile, kk - sub);
        t.lm0 = j;
        t.nlm = 1;
        t.flags = kTileLong;
        tiles.push_back(t);
      }
      obs += kk;
      continue;
    }
    if (open && (cur.n + kk > kTile || cur.nlm >= kTileLm)) {
      fill(l + 1);
      close();
    }
    place(l);
  }
  close();
}

// Canonical (reference) order and k-groups, built on first export request.
int build_canonical_order(Ctx& c) {
  if (c.have_order) return POBA_OK;
  const int64_t n = c.n_obs, n_pt = c.n_pt;
  const int B = 256;
  cudaStream_t s = c.stream;
  const int bc = std::max(1, bitlen((uint64_t)(c.n_cam - 1)));
  const int bp = std::max(1, bitlen((uint64_t)(n_pt - 1)));
  const int bk = bitlen((uint64_t)c.k_max);
  if (bk + bp + bc > 64) return fail(POBA_EINVAL, "ordering key exceeds 64 bits");
  {
    DBuf ka, kb, va, vb;
    PTRY(ka.alloc(n * 8));
    PTRY(kb.alloc(n * 8));
    PTRY(va.alloc(n * 4));
    PTRY(c.order.alloc(n * 4));
    k_canon_keys<<<grid_for(n, B), B, 0, s>>>(c.cam_file.as<int>(), c.pt_file.as<int>(), c.kpt.as<int>(), n, bc, bp,
                                             ka.as<uint64_t>(), va.as<int>());
    c.launches++;
    PTRY(sort_pairs(c, ka.as<uint64_t>(), kb.as<uint64_t>(), va.as<int>(), c.order.as<int>(), n, bk + bp + bc));
    PCK(cudaStreamSynchronize(s));  // scoped temporaries are freed below
  }
  // k-groups from landmarks sorted by (k, pt)
  std::vector<uint64_t> lk(n_pt);
  {
    DBuf ka, kb;
    PTRY(ka.alloc(n_pt * 8));
    PTRY(kb.alloc(n_pt * 8));
    k_lm_keys<<<grid_for(n_pt, B), B, 0, s>>>(c.kpt.as<int>(), n_pt, bp, ka.as<uint64_t>());
    c.launches++;
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), n_pt, bk + bp));
    PCK(cudaMemcpyAsync(lk.data(), kb.p, n_pt * 8, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
  }
  c.grp_k.clear();
  c.grp_start.clear();
  c.grp_n.clear();
  int64_t off = 0;
  for (int64_t j = 0; j < n_pt;) {
    const int64_t k = (int64_t)(lk[j] >> bp);
    int64_t e = j;
    while (e < n_pt && (int64_t)(lk[e] >> bp) == k) ++e;
    c.grp_k.push_back(k);
    c.grp_start.push_back(off);
    c.grp_n.push_back(e - j);
    off += k * (e - j);
    j = e;
  }
  c.have_order = true;
  return POBA_OK;
}

// (re)allocate the tile-block store for the context's precision and write the metadata
int alloc_store(Ctx& c) {
  const size_t bytes = (size_t)(c.precision == 32 ? kTileBlockF32 : kTileBlock) * (size_t)c.n_tiles;
  c.J.release();
  PTRY(c.J.alloc(bytes));
  PCK(cudaMemsetAsync(c.J.p, 0, bytes, c.stream));
  if (c.precision == 32)
    k_pack_meta<true><<<c.n_tiles, kTile, 0, c.stream>>>(c.tiles.as<Tile>(), c.slot_s.as<int>(),
                                                         c.lidx_s.as<uint8_t>(), c.J.p);
  else
    k_pack_meta<false><<<c.n_tiles, kTile, 0, c.stream>>>(c.tiles.as<Tile>(), c.slot_s.as<int>(),
                                                          c.lidx_s.as<uint8_t>(), c.J.p);
  c.launches++;
  PCK(cudaGetLastError());
  PCK(cudaStreamSynchronize(c.stream));
  return POBA_OK;
}

// switch the block-storage precision (PoBA-32 / PoBA-64); the store must be re-linearized
int set_precision_device(Ctx& c, int bits) {
  if (bits != 32 && bits != 64) return fail(POBA_EINVAL, "precision must be 32 or 64, got " + std::to_string(bits));
  if (bits == c.precision) return POBA_OK;
  c.precision = bits;
  c.drop_graphs();
  c.have_lin = c.have_damp = c.have_solution = c.have_delta_l = false;
  if (c.have_problem) PTRY(alloc_store(c));
  return POBA_OK;
}

namespace {

// Bank-aware renumbering of one chunk's accumulator slots (host).  The term
// kernel's apply does 16-B shared-memory accesses to the 80-B record of each
// distinct camera of a tile (its lowest lane); a 16-B access is served eight
// lanes at a time and slot s's j-th piece lies in bank group (5 s + j) mod 8,
// so lanes of one eight-lane quarter whose slots agree mod 8 serialise.
// Slots are renumbered so that cameras sharing quarters tend to differ mod 8:
// colour = slot mod 8; greedy colouring (most-seen camera first) followed by
// local-search passes that move a camera to the colour it shares the fewest
// quarters with.  Colour classes may exceed n/8 by kSlotSlack (the chunk cut
// leaves room), so the numbering can have holes: colour c's k-th camera gets
// slot 8k + c, the chunk's slot count becomes 8 x (largest class), and a hole's
// partial is written as zeros and never merged (camera -1).  Only the
// numbering changes -- every sum keeps its order, so results are bitwise
// unchanged.  `group` lanes form one colouring group (8: a quarter).
// Returns the chunk's new camera-of-slot list (size = new slot count).
std::vector<int> color_chunk_slots(const std::vector<Tile>& tiles, const Chunk& q, std::vector<int>& obs_slot,
                                   const std::vector<int>& part_cam, int group, int passes) {
  const int n = q.nslot;
  std::vector<int> cam_of(part_cam.begin() + q.part0, part_cam.begin() + q.part0 + n);
  if (n <= 8) return cam_of;
  // quarters of leader lanes (first lane of each camera in its tile)
  std::vector<int> occ_q, occ_s;  // quarter id, old slot of each leader
  std::vector<int> seen(n, -1);
  int nq = 0;
  for (int ti = q.tile0; ti < q.tile1; ++ti) {
    const int64_t s0 = (int64_t)ti * kTile;
    for (int i = 0; i < tiles[ti].n; ++i) {
      const int sl = obs_slot[s0 + i];
      if (seen[sl] == ti) continue;
      seen[sl] = ti;
      occ_q.push_back(nq + i / group);
      occ_s.push_back(sl);
    }
    nq += kTile / group;
  }
  std::vector<int> off(n + 1, 0), qs(occ_q.size());
  for (int sl : occ_s) off[sl + 1]++;
  for (int k = 0; k < n; ++k) off[k + 1] += off[k];
  {
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (size_t k = 0; k < occ_q.size(); ++k) qs[pos[occ_s[k]]++] = occ_q[k];
  }
  std::vector<int> order(n);
  for (int k = 0; k < n; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
  std::vector<uint8_t> qcnt((size_t)nq * 8, 0);
  std::vector<int> color(n, -1), used(8, 0);
  const int cap = (n + 7) / 8 + kSlotSlack;
  auto costs = [&](int sl, int64_t* cost) {
    for (int c = 0; c < 8; ++c) cost[c] = 0;
    for (int k = off[sl]; k < off[sl + 1]; ++k) {
      const uint8_t* qc = &qcnt[(size_t)qs[k] * 8];
      for (int c = 0; c < 8; ++c) cost[c] += qc[c];
    }
  };
  auto place = [&](int sl, int c, int d) {
    for (int k = off[sl]; k < off[sl + 1]; ++k) qcnt[(size_t)qs[k] * 8 + c] += d;
    used[c] += d;
  };
  int64_t cost[8];
  for (int sl : order) {
    costs(sl, cost);
    int best = -1;
    for (int c = 0; c < 8; ++c) {
      if (used[c] >= cap) continue;
      if (best < 0 || cost[c] < cost[best] || (cost[c] == cost[best] && used[c] < used[best])) best = c;
    }
    color[sl] = best;
    place(sl, best, 1);
  }
  for (int pass = 0; pass < passes; ++pass) {
    int moved = 0;
    for (int sl : order) {
      const int cur = color[sl];
      place(sl, cur, -1);
      costs(sl, cost);
      int best = cur;
      for (int c = 0; c < 8; ++c)
        if (c != cur && used[c] < cap && cost[c] < cost[best]) best = c;
      color[sl] = best;
      place(sl, best, 1);
      moved += best != cur;
    }
    if (!moved) break;
  }
  int rows = 0;
  for (int c = 0; c < 8; ++c) rows = std::max(rows, used[c]);
  std::vector<int> slot_new(n), next(8, 0), cams(8 * rows, -1);
  for (int sl = 0; sl < n; ++sl) slot_new[sl] = 8 * next[color[sl]]++ + color[sl];
  for (int sl = 0; sl < n; ++sl) cams[slot_new[sl]] = cam_of[sl];
  while (!cams.empty() && cams.back() < 0) cams.pop_back();  // trailing holes need no partial
  for (int ti = q.tile0; ti < q.tile1; ++ti) {
    const int64_t s0 = (int64_t)ti * kTile;
    for (int i = 0; i < tiles[ti].n; ++i) obs_slot[s0 + i] = slot_new[obs_slot[s0 + i]];
  }
  return cams;
}

// Drop the holes of a chunk's slot numbering (cameras -1) so that a second
// colouring round starts from dense slots and stays within kAccSlots.
std::vector<int> compact_chunk_slots(const std::vector<Tile>& tiles, const Chunk& q, std::vector<int>& obs_slot,
                                     const std::vector<int>& part_cam) {
  std::vector<int> remap(q.nslot, -1), cams;
  for (int sl = 0; sl < q.nslot; ++sl)
    if (part_cam[q.part0 + sl] >= 0) {
      remap[sl] = (int)cams.size();
      cams.push_back(part_cam[q.part0 + sl]);
    }
  for (int ti = q.tile0; ti < q.tile1; ++ti) {
    const int64_t s0 = (int64_t)ti * kTile;
    for (int i = 0; i < tiles[ti].n; ++i) obs_slot[s0 + i] = remap[obs_slot[s0 + i]];
  }
  return cams;
}

// Within-run lane order of one tile.  The accumulator apply of the term kernel
// accesses 16-B pieces of 80-B slot records: the 8 lanes of a quarter-warp are
// served by one shared-memory wavefront only if their slots differ mod 8 (the
// slot colouring's "colour").  Landmark runs must stay contiguous (segmented
// scan), but a run's observations may take any order: each position of a run,
// in lane order, takes the remaining observation whose colour is least used by
// the camera leaders already placed in that position's quarter (a camera
// already placed at a lower lane is pre-summed, not applied: free anywhere).
// Writes perm[new lane] = old lane.
void order_tile_lanes(const Tile& t, const int* slot, const uint8_t* lidx, int* perm) {
  int cnt[4][8] = {};
  int used = 0;  // bitmask of old lanes already placed
  int placed_slots[kTile];
  int n_placed = 0;
  for (int a = 0; a < t.n;) {
    int b = a + 1;
    while (b < t.n && lidx[b] == lidx[a]) ++b;
    for (int pos = a; pos < b; ++pos) {
      const int qd = pos >> 3;
      int best = -1, best_cost = 1 << 30;
      for (int i = a; i < b; ++i) {
        if (used & (1 << i)) continue;
        bool dup = false;
        for (int k = 0; k < n_placed; ++k) dup |= placed_slots[k] == slot[i];
        const int cost = dup ? -1 : cnt[qd][slot[i] & 7];
        if (cost < best_cost) {
          best_cost = cost;
          best = i;
        }
      }
      used |= 1 << best;
      perm[pos] = best;
      if (best_cost >= 0) {
        cnt[qd][slot[best] & 7]++;
        placed_slots[n_placed++] = slot[best];
      }
    }
    a = b;
  }
}

}  // namespace

int build_structure(Ctx& c, const int64_t* h_cam, const int64_t* h_pt, const double* h_pix) {
  const int64_t n = c.n_obs, n_cam = c.n_cam, n_pt = c.n_pt;
  const int B = 256;
  cudaStream_t s = c.stream;
  if (n >= (1ll << 31) - 1 || n_pt >= (1ll << 31) - 1 || n_cam >= (1ll << 24))
    return fail(POBA_EINVAL, "problem too large for 32-bit observation indexing");
  c.have_order = false;
  c.drop_graphs();

  // --- upload + validate indices, histograms ---------------------------------------
  DBuf cam64, pt64, kcam, flag;
  PTRY(cam64.alloc(n * 8));
  PTRY(pt64.alloc(n * 8));
  PCK(cudaMemcpyAsync(cam64.p, h_cam, n * 8, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(pt64.p, h_pt, n * 8, cudaMemcpyHostToDevice, s));
  PTRY(c.cam_file.alloc(n * 4));
  PTRY(c.pt_file.alloc(n * 4));
  PTRY(c.kpt.alloc(n_pt * 4));
  PTRY(kcam.alloc(n_cam * 4));
  PTRY(flag.alloc(16));
  PCK(cudaMemsetAsync(c.kpt.p, 0, n_pt * 4, s));
  PCK(cudaMemsetAsync(kcam.p, 0, n_cam * 4, s));
  int hflag[4] = {0, INT32_MAX, INT32_MIN, 0};
  PCK(cudaMemcpyAsync(flag.p, hflag, 16, cudaMemcpyHostToDevice, s));
  k_convert_idx<<<grid_for(n, B), B, 0, s>>>(cam64.as<int64_t>(), pt64.as<int64_t>(), n, n_cam, n_pt,
                                            c.cam_file.as<int>(), c.pt_file.as<int>(), c.kpt.as<int>(),
                                            kcam.as<int>(), flag.as<int>());
  k_minmax<<<std::min<unsigned>(grid_for(n_pt, B), 1024), B, 0, s>>>(c.kpt.as<int>(), n_pt, flag.as<int>() + 1);
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
  const int bc = std::max(1, bitlen((uint64_t)(n_cam - 1)));
  const int bp = std::max(1, bitlen((uint64_t)(n_pt - 1)));
  if (bp + bc > 64) return fail(POBA_EINVAL, "store key exceeds 64 bits");

  // --- tiles (host greedy packing of landmarks in index order) + this rank's shard -------
  std::vector<int> hk(n_pt);
  PTRY(poba::copy_sync(c, hk.data(), c.kpt.p, n_pt * 4, cudaMemcpyDeviceToHost));
  TilePlan plan;
  plan_tiles(hk.data(), n_pt, plan);
  std::vector<int64_t>& lm_first = plan.lm_first;
  std::vector<Tile>& gt = plan.tiles;
  size_t t_lo = 0, t_hi = gt.size();
  if (c.nranks > 1) {
    t_lo = shard_cut(plan, n, c.rank, c.nranks);
    t_hi = shard_cut(plan, n, c.rank + 1, c.nranks);
  }
  if (t_hi <= t_lo) return fail(POBA_EINVAL, "shard received no landmarks (too many ranks)");
  c.lm_lo = gt[t_lo].lm0;
  c.lm_hi = (t_hi < gt.size()) ? gt[t_hi].lm0 : n_pt;
  c.n_lm_l = c.lm_hi - c.lm_lo;
  const int64_t obs_lo = lm_first[c.lm_lo];
  c.n_obs_l = lm_first[c.lm_hi] - obs_lo;
  // this rank's landmarks re-packed with lookahead; the device works in the
  // resulting STORE landmark order (lm_order: store j -> file landmark lm_lo + lm_order[j])
  std::vector<Tile> tiles;
  pack_landmarks(hk.data() + c.lm_lo, c.n_lm_l, kPackWindow, tiles, c.lm_order_host);
  c.long_host.clear();
  for (auto& t : tiles) {
    if ((t.flags & kTileLong) && (c.long_host.empty() || c.long_host.back() != t.lm0)) c.long_host.push_back(t.lm0);
    if (!(t.flags & kTileLong)) {  // segmented-scan depth for the tile's longest landmark
      int kmax = 1;
      for (int q = 0; q < t.nlm; ++q) kmax = std::max(kmax, hk[c.lm_lo + c.lm_order_host[t.lm0 + q]]);
      int steps = 0;
      while ((1 << steps) < kmax) ++steps;
      t.flags |= steps << kTileScanShift;
    }
  }
  c.n_tiles = (int)tiles.size();
  c.n_long = (int)c.long_host.size();
  c.n_slots = (int64_t)c.n_tiles * kTile;
  const int64_t ns = c.n_slots, nl = c.n_obs_l, nlm = c.n_lm_l;

  // --- per-landmark slot maps ------------------------------------------------------------------
  // file-local (for placing the (pt, cam)-sorted observations) and store-local (kernels)
  std::vector<int> f_slot0(nlm), h_first(nlm + 1), s_slot0(nlm), s_k(nlm);
  std::vector<uint8_t> f_tidx(nlm);
  for (int64_t j = 0; j < nlm; ++j) h_first[j] = (int)(lm_first[c.lm_lo + j] - obs_lo);
  h_first[nlm] = (int)nl;
  for (int ti = 0; ti < c.n_tiles; ++ti) {
    const Tile& t = tiles[ti];
    if ((t.flags & kTileLong) && ti > 0 && (tiles[ti - 1].flags & kTileLong) && tiles[ti - 1].lm0 == t.lm0) continue;
    int off = 0;
    for (int q = 0; q < t.nlm; ++q) {
      const int j = t.lm0 + q;
      const int l = c.lm_order_host[j];
      f_slot0[l] = ti * kTile + off;
      f_tidx[l] = (t.flags & kTileLong) ? 0 : (uint8_t)q;
      s_slot0[j] = f_slot0[l];
      s_k[j] = hk[c.lm_lo + l];
      off += s_k[j];
    }
  }
  PTRY(c.lm_slot0.alloc(std::max<int64_t>(nlm, 1) * 4));
  PTRY(c.lm_k.alloc(std::max<int64_t>(nlm, 1) * 4));
  PTRY(c.lm_perm.alloc(std::max<int64_t>(nlm, 1) * 4));
  PCK(cudaMemcpyAsync(c.lm_slot0.p, s_slot0.data(), nlm * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(c.lm_k.p, s_k.data(), nlm * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaMemcpyAsync(c.lm_perm.p, c.lm_order_host.data(), nlm * 4, cudaMemcpyHostToDevice, s));
  {  // cuts of the pipelined landmark transfers (see Ctx::xf_*)
    const int P = kXferPieces;
    std::vector<int> inv(std::max<int64_t>(nlm, 1), 0);
    for (int64_t j = 0; j < nlm; ++j) inv[c.lm_order_host[j]] = (int)j;
    std::vector<int> up_max(nlm), dn_max(nlm);  // prefix maxima of store->file and file->store
    for (int64_t j = 0; j < nlm; ++j) {
      up_max[j] = std::max(j ? up_max[j - 1] : -1, c.lm_order_host[j]);
      dn_max[j] = std::max(j ? dn_max[j - 1] : -1, inv[j]);
    }
    c.xf_file.assign(P + 1, 0);
    c.xf_up_lm.assign(P + 1, 0);
    c.xf_dn_lm.assign(P + 1, 0);
    c.xf_up_tile.assign(P + 1, 0);
    c.xf_dn_tile.assign(P + 1, 0);
    for (int i = 0; i <= P; ++i) {
      const int64_t f = nlm * i / P;
      c.xf_file[i] = f;
      // store landmarks whose file rows all lie below f: a prefix (up_max is monotone)
      c.xf_up_lm[i] = std::lower_bound(up_max.begin(), up_max.end(), (int)f) - up_max.begin();
      c.xf_dn_lm[i] = f ? (int64_t)dn_max[f - 1] + 1 : 0;
      int tu = 0, td = 0;
      while (tu < c.n_tiles && tiles[tu].lm0 + tiles[tu].nlm <= c.xf_up_lm[i]) ++tu;
      while (td < c.n_tiles && tiles[td].lm0 < c.xf_dn_lm[i]) ++td;
      c.xf_up_tile[i] = tu;
      c.xf_dn_tile[i] = td;
    }
    c.xf_up_tile[P] = c.xf_dn_tile[P] = c.n_tiles;
    PTRY(c.lm_inv.alloc(std::max<int64_t>(nlm, 1) * 4));
    PCK(cudaMemcpyAsync(c.lm_inv.p, inv.data(), nlm * 4, cudaMemcpyHostToDevice, s));
  }
  if (c.n_long) {
    PTRY(c.long_lm.alloc(c.n_long * 4));
    PCK(cudaMemcpyAsync(c.long_lm.p, c.long_host.data(), c.n_long * 4, cudaMemcpyHostToDevice, s));
  }

  // --- store order: stable sort of (pt, cam), then place local observations in slots -------------
  PTRY(c.cam_s.alloc(ns * 4));
  PTRY(c.file_s.alloc(ns * 4));
  PTRY(c.pix_s.alloc(ns * 16));
  PTRY(c.lidx_s.alloc(ns));
  PCK(cudaMemsetAsync(c.cam_s.p, 0, ns * 4, s));
  k_fill_i32<<<grid_for(ns, B), B, 0, s>>>(c.file_s.as<int>(), ns, -1);
  PCK(cudaMemsetAsync(c.pix_s.p, 0, ns * 16, s));
  PCK(cudaMemsetAsync(c.lidx_s.p, 0, ns, s));
  c.launches++;
  {
    DBuf ka, kb, va, vb, pixf, dfirst, dtidx, dslot0;
    PTRY(ka.alloc(n * 8));
    PTRY(kb.alloc(n * 8));
    PTRY(va.alloc(n * 4));
    PTRY(vb.alloc(n * 4));
    k_store_keys<<<grid_for(n, B), B, 0, s>>>(c.cam_file.as<int>(), c.pt_file.as<int>(), n, bc, ka.as<uint64_t>(),
                                             va.as<int>());
    c.launches++;
    PTRY(sort_pairs(c, ka.as<uint64_t>(), kb.as<uint64_t>(), va.as<int>(), vb.as<int>(), n, bp + bc));
    if (h_pix) {
      PTRY(pixf.alloc(n * 16));
      PCK(cudaMemcpyAsync(pixf.p, h_pix, n * 16, cudaMemcpyHostToDevice, s));
    }
    PTRY(dfirst.alloc((nlm + 1) * 4));
    PTRY(dtidx.alloc(std::max<int64_t>(nlm, 1)));
    PCK(cudaMemcpyAsync(dfirst.p, h_first.data(), (nlm + 1) * 4, cudaMemcpyHostToDevice, s));
    PTRY(dslot0.alloc(std::max<int64_t>(nlm, 1) * 4));
    PCK(cudaMemcpyAsync(dtidx.p, f_tidx.data(), nlm, cudaMemcpyHostToDevice, s));
    PCK(cudaMemcpyAsync(dslot0.p, f_slot0.data(), nlm * 4, cudaMemcpyHostToDevice, s));
    k_fill_slots<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), vb.as<int>(), obs_lo, nl, bc, c.lm_lo,
                                              dfirst.as<int>(), dslot0.as<int>(), dtidx.as<uint8_t>(),
                                              h_pix ? pixf.as<double2>() : nullptr, c.cam_s.as<int>(),
                                              c.file_s.as<int>(), c.pix_s.as<double2>(), c.lidx_s.as<uint8_t>());
    c.launches++;
    PCK(cudaStreamSynchronize(s));
  }
  c.have_pixels = h_pix != nullptr;

  // --- term-kernel work: CTA tile ranges, chunks, camera slots (host) ----------------------------
  // Each CTA of the term kernel owns a contiguous tile range (balanced by
  // observations); the range is cut greedily into chunks whose distinct cameras
  // fit the shared-memory accumulator table (kAccSlots records).  Slots are
  // numbered in first-appearance order; partial p = part0 + slot of a chunk
  // holds that camera's sum over the chunk.
  std::vector<int> obs_slot(ns, 0);
  std::vector<uint8_t> obs_meta_hi(ns, 0);  // apply lane of each slot: source lane (bits 0-4), active (bit 5)
  std::vector<Chunk> chunks;
  std::vector<int> part_cam;  // camera of each partial
  {
    std::vector<int> hcam(ns);
    PTRY(poba::copy_sync(c, hcam.data(), c.cam_s.p, ns * 4, cudaMemcpyDeviceToHost));
    // (sized with the gather layout's warp count; only problems smaller than one round per SM differ)
    const int n_cta = std::max(1, std::min(c.n_sm * kTermCtas, (c.n_tiles + kTermWarps - 1) / kTermWarps));
    std::vector<int64_t> cum(c.n_tiles + 1, 0);
    for (int i = 0; i < c.n_tiles; ++i) cum[i + 1] = cum[i] + tiles[i].n;
    std::vector<int2> cta(n_cta);
    int prev = 0;
    for (int b = 0; b < n_cta; ++b) {
      int e = c.n_tiles;
      if (b + 1 < n_cta) {
        const int64_t want = (nl * (b + 1)) / n_cta;
        e = (int)(std::lower_bound(cum.begin(), cum.end(), want) - cum.begin());
        e = std::min(std::max(e, prev + 1), c.n_tiles - (n_cta - 1 - b));
      }
      cta[b] = make_int2(prev, e);
      prev = e;
    }
    std::vector<int> stamp(n_cam, -1), tstamp(n_cam, -1), slot_of(n_cam, 0);
    // Camera-side layout of the term kernel (TermShape).  With the table layout
    // a chunk's term records are loaded into shared memory by all warps of the
    // CTA at a round boundary (a round = kTermWarps consecutive tiles, one per
    // warp), so chunks start only at rounds of the CTA's range, and the table
    // has fewer slots.  It is taken when the camera working set of the CTA
    // ranges still fits: at most kChunkTMaxGrowth times the gather layout's
    // partials (dry run of the chunk cut for both); POBA_TERM_CHUNK_T=0/1 forces.
    auto count_partials = [&](int cap, int align) -> int64_t {
      std::vector<int> st(n_cam, -1), ts(n_cam, -1);
      int64_t total = 0;
      int chn = 0;
      for (int b = 0; b < n_cta; ++b) {
        int cnt = 0;
        bool open = false;
        for (int ti = cta[b].x; ti < cta[b].y; ++ti) {
          const bool may_cut = (ti - cta[b].x) % align == 0;
          if (may_cut || !open) {
            int fresh = 0;
            for (int tj = ti; tj < std::min(ti + align, cta[b].y); ++tj)
              for (int i = 0; i < tiles[tj].n; ++i) {
                const int cam = hcam[(int64_t)tj * kTile + i];
                if (ts[cam] == ti) continue;
                ts[cam] = ti;
                if (!open || st[cam] != chn) ++fresh;
              }
            if (!open || cnt + fresh > cap) {
              if (open) ++chn;
              open = true;
              cnt = 0;
            }
          }
          for (int i = 0; i < tiles[ti].n; ++i) {
            const int cam = hcam[(int64_t)ti * kTile + i];
            if (st[cam] != chn) {
              st[cam] = chn;
              ++cnt;
              ++total;
            }
          }
        }
        if (open) ++chn;
      }
      return total;
    };
    const int cap_gather = TermShape<false>::kAccSlots - 8 * kSlotSlack;
    const int cap_table = TermShape<true>::kAccSlots - 8 * kSlotSlack;
    const char* force = getenv("POBA_TERM_CHUNK_T");
    if (force) {
      c.chunk_t = atoi(force) != 0;
    } else {
      const int64_t pg = count_partials(cap_gather, 1), pt = count_partials(cap_table, TermShape<true>::kWarps);
      c.chunk_t = (double)pt <= kChunkTMaxGrowth * (double)pg;
    }
    const int align = c.chunk_t ? TermShape<true>::kWarps : 1;
    const int cap_slots = c.chunk_t ? cap_table : cap_gather;
    std::vector<int> rstamp(n_cam, -1);
    for (int b = 0; b < n_cta; ++b) {
      int ch = -1, cnt = 0;
      for (int ti = cta[b].x; ti < cta[b].y; ++ti) {
        Tile& t = tiles[ti];
        const int64_t s0 = (int64_t)ti * kTile;
        int fresh = 0;
        bool dup = false;
        for (int i = 0; i < t.n; ++i) {
          const int cam = hcam[s0 + i];
          if (tstamp[cam] == ti) {
            dup = true;
            continue;
          }
          tstamp[cam] = ti;
          if (ch < 0 || stamp[cam] != ch) ++fresh;
        }
        const bool may_cut = (ti - cta[b].x) % align == 0;
        if (align > 1 && may_cut) {  // new cameras of the whole round
          fresh = 0;
          for (int tj = ti; tj < std::min(ti + align, cta[b].y); ++tj)
            for (int i = 0; i < tiles[tj].n; ++i) {
              const int cam = hcam[(int64_t)tj * kTile + i];
              if (rstamp[cam] == ti) continue;
              rstamp[cam] = ti;
              if (ch < 0 || stamp[cam] != ch) ++fresh;
            }
        }
        if (ch < 0 || (may_cut && cnt + fresh > cap_slots)) {
          if (ch >= 0) chunks.back().tile1 = ti;
          chunks.push_back(Chunk{ti, ti, (int)part_cam.size(), 0});
          ch = (int)chunks.size() - 1;
          cnt = 0;
        }
        for (int i = 0; i < t.n; ++i) {
          const int cam = hcam[s0 + i];
          if (stamp[cam] != ch) {
            stamp[cam] = ch;
            slot_of[cam] = cnt++;
            part_cam.push_back(cam);
          }
          obs_slot[s0 + i] = slot_of[cam];
        }
        chunks.back().nslot = cnt;
        t.chunk = ch;
        if (dup) t.flags |= kTileDupCam;
      }
      chunks.back().tile1 = cta[b].y;
    }
    for (const Chunk& q : chunks) tiles[q.tile1 - 1].flags |= kTileChunkLast;
    if (!getenv("POBA_NO_SLOT_COLOR")) {
      // lanes per colouring group: with the apply-lane permutation (below) a
      // tile's cameras can be dealt to any quarter, so what matters is that no
      // colour has more than four cameras in a TILE (group 32) and the order
      // of lanes inside a run no longer matters (no lane-ordering rounds);
      // without it the colouring works per quarter (group 8) as in round 1
      const bool perm_on = !getenv("POBA_NO_APPLY_PERM");
      const char* g = getenv("POBA_SLOT_GROUP");  // A/B override: 8, 16 or 32
      const int group = (g && (atoi(g) == 8 || atoi(g) == 16 || atoi(g) == 32)) ? atoi(g) : (perm_on ? 32 : 8);
      const char* ps = getenv("POBA_SLOT_PASSES");  // A/B: local-search passes after the greedy colouring
      const int passes = ps ? std::max(0, atoi(ps)) : kSlotPasses;
      std::vector<int> pc;  // rebuilt camera of every partial (-1: hole)
      pc.reserve(part_cam.size() + chunks.size() * 8 * kSlotSlack);
      for (Chunk& q : chunks) {
        std::vector<int> cams = color_chunk_slots(tiles, q, obs_slot, part_cam, group, passes);
        q.part0 = (int)pc.size();
        q.nslot = (int)cams.size();
        pc.insert(pc.end(), cams.begin(), cams.end());
      }
      part_cam.swap(pc);
      // rounds of within-run lane ordering (host permutation of the tile's
      // slots, applied to the device slot arrays) and re-colouring
      const char* lr = getenv("POBA_LANE_ROUNDS");  // A/B: 0 disables
      const int rounds = lr ? std::max(0, atoi(lr)) : (perm_on ? 0 : kLaneRounds);
      if (rounds > 0) {
        std::vector<uint8_t> hl(ns);
        PTRY(poba::copy_sync(c, hl.data(), c.lidx_s.p, ns, cudaMemcpyDeviceToHost));
        std::vector<int> perm(ns), tmp_slot(ns), tmp_cam(ns);
        std::vector<int> total(ns);
        for (int64_t q = 0; q < ns; ++q) total[q] = (int)q;  // composed new -> original slot
        for (int round = 0; round < rounds; ++round) {
          for (int64_t q = 0; q < ns; ++q) perm[q] = (int)q;
          for (int ti = 0; ti < c.n_tiles; ++ti) {
            if (tiles[ti].flags & kTileLong) continue;
            const int64_t s0 = (int64_t)ti * kTile;
            int lp[kTile];
            order_tile_lanes(tiles[ti], &obs_slot[s0], &hl[s0], lp);
            for (int i = 0; i < tiles[ti].n; ++i) perm[s0 + i] = (int)(s0 + lp[i]);
          }
          for (int64_t q = 0; q < ns; ++q) {
            tmp_slot[q] = obs_slot[perm[q]];
            tmp_cam[q] = hcam[perm[q]];
          }
          obs_slot.swap(tmp_slot);
          hcam.swap(tmp_cam);
          for (int64_t q = 0; q < ns; ++q) tmp_slot[q] = total[perm[q]];
          total.swap(tmp_slot);
          std::vector<int> pc2;
          pc2.reserve(part_cam.size());
          for (Chunk& q : chunks) {
            std::vector<int> dense = compact_chunk_slots(tiles, q, obs_slot, part_cam);
            // colour the dense numbering: color_chunk_slots reads the chunk's
            // cameras from part_cam[part0, part0 + nslot)
            Chunk qd = q;
            qd.part0 = 0;
            qd.nslot = (int)dense.size();
            std::vector<int> cams = color_chunk_slots(tiles, qd, obs_slot, dense, group, passes);
            q.part0 = (int)pc2.size();
            q.nslot = (int)cams.size();
            pc2.insert(pc2.end(), cams.begin(), cams.end());
          }
          part_cam.swap(pc2);
        }
        DBuf dperm, c2, f2, p2;
        PTRY(dperm.alloc(ns * 4));
        PTRY(c2.alloc(ns * 4));
        PTRY(f2.alloc(ns * 4));
        PTRY(p2.alloc(ns * 16));
        PCK(cudaMemcpyAsync(dperm.p, total.data(), ns * 4, cudaMemcpyHostToDevice, s));
        k_permute_slots<<<grid_for(ns, B), B, 0, s>>>(dperm.as<int>(), ns, c.cam_s.as<int>(), c.file_s.as<int>(),
                                                     c.pix_s.as<double2>(), c2.as<int>(), f2.as<int>(),
                                                     p2.as<double2>());
        c.launches++;
        PCK(cudaGetLastError());
        PCK(cudaMemcpyAsync(c.cam_s.p, c2.p, ns * 4, cudaMemcpyDeviceToDevice, s));
        PCK(cudaMemcpyAsync(c.file_s.p, f2.p, ns * 4, cudaMemcpyDeviceToDevice, s));
        PCK(cudaMemcpyAsync(c.pix_s.p, p2.p, ns * 16, cudaMemcpyDeviceToDevice, s));
        PCK(cudaStreamSynchronize(s));
      }
    }
    // Apply lanes.  The term kernel adds each distinct camera of a tile (held by
    // its lowest lane after the duplicate pre-sum) to its accumulator record
    // with 16-B accesses, served one eight-lane quarter at a time; lanes of a
    // quarter whose slots agree mod 8 serialise.  Which lane performs a
    // camera's access is free, so each tile carries a lane permutation: lane d
    // pulls the contribution of lane src(d) with warp shuffles and applies it
    // (bits 26-30 of its metadata word: src, bit 31: active).  The cameras of
    // a colour class are spread over the four quarters, so a quarter holds two
    // slots of one colour only if the tile has more than four of that colour.
    if (!getenv("POBA_NO_APPLY_PERM")) {
      std::vector<int> seen(n_cam, -1);
      for (int ti = 0; ti < c.n_tiles; ++ti) {
        const int64_t s0 = (int64_t)ti * kTile;
        int by_col[8][kTile], n_col[8] = {};
        for (int i = 0; i < tiles[ti].n; ++i) {
          const int cam = hcam[s0 + i];
          if (seen[cam] == ti) continue;  // not the camera's lowest lane
          seen[cam] = ti;
          const int col = obs_slot[s0 + i] & 7;
          by_col[col][n_col[col]++] = i;
        }
        int order[8] = {0, 1, 2, 3, 4, 5, 6, 7};
        std::sort(order, order + 8, [&](int a, int b) { return n_col[a] != n_col[b] ? n_col[a] > n_col[b] : a < b; });
        // a quarter costs its largest colour multiplicity: place each camera where
        // that grows least (colours in decreasing size, so the doubles of a colour
        // with more than four cameras land in quarters that already have a double)
        int load[4] = {}, has[4][8] = {}, qmax[4] = {};
        int src_of[kTile];
        for (int d = 0; d < kTile; ++d) src_of[d] = -1;
        for (int oc = 0; oc < 8; ++oc) {
          const int col = order[oc];
          for (int k = 0; k < n_col[col]; ++k) {
            int best = -1, best_grow = 0;
            for (int qq = 0; qq < 4; ++qq) {
              if (load[qq] >= 8) continue;
              const int grow = std::max(qmax[qq], has[qq][col] + 1) - qmax[qq];
              if (best < 0 || grow < best_grow || (grow == best_grow && has[qq][col] < has[best][col]) ||
                  (grow == best_grow && has[qq][col] == has[best][col] && load[qq] < load[best])) {
                best = qq;
                best_grow = grow;
              }
            }
            src_of[best * 8 + load[best]] = by_col[col][k];
            load[best]++;
            has[best][col]++;
            qmax[best] = std::max(qmax[best], has[best][col]);
          }
        }
        for (int d = 0; d < kTile; ++d)
          obs_meta_hi[s0 + d] = src_of[d] >= 0 ? (uint8_t)(src_of[d] | 32) : (uint8_t)d;
      }
    } else {
      std::vector<int> seen(n_cam, -1);
      for (int ti = 0; ti < c.n_tiles; ++ti) {
        const int64_t s0 = (int64_t)ti * kTile;
        for (int d = 0; d < kTile; ++d) obs_meta_hi[s0 + d] = (uint8_t)d;
        for (int i = 0; i < tiles[ti].n; ++i) {
          const int cam = hcam[s0 + i];
          if (seen[cam] == ti) continue;
          seen[cam] = ti;
          obs_meta_hi[s0 + i] = (uint8_t)(i | 32);
        }
      }
    }
    if (getenv("POBA_SLOT_STATS")) {  // bank-conflict model: sum over quarters of the largest residue class
      int64_t wf = 0, ideal = 0;
      for (int ti = 0; ti < c.n_tiles; ++ti) {
        const int64_t s0 = (int64_t)ti * kTile;
        int cnt[4][8] = {};
        for (int d = 0; d < kTile; ++d) {
          if (!(obs_meta_hi[s0 + d] & 32)) continue;
          cnt[d / 8][obs_slot[s0 + (obs_meta_hi[s0 + d] & 31)] & 7]++;
        }
        for (int qq = 0; qq < 4; ++qq) {
          int mx = 0, tot = 0;
          for (int r = 0; r < 8; ++r) {
            mx = std::max(mx, cnt[qq][r]);
            tot += cnt[qq][r];
          }
          wf += mx;
          ideal += tot ? 1 : 0;
        }
      }
      fprintf(stderr, "poba slot stats: %d chunks, %zu partials, %.3f wavefronts per apply access per tile (ideal %.3f)\n",
              (int)chunks.size(), part_cam.size(), (double)wf / c.n_tiles, (double)ideal / c.n_tiles);
    }
    c.n_cta = n_cta;
    PTRY(c.cta_tiles.alloc(n_cta * sizeof(int2)));
    PTRY(poba::copy_sync(c, c.cta_tiles.p, cta.data(), n_cta * sizeof(int2), cudaMemcpyHostToDevice));
  }
  c.n_chunks = (int)chunks.size();
  c.n_partials = (int)part_cam.size();
  c.max_slots = 0;
  for (auto& q : chunks) c.max_slots = std::max(c.max_slots, q.nslot);
  c.chunks_host = chunks;
  PTRY(c.chunks.alloc(chunks.size() * sizeof(Chunk)));
  PTRY(poba::copy_sync(c, c.chunks.p, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  PTRY(c.tiles.alloc(tiles.size() * sizeof(Tile)));
  PTRY(poba::copy_sync(c, c.tiles.p, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  {  // compact kernel descriptors
    std::vector<TileK> tk(c.n_tiles);
    std::vector<int> cta_end(c.n_tiles, 0);  // end of the CTA range holding each tile
    {
      std::vector<int2> cta(c.n_cta);
      PTRY(poba::copy_sync(c, cta.data(), c.cta_tiles.p, c.n_cta * sizeof(int2), cudaMemcpyDeviceToHost));
      for (const int2& r : cta)
        for (int i = r.x; i < r.y; ++i) cta_end[i] = r.y;
    }
    for (int i = 0; i < c.n_tiles; ++i) {
      const Chunk& ch = chunks[tiles[i].chunk];
      const int nx = i + (c.chunk_t ? TermShape<true>::kWarps : TermShape<false>::kWarps);  // same warp's next tile
      const bool has = nx < cta_end[i];
      tk[i] = TileK{tiles[i].n, tiles[i].lm0, tiles[i].nlm, tiles[i].flags, ch.part0, ch.nslot,
                    has ? (tiles[nx].n | (tiles[nx].nlm << 8)) : 0, has ? tiles[nx].lm0 : 0};
    }
    PTRY(c.tilek.alloc(c.n_tiles * sizeof(TileK)));
    PTRY(poba::copy_sync(c, c.tilek.p, tk.data(), c.n_tiles * sizeof(TileK), cudaMemcpyHostToDevice));
  }
  {  // camera -> partials, chunk order
    const int n_u = c.n_partials;
    std::vector<int> off(n_cam + 1, 0), idx(std::max(n_u, 1));
    for (int p = 0; p < n_u; ++p)
      if (part_cam[p] >= 0) off[part_cam[p] + 1]++;  // holes of the slot numbering are never merged
    for (int64_t q = 0; q < n_cam; ++q) off[q + 1] += off[q];
    std::vector<int> pos(off.begin(), off.end() - 1);
    for (int p = 0; p < n_u; ++p)
      if (part_cam[p] >= 0) idx[pos[part_cam[p]]++] = p;
    PTRY(c.part_idx.alloc(std::max(n_u, 1) * 4));
    PTRY(poba::copy_sync(c, c.part_idx.p, idx.data(), std::max(n_u, 1) * 4, cudaMemcpyHostToDevice));
    PTRY(c.part_cam_off.alloc((n_cam + 1) * 4));
    PTRY(poba::copy_sync(c, c.part_cam_off.p, off.data(), (n_cam + 1) * 4, cudaMemcpyHostToDevice));
    PTRY(c.part_cam.alloc(std::max(n_u, 1) * 4));
    if (n_u) PTRY(poba::copy_sync(c, c.part_cam.p, part_cam.data(), (size_t)n_u * 4, cudaMemcpyHostToDevice));
  }
  DBuf ka, kb;
  PTRY(ka.alloc(ns * 8));
  PTRY(kb.alloc(ns * 8));

  // camera-major permutation of slots for the U0 / b_p reduction
  {
    k_cam_slot_keys<<<c.n_tiles, kTile, 0, s>>>(c.tiles.as<Tile>(), c.cam_s.as<int>(), ka.as<uint64_t>());
    PTRY(sort_keys(c, ka.as<uint64_t>(), kb.as<uint64_t>(), ns, 64));
    PTRY(c.cperm.alloc(nl * 4));
    k_low32<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), nl, c.cperm.as<int>());
    PTRY(c.lm_c.alloc(std::max<int64_t>(nl, 1) * 4));
    PTRY(c.file_c.alloc(std::max<int64_t>(nl, 1) * 4));
    if (h_pix) PTRY(c.pix_c.alloc(std::max<int64_t>(nl, 1) * 16));
    k_cam_major_gather<<<grid_for(nl, B), B, 0, s>>>(c.cperm.as<int>(), nl, c.tiles.as<Tile>(),
                                                    c.lidx_s.as<uint8_t>(), c.pix_s.as<double2>(),
                                                    c.file_s.as<int>(), c.lm_c.as<int>(),
                                                    h_pix ? c.pix_c.as<double2>() : nullptr, c.file_c.as<int>());
    c.launches++;
    DBuf deg, ccnt;
    PTRY(deg.alloc((n_cam + 1) * 4));
    PTRY(ccnt.alloc((n_cam + 1) * 4));
    PCK(cudaMemsetAsync(deg.p, 0, (n_cam + 1) * 4, s));
    k_cam_degree<<<grid_for(nl, B), B, 0, s>>>(kb.as<uint64_t>(), nl, deg.as<int>());
    k_cc_counts<<<grid_for(n_cam, B), B, 0, s>>>(deg.as<int>(), n_cam, ccnt.as<int>());
    PCK(cudaMemsetAsync(ccnt.as<int>() + n_cam, 0, 4, s));
    c.launches += 4;
    PTRY(c.cam_start.alloc((n_cam + 1) * 4));
    PTRY(excl_sum(c, deg.as<int>(), c.cam_start.as<int>(), n_cam + 1));
    PTRY(c.cc_cam_off.alloc((n_cam + 1) * 4));
    PTRY(excl_sum(c, ccnt.as<int>(), c.cc_cam_off.as<int>(), n_cam + 1));
    int ncc = 0;
    PCK(cudaMemcpyAsync(&ncc, c.cc_cam_off.as<int>() + n_cam, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    c.n_cchunks = ncc;
    PTRY(c.cc_cam.alloc((size_t)std::max(ncc, 1) * 4));
    k_cc_cam<<<grid_for(n_cam, B), B, 0, s>>>(c.cc_cam_off.as<int>(), n_cam, c.cc_cam.as<int>());
    c.launches++;
    PCK(cudaGetLastError());
  }

  // --- store rows (J + metadata) and work buffers ------------------------------------------------------------
  PTRY(c.Rz.alloc((size_t)ns * 16));
  PCK(cudaMemsetAsync(c.Rz.p, 0, (size_t)ns * 16, s));
  PTRY(c.slot_s.alloc(ns * 4));
  for (int64_t q = 0; q < ns; ++q) obs_slot[q] |= (int)((uint32_t)obs_meta_hi[q] << 26);  // metadata bits 26-31
  PCK(cudaMemcpyAsync(c.slot_s.p, obs_slot.data(), ns * 4, cudaMemcpyHostToDevice, s));
  PCK(cudaStreamSynchronize(s));  // obs_slot is a local vector
  PTRY(alloc_store(c));
  const int64_t nc = n_cam, nlm1 = std::max<int64_t>(nlm, 1);
  // sharded: the camera step finalizes rank slices of cam_ls cameras (>= 4, the
  // slice's first four t records carry its norm totals); per-camera vectors
  // that are all-gathered by slices are padded to nranks * cam_ls rows
  c.cam_ls = c.nranks > 1 ? std::max<int64_t>(4, (nc + c.nranks - 1) / c.nranks) : nc;
  const int64_t ncp = c.nranks > 1 ? c.cam_ls * c.nranks : nc;
  for (DBuf* b : {&c.cams, &c.cams_trial, &c.bp, &c.Dp, &c.rvec}) PTRY(b->alloc(nc * 9 * 8));
  for (DBuf* b : {&c.bt, &c.xvec}) PTRY(b->alloc(ncp * 9 * 8));
  for (DBuf* b : {&c.tvec, &c.ctmp, &c.ctmp2}) PTRY(b->alloc(ncp * kTStride * 8));
  for (DBuf* b : {&c.cams_prep, &c.trial_prep}) PTRY(b->alloc(nc * 16 * 8));
  for (DBuf* b : {&c.U0, &c.Uinv, &c.Ud}) PTRY(b->alloc(nc * 45 * 8));
  for (DBuf* b : {&c.points, &c.bl, &c.Dl, &c.dl, &c.ltmp}) PTRY(b->alloc(nlm1 * 3 * 8));
  for (DBuf* b : {&c.V0, &c.Vinv, &c.Vd}) PTRY(b->alloc(nlm1 * 6 * 8));
  PTRY(c.cc_part.alloc(std::max(c.n_cchunks, 1) * 54 * 8));
  PTRY(c.partials.alloc(std::max(c.n_partials, 1) * kTStride * 8));
  PTRY(c.state.alloc(sizeof(SeriesState)));
  PTRY(c.blk_part.alloc((grid_for(n_cam, 8) + 8) * 4 * 8));
  PTRY(c.flag.alloc(64));
  PTRY(c.red.alloc(64 * 8));
  PCK(cudaMemsetAsync(c.state.p, 0, sizeof(SeriesState), s));
  PCK(cudaStreamSynchronize(s));
  c.have_problem = true;
  c.have_lin = c.have_damp = c.have_solution = c.have_delta_l = c.have_points = false;
  return POBA_OK;
}

}  // namespace poba
