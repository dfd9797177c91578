// C-ABI entry points of libpoba (see include/poba.h for the contract and the
// reference function each entry point replaces).
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>

#include "poba_internal.h"

struct poba_ctx {
  poba::Ctx c;
};

namespace poba {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

const NcclApi* nccl_api() {
  static NcclApi api;
  static int state = 0;  // 0 untried, 1 ok, -1 failed
  static std::string why;
  if (state == 1) return &api;
  if (state == -1) {
    set_error(why);
    return nullptr;
  }
  void* h = nullptr;
  const char* env = getenv("POBA_NCCL_LIB");
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. PyTorch's)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    state = -1;
    why = std::string("cannot load libnccl.so.2: ") + dlerror();
    set_error(why);
    return nullptr;
  }
  bool ok = true;
  auto sym = [&](const char* name) -> void* {
    void* p = dlsym(h, name);
    if (!p) ok = false;
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  if (!ok) {
    state = -1;
    why = "libnccl.so.2 lacks a required symbol";
    set_error(why);
    return nullptr;
  }
  state = 1;
  return &api;
}

// ---- in-process virtual ranks ------------------------------------------------
// A LocalGroup lets nranks contexts on ONE device (one host thread each) run
// the sharded path with the same collectives the NCCL communicator provides.
// Ranks meet at a host barrier after their stream has drained, so no kernel
// ever waits on another rank's kernel; every rank then reduces all ranks'
// buffers (same device) in rank order into its own scratch, and a second
// barrier keeps the sources alive until everyone has read them.
struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  const double* src[kMaxLocalRanks] = {};
  // false on timeout (a rank failed or never arrived): the group is poisoned
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

namespace {

struct RankPtrs {
  const double* p[kMaxLocalRanks];
};

// out[i] = op over ranks r = 0..n-1 of p[r][i], in rank order
template <bool kMax>
__global__ void k_rank_reduce(RankPtrs src, int n, size_t len, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
    double v = src.p[0][i];
    for (int r = 1; r < n; ++r) v = kMax ? fmax(v, src.p[r][i]) : v + src.p[r][i];
    out[i] = v;
  }
}

int group_fail() { return fail(POBA_ENCCL, "local rank group: a rank failed or timed out at a collective"); }

// kind 0 sum, 1 max, 2 gather (dst gets n values per rank, rank order),
// 3 exchange (dst slice j <- rank j's src slice [rank], n values per slice)
int local_collective(Ctx& c, int kind, const double* d_src, double* d_dst, size_t n) {
  LocalGroup& g = *c.group;
  PCK(cudaStreamSynchronize(c.stream));
  {
    std::lock_guard<std::mutex> lk(g.m);
    g.src[c.rank] = d_src;
  }
  if (!g.barrier()) return group_fail();
  RankPtrs rp;
  for (int r = 0; r < g.n; ++r) rp.p[r] = g.src[r];
  if (kind == 2) {
    for (int r = 0; r < g.n; ++r)
      if (d_dst + r * n != rp.p[r])  // in place: this rank's own slice is already there
        PCK(cudaMemcpyAsync(d_dst + r * n, rp.p[r], n * 8, cudaMemcpyDeviceToDevice, c.stream));
  } else if (kind == 3) {
    for (int r = 0; r < g.n; ++r)
      PCK(cudaMemcpyAsync(d_dst + r * n, rp.p[r] + (size_t)c.rank * n, n * 8, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    PTRY(c.coll_tmp.alloc(n * 8));
    const unsigned nb = (unsigned)std::min<size_t>((n + 255) / 256, 1184);
    if (kind == 1) k_rank_reduce<true><<<nb, 256, 0, c.stream>>>(rp, g.n, n, c.coll_tmp.as<double>());
    else k_rank_reduce<false><<<nb, 256, 0, c.stream>>>(rp, g.n, n, c.coll_tmp.as<double>());
    PCK(cudaGetLastError());
  }
  PCK(cudaStreamSynchronize(c.stream));
  if (!g.barrier()) return group_fail();
  if (kind < 2) PCK(cudaMemcpyAsync(d_dst, c.coll_tmp.p, n * 8, cudaMemcpyDeviceToDevice, c.stream));
  return POBA_OK;
}

// dst[j] (slice of `per` values) += ... : the rank-order sum of the R received slices
__global__ void k_slice_sum(const double* recv, int nranks, size_t per, double* out) {  // out may alias slice 0
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
    double v = recv[i];
    for (int r = 1; r < nranks; ++r) v += recv[(size_t)r * per + i];
    out[i] = v;
  }
}

}  // namespace

// all-to-all of equal slices: d_dst slice j <- rank j's d_src slice [rank]
int exchange_slices(Ctx& c, const double* d_src, double* d_dst, size_t per) {
  if (c.nranks <= 1) return copy_sync(c, d_dst, d_src, per * 8, cudaMemcpyDeviceToDevice);
  if (c.group) return local_collective(c, 3, d_src, d_dst, per);
  PNCCL(GroupStart());
  for (int r = 0; r < c.nranks; ++r) {
    if (r == c.rank) continue;
    PNCCL(Send(d_src + (size_t)r * per, per, ncclFloat64, r, c.comm, c.stream));
    PNCCL(Recv(d_dst + (size_t)r * per, per, ncclFloat64, r, c.comm, c.stream));
  }
  PNCCL(GroupEnd());
  PCK(cudaMemcpyAsync(d_dst + (size_t)c.rank * per, d_src + (size_t)c.rank * per, per * 8, cudaMemcpyDeviceToDevice,
                      c.stream));
  return POBA_OK;
}

// Deterministic all-reduce (sum): every element is summed over ranks in rank
// order r = 0, 1, ..., R-1 by the rank owning its slice, then all-gathered.
// The result is bitwise the same on every rank, from run to run, and for any
// NCCL algorithm / protocol / channel choice (the collectives only move data),
// and bitwise equal to the virtual-rank group's reduction.  Same NVLink bytes
// as a ring all-reduce (a reduce-scatter's worth out, an all-gather's worth in).
int allreduce_ordered(Ctx& c, double* d_buf, size_t n) {
  if (c.nranks <= 1) return POBA_OK;
  const size_t R = (size_t)c.nranks;
  const size_t per = (n + R - 1) / R;
  PTRY(c.xch_send.alloc(R * per * 8));
  PTRY(c.xch_recv.alloc(R * per * 8));
  double* snd = c.xch_send.as<double>();
  double* rcv = c.xch_recv.as<double>();
  if (R * per > n) PCK(cudaMemsetAsync(snd + n, 0, (R * per - n) * 8, c.stream));
  PCK(cudaMemcpyAsync(snd, d_buf, n * 8, cudaMemcpyDeviceToDevice, c.stream));
  PTRY(exchange_slices(c, snd, rcv, per));
  const unsigned nb = (unsigned)std::min<size_t>((per + 255) / 256, 1184);
  k_slice_sum<<<std::max(1u, nb), 256, 0, c.stream>>>(rcv, c.nranks, per, rcv);  // slice 0 of rcv: my sums
  c.launches++;
  PCK(cudaGetLastError());
  PTRY(allgather(c, rcv, snd, per));
  PCK(cudaMemcpyAsync(d_buf, snd, n * 8, cudaMemcpyDeviceToDevice, c.stream));
  return POBA_OK;
}

int allreduce_sum(Ctx& c, double* d_buf, size_t n) { return allreduce_ordered(c, d_buf, n); }

int allreduce_max(Ctx& c, double* d_buf, size_t n) {
  if (c.nranks <= 1) return POBA_OK;
  if (c.group) return local_collective(c, 1, d_buf, d_buf, n);
  PNCCL(AllReduce(d_buf, d_buf, n, ncclFloat64, ncclMax, c.comm, c.stream));
  return POBA_OK;
}

// sharded contexts: every rank updated only its slice of a per-camera vector
// (x, b_tilde) -- all-gather the slices (rows of `width` doubles), in place
int gather_cam_slices(Ctx& c, double* d_vec, int width) {
  if (c.nranks <= 1) return POBA_OK;
  const size_t per = (size_t)c.cam_ls * width;
  return allgather(c, d_vec + (size_t)c.rank * per, d_vec, per);
}

int allgather(Ctx& c, const double* d_src, double* d_dst, size_t n) {
  if (c.nranks <= 1) return copy_sync(c, d_dst, d_src, n * 8, cudaMemcpyDeviceToDevice);
  if (c.group) return local_collective(c, 2, d_src, d_dst, n);
  PNCCL(AllGather(d_src, d_dst, n, ncclFloat64, c.comm, c.stream));
  return POBA_OK;
}

namespace {

void unpack9(const double* p45, double* out81) {
  for (int i = 0; i < 9; ++i)
    for (int j = i; j < 9; ++j) {
      const double v = p45[i * 9 - i * (i - 1) / 2 + (j - i)];
      out81[i * 9 + j] = v;
      out81[j * 9 + i] = v;
    }
}

void unpack3(const double* p6, double* out9) {
  const int idx[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
  for (int q = 0; q < 9; ++q) out9[q] = p6[idx[q]];
}

}  // namespace

// landmark arrays: this rank owns file landmarks [lm_lo, lm_hi); host arrays are
// full (n_pt rows, file order); the device keeps them in store order
// (store j <-> file lm_lo + lm_perm[j]), permuted on the device.
// dst row j <- src row idx[j], j in [j0, j1)
__global__ void k_lm_gather(const double* __restrict__ src, const int* __restrict__ idx, int64_t j0, int64_t j1,
                            int width, double* __restrict__ dst) {
  const int64_t q = j0 * width + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= j1 * width) return;
  const int64_t j = q / width;
  dst[q] = src[(int64_t)idx[j] * width + (q - j * width)];
}
__global__ void k_lm_scatter(const double* __restrict__ src, const int* __restrict__ perm, int64_t n, int width,
                             double* __restrict__ dst) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n * width) return;
  const int64_t j = q / width;
  dst[(int64_t)perm[j] * width + (q - j * width)] = src[q];
}

// Large host<->device copies of pageable memory go through a pinned staging
// buffer owned by the context and a few host threads (CUDA's own pageable path
// runs at a few GB/s); pinned user memory is copied directly.
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = 1u << 20;
  const int nt = (int)std::min<size_t>(8, (bytes + kChunk - 1) / kChunk);
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const size_t o = (size_t)t * per;
    if (o >= bytes) break;
    th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(per, bytes - o)); });
  }
  for (auto& x : th) x.join();
}

int pinned_stage(Ctx& c, size_t bytes) {
  if (c.host_stage_bytes >= bytes) return POBA_OK;
  if (c.host_stage) cudaFreeHost(c.host_stage);
  c.host_stage = nullptr;
  c.host_stage_bytes = 0;
  PCK(cudaHostAlloc(&c.host_stage, bytes, cudaHostAllocDefault));
  c.host_stage_bytes = bytes;
  return POBA_OK;
}

int host_to_device(Ctx& c, void* d_dst, const void* h_src, size_t bytes) {  // synchronous
  if (bytes < (4u << 20) || is_pinned(h_src)) {
    PCK(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, c.stream));
    return POBA_OK;
  }
  PCK(cudaStreamSynchronize(c.stream));  // the staging buffer may still feed an earlier copy
  PTRY(pinned_stage(c, bytes));
  par_memcpy(c.host_stage, h_src, bytes);
  PCK(cudaMemcpyAsync(d_dst, c.host_stage, bytes, cudaMemcpyHostToDevice, c.stream));
  PCK(cudaStreamSynchronize(c.stream));
  return POBA_OK;
}

int device_to_host(Ctx& c, void* h_dst, const void* d_src, size_t bytes) {
  if (bytes < (4u << 20) || is_pinned(h_dst)) {
    PCK(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, c.stream));
    PCK(cudaStreamSynchronize(c.stream));
    return POBA_OK;
  }
  // pipelined: the DMA of piece i+1 overlaps the host copy of piece i
  PTRY(pinned_stage(c, bytes));
  constexpr int kPieces = 8;
  const size_t piece = ((bytes + kPieces - 1) / kPieces + 4095) & ~(size_t)4095;
  std::vector<cudaEvent_t> ev;
  for (size_t o = 0; o < bytes; o += piece) {
    cudaEvent_t e;
    PCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PCK(cudaMemcpyAsync((char*)c.host_stage + o, (const char*)d_src + o, std::min(piece, bytes - o),
                        cudaMemcpyDeviceToHost, c.stream));
    PCK(cudaEventRecord(e, c.stream));
    ev.push_back(e);
  }
  int st = POBA_OK;
  for (size_t k = 0; k < ev.size(); ++k) {
    const size_t o = k * piece;
    if (st == POBA_OK && cudaEventSynchronize(ev[k]) != cudaSuccess) st = fail(POBA_ECUDA, "device_to_host");
    if (st == POBA_OK) par_memcpy((char*)h_dst + o, (const char*)c.host_stage + o, std::min(piece, bytes - o));
    cudaEventDestroy(ev[k]);
  }
  return st;
}

int lm_upload(Ctx& c, const double* host_full, int width, double* d_local) {
  if (c.n_lm_l == 0) return POBA_OK;
  PTRY(c.lm_stage.alloc(c.n_lm_l * width * 8));
  PTRY(host_to_device(c, c.lm_stage.p, host_full + c.lm_lo * width, c.n_lm_l * width * 8));
  k_lm_gather<<<grid_for(c.n_lm_l * width, 256), 256, 0, c.stream>>>(c.lm_stage.as<double>(), c.lm_perm.as<int>(), 0,
                                                                     c.n_lm_l, width, d_local);
  c.launches++;
  PCK(cudaGetLastError());
  return POBA_OK;
}
int lm_download(Ctx& c, const double* d_local, int width, double* host_full) {
  if (c.n_lm_l == 0) return POBA_OK;
  PTRY(c.lm_stage.alloc(c.n_lm_l * width * 8));
  k_lm_scatter<<<grid_for(c.n_lm_l * width, 256), 256, 0, c.stream>>>(d_local, c.lm_perm.as<int>(), c.n_lm_l, width,
                                                                      c.lm_stage.as<double>());
  c.launches++;
  PCK(cudaGetLastError());
  return device_to_host(c, host_full + c.lm_lo * width, c.lm_stage.p, c.n_lm_l * width * 8);
}

// ---- pipelined landmark transfers (single GPU) ---------------------------------------------
// The landmark range is cut into kXferPieces file-order pieces (cuts planned in
// build_structure).  Upload: piece i is copied on the transfer stream while the
// library stream permutes and consumes the store landmarks whose file rows have
// all arrived; download: the library stream produces a prefix of store
// landmarks, permutes the file-order piece it completes, and the transfer
// stream copies it out while the next prefix is computed.
bool xfer_pipelined(const Ctx& c, int width) {
  size_t min_bytes = kXferMinBytes;
  if (const char* e = getenv("POBA_XFER_MIN_BYTES")) min_bytes = (size_t)strtoull(e, nullptr, 10);  // tests
  return c.nranks == 1 && (int)c.xf_file.size() == kXferPieces + 1 && c.n_lm_l > 0 &&
         (size_t)c.n_lm_l * width * 8 >= min_bytes;
}

int xfer_begin(Ctx& c, int width, bool pinned) {
  if (!c.xfer) {
    PCK(cudaStreamCreateWithFlags(&c.xfer, cudaStreamNonBlocking));
    for (auto& e : c.xfer_ev) PCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const size_t bytes = (size_t)c.n_lm_l * width * 8;
  PTRY(c.lm_stage.alloc(bytes));
  if (!pinned) PTRY(pinned_stage(c, bytes));
  // transfers start after everything already queued on the library stream
  PCK(cudaEventRecord(c.xfer_ev[2 * kXferPieces], c.stream));
  PCK(cudaStreamWaitEvent(c.xfer, c.xfer_ev[2 * kXferPieces], 0));
  return POBA_OK;
}

int lm_upload_piece(Ctx& c, const double* host_full, int width, double* d_local, int i, bool pinned) {
  const int64_t f0 = c.xf_file[i], f1 = c.xf_file[i + 1];
  const size_t off = (size_t)f0 * width * 8, bytes = (size_t)(f1 - f0) * width * 8;
  const char* src = reinterpret_cast<const char*>(host_full + c.lm_lo * width) + off;
  char* stage = c.lm_stage.as<char>() + off;
  if (bytes) {
    if (pinned) {
      PCK(cudaMemcpyAsync(stage, src, bytes, cudaMemcpyHostToDevice, c.xfer));
    } else {  // the host copy of piece i overlaps the device work of piece i - 1
      par_memcpy(static_cast<char*>(c.host_stage) + off, src, bytes);
      PCK(cudaMemcpyAsync(stage, static_cast<char*>(c.host_stage) + off, bytes, cudaMemcpyHostToDevice, c.xfer));
    }
  }
  PCK(cudaEventRecord(c.xfer_ev[i], c.xfer));
  PCK(cudaStreamWaitEvent(c.stream, c.xfer_ev[i], 0));
  const int64_t s0 = c.xf_up_lm[i], s1 = c.xf_up_lm[i + 1];
  if (s1 > s0) {
    k_lm_gather<<<grid_for((s1 - s0) * width, 256), 256, 0, c.stream>>>(c.lm_stage.as<double>(), c.lm_perm.as<int>(),
                                                                       s0, s1, width, d_local);
    c.launches++;
  }
  PCK(cudaGetLastError());
  return POBA_OK;
}

int lm_download_piece(Ctx& c, const double* d_local, int width, double* host_full, int i, bool pinned) {
  const int64_t f0 = c.xf_file[i], f1 = c.xf_file[i + 1];
  const size_t off = (size_t)f0 * width * 8, bytes = (size_t)(f1 - f0) * width * 8;
  if (f1 > f0) {
    k_lm_gather<<<grid_for((f1 - f0) * width, 256), 256, 0, c.stream>>>(d_local, c.lm_inv.as<int>(), f0, f1, width,
                                                                       c.lm_stage.as<double>());
    c.launches++;
    PCK(cudaGetLastError());
  }
  PCK(cudaEventRecord(c.xfer_ev[i], c.stream));
  PCK(cudaStreamWaitEvent(c.xfer, c.xfer_ev[i], 0));
  if (bytes) {
    char* dst = pinned ? reinterpret_cast<char*>(host_full + c.lm_lo * width) + off
                       : static_cast<char*>(c.host_stage) + off;
    PCK(cudaMemcpyAsync(dst, c.lm_stage.as<char>() + off, bytes, cudaMemcpyDeviceToHost, c.xfer));
  }
  PCK(cudaEventRecord(c.xfer_ev[kXferPieces + i], c.xfer));
  return POBA_OK;
}

int lm_download_finish(Ctx& c, double* host_full, int width, bool pinned) {
  if (!pinned) {  // host copies of finished pieces overlap the DMA of later ones
    for (int i = 0; i < kXferPieces; ++i) {
      PCK(cudaEventSynchronize(c.xfer_ev[kXferPieces + i]));
      const size_t off = (size_t)c.xf_file[i] * width * 8;
      const size_t bytes = (size_t)(c.xf_file[i + 1] - c.xf_file[i]) * width * 8;
      if (bytes)
        par_memcpy(reinterpret_cast<char*>(host_full + c.lm_lo * width) + off,
                   static_cast<char*>(c.host_stage) + off, bytes);
    }
  }
  PCK(cudaStreamSynchronize(c.xfer));
  return POBA_OK;
}

namespace {

int copy_down(Ctx& c, const DBuf& src, size_t bytes, std::vector<double>& out) {
  out.resize(bytes / 8);
  PCK(cudaMemcpyAsync(out.data(), src.p, bytes, cudaMemcpyDeviceToHost, c.stream));
  PCK(cudaStreamSynchronize(c.stream));
  return POBA_OK;
}

}  // namespace

}  // namespace poba

using poba::Ctx;
using poba::DBuf;

#define CTX_CHECK(ctx)                                                              \
  do {                                                                              \
    if (!(ctx)) return poba::fail(POBA_EINVAL, "null context");                    \
    cudaError_t e_ = cudaSetDevice((ctx)->c.device);                                \
    if (e_ != cudaSuccess) return poba::fail(POBA_ECUDA, cudaGetErrorString(e_));   \
  } while (0)
#define NEED(cond, msg)                                   \
  do {                                                    \
    if (!(cond)) return poba::fail(POBA_EINVAL, (msg));   \
  } while (0)

extern "C" {

const char* poba_last_error(void) { return poba::g_err.c_str(); }
int poba_version(void) { return 1; }

static int create_common(int device, poba_ctx** out) {
  if (!out) return poba::fail(POBA_EINVAL, "null output pointer");
  int n = 0;
  PCK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return poba::fail(POBA_EINVAL, "no such CUDA device");
  PCK(cudaSetDevice(device));
  poba_ctx* x = new poba_ctx();
  x->c.device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&x->c.stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete x;
    return poba::fail(POBA_ECUDA, cudaGetErrorString(e));
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) x->c.n_sm = prop.multiProcessorCount;
  *out = x;
  return POBA_OK;
}

int poba_create(int device, poba_ctx** out) { return create_common(device, out); }

int poba_nccl_unique_id(void* out) {
  if (!out) return poba::fail(POBA_EINVAL, "null output pointer");
  ncclUniqueId id;
  PNCCL(GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return POBA_OK;
}

int poba_create_sharded(int device, int rank, int nranks, const void* nccl_id, poba_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return poba::fail(POBA_EINVAL, "bad rank / nranks");
  PTRY(create_common(device, out));
  Ctx& c = (*out)->c;
  c.rank = rank;
  c.nranks = nranks;
  if (nranks > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    const poba::NcclApi* api = poba::nccl_api();
    ncclResult_t r = api ? api->CommInitRank(&c.comm, nranks, id, rank) : ncclSystemError;
    if (r != ncclSuccess) {
      std::string msg = api ? std::string("ncclCommInitRank: ") + api->GetErrorString(r) : poba::g_err;
      poba_destroy(*out);
      *out = nullptr;
      return poba::fail(POBA_ENCCL, msg);
    }
  }
  return POBA_OK;
}

int poba_local_group_create(int nranks, void** out) {
  if (!out) return poba::fail(POBA_EINVAL, "null output pointer");
  if (nranks < 1 || nranks > poba::kMaxLocalRanks) return poba::fail(POBA_EINVAL, "bad rank / nranks");
  poba::LocalGroup* g = new poba::LocalGroup();
  g->n = nranks;
  *out = g;
  return POBA_OK;
}

int poba_local_group_destroy(void* group) {
  delete static_cast<poba::LocalGroup*>(group);
  return POBA_OK;
}

int poba_create_local(int device, int rank, int nranks, void* group, poba_ctx** out) {
  poba::LocalGroup* g = static_cast<poba::LocalGroup*>(group);
  if (!g || g->n != nranks || rank < 0 || rank >= nranks) return poba::fail(POBA_EINVAL, "bad rank / nranks");
  PTRY(create_common(device, out));
  (*out)->c.rank = rank;
  (*out)->c.nranks = nranks;
  (*out)->c.group = g;
  return POBA_OK;
}

int poba_destroy(poba_ctx* ctx) {
  if (!ctx) return POBA_OK;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.comm && poba::nccl_api()) poba::nccl_api()->CommDestroy(ctx->c.comm);
  if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  delete ctx;
  return POBA_OK;
}

int poba_set_problem(poba_ctx* ctx, int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_idx,
                     const int64_t* pt_idx, const double* pixels) {
  CTX_CHECK(ctx);
  NEED(n_cam > 0 && n_pt > 0 && n_obs > 0, "problem has no observations");
  NEED(cam_idx && pt_idx, "null index arrays");
  Ctx& c = ctx->c;
  c.n_cam = n_cam;
  c.n_pt = n_pt;
  c.n_obs = n_obs;
  c.have_problem = false;
  PTRY(poba::build_structure(c, cam_idx, pt_idx, pixels));
  return POBA_OK;
}

int poba_set_precision(poba_ctx* ctx, int bits) {
  CTX_CHECK(ctx);
  return poba::set_precision_device(ctx->c, bits);
}

int poba_problem_info(poba_ctx* ctx, int64_t* info) {
  CTX_CHECK(ctx);
  NEED(info, "null output");
  const Ctx& c = ctx->c;
  size_t bytes = 0;
  for (const DBuf* b : {&c.cam_file, &c.pt_file, &c.kpt, &c.order, &c.tiles, &c.tilek, &c.chunks, &c.cta_tiles,
                        &c.cam_s, &c.file_s, &c.pix_s, &c.lidx_s, &c.lm_slot0, &c.lm_k,
                        &c.part_cam_off, &c.part_idx, &c.long_lm, &c.cperm, &c.cam_start, &c.cc_cam_off, &c.cc_cam, &c.lm_c, &c.pix_c, &c.file_c, &c.J,
                        &c.Rz, &c.cams, &c.cams_prep, &c.cams_trial, &c.trial_prep, &c.U0, &c.bp, &c.Dp, &c.Uinv,
                        &c.Ud, &c.bt, &c.tvec, &c.xvec, &c.rvec, &c.cc_part, &c.partials, &c.points, &c.V0, &c.bl,
                        &c.Dl, &c.Vinv, &c.Vd, &c.dl, &c.ltmp, &c.ctmp, &c.ctmp2})
    bytes += b->bytes;
  const int64_t v[16] = {c.have_order ? (int64_t)c.grp_k.size() : -1, c.n_tiles, c.n_chunks, c.n_partials,
                         c.n_obs_l, c.n_slots, c.lm_lo, c.lm_hi, c.max_slots, c.n_long, (int64_t)bytes, c.k_max,
                         c.n_cam, c.n_pt, c.n_obs, c.rank};
  std::memcpy(info, v, sizeof(v));
  return POBA_OK;
}

int poba_term_layout(poba_ctx* ctx, int* table) {
  CTX_CHECK(ctx);
  NEED(table, "null output");
  NEED(ctx->c.have_problem, "no problem");
  *table = ctx->c.chunk_t ? 1 : 0;
  return POBA_OK;
}

int poba_get_ordering(poba_ctx* ctx, int64_t* order, int64_t* cam_sorted, int64_t* pt_sorted) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem, "no problem set");
  PTRY(poba::build_canonical_order(c));
  const int64_t n = c.n_obs;
  std::vector<int> o(n), cf, pf;
  PTRY(poba::copy_sync(c, o.data(), c.order.p, n * 4, cudaMemcpyDeviceToHost));
  if (cam_sorted) {
    cf.resize(n);
    PTRY(poba::copy_sync(c, cf.data(), c.cam_file.p, n * 4, cudaMemcpyDeviceToHost));
  }
  if (pt_sorted) {
    pf.resize(n);
    PTRY(poba::copy_sync(c, pf.data(), c.pt_file.p, n * 4, cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i < n; ++i) {
    if (order) order[i] = o[i];
    if (cam_sorted) cam_sorted[i] = cf[o[i]];
    if (pt_sorted) pt_sorted[i] = pf[o[i]];
  }
  return POBA_OK;
}

int poba_get_groups(poba_ctx* ctx, int64_t cap, int64_t* n_groups, int64_t* k, int64_t* start, int64_t* n) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem, "no problem set");
  PTRY(poba::build_canonical_order(c));
  *n_groups = (int64_t)c.grp_k.size();
  for (int64_t g = 0; g < std::min<int64_t>(cap, *n_groups); ++g) {
    if (k) k[g] = c.grp_k[g];
    if (start) start[g] = c.grp_start[g];
    if (n) n[g] = c.grp_n[g];
  }
  return POBA_OK;
}

int poba_set_points(poba_ctx* ctx, const double* points) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem, "no problem set");
  NEED(points, "null points");
  PTRY(poba::lm_upload(c, points, 3, c.points.as<double>()));
  PCK(cudaStreamSynchronize(c.stream));
  c.have_points = true;
  return POBA_OK;
}

int poba_get_points(poba_ctx* ctx, double* points) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_points, "no device points");
  return poba::lm_download(c, c.points.as<double>(), 3, points);
}

// every rank's landmark rows, gathered (a sharded context's poba_get_points
// fills only its own rows): the ranks' (lm_lo, n_lm_l) pairs are all-gathered
// first, then the file-order rows padded to the largest shard, so the gather
// is exact (no arithmetic on the values).
int poba_get_points_all(poba_ctx* ctx, double* points) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_points, "no device points");
  NEED(points, "null points");
  if (c.nranks <= 1) return poba::lm_download(c, c.points.as<double>(), 3, points);
  const int R = c.nranks;
  DBuf d_rng, d_all;
  PTRY(d_rng.alloc(2 * 8));
  PTRY(d_all.alloc((size_t)2 * R * 8));
  const double rng[2] = {(double)c.lm_lo, (double)c.n_lm_l};
  PTRY(poba::copy_sync(c, d_rng.p, rng, sizeof rng, cudaMemcpyHostToDevice));
  PTRY(poba::allgather(c, d_rng.as<double>(), d_all.as<double>(), 2));
  std::vector<double> all(2 * R);
  PTRY(poba::copy_sync(c, all.data(), d_all.p, all.size() * 8, cudaMemcpyDeviceToHost));
  int64_t maxn = 1;
  for (int r = 0; r < R; ++r) maxn = std::max<int64_t>(maxn, (int64_t)all[2 * r + 1]);
  DBuf d_mine, d_rows;
  PTRY(d_mine.alloc((size_t)maxn * 3 * 8));
  PTRY(d_rows.alloc((size_t)R * maxn * 3 * 8));
  PCK(cudaMemsetAsync(d_mine.p, 0, (size_t)maxn * 3 * 8, c.stream));
  if (c.n_lm_l > 0) {
    poba::k_lm_scatter<<<poba::grid_for(c.n_lm_l * 3, 256), 256, 0, c.stream>>>(c.points.as<double>(), c.lm_perm.as<int>(),
                                                                    c.n_lm_l, 3, d_mine.as<double>());
    c.launches++;
    PCK(cudaGetLastError());
  }
  PTRY(poba::allgather(c, d_mine.as<double>(), d_rows.as<double>(), (size_t)maxn * 3));
  std::vector<double> rows((size_t)R * maxn * 3);
  PTRY(poba::copy_sync(c, rows.data(), d_rows.p, rows.size() * 8, cudaMemcpyDeviceToHost));
  for (int r = 0; r < R; ++r) {
    const int64_t lo = (int64_t)all[2 * r], n = (int64_t)all[2 * r + 1];
    std::memcpy(points + lo * 3, rows.data() + (size_t)r * maxn * 3, (size_t)n * 3 * 8);
  }
  return POBA_OK;
}

int poba_accept_points(poba_ctx* ctx) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_points && c.have_delta_l, "no back-substituted landmark step");
  return poba::points_accept_device(c);
}

int poba_linearize(poba_ctx* ctx, const double* cam_params, const double* points, int64_t* n_invalid) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem, "no problem set");
  NEED(c.have_pixels, "problem was set without pixels");
  NEED(cam_params, "null camera parameters");
  const bool piped = points && poba::xfer_pipelined(c, 3);
  if (points && !piped) PTRY(poba_set_points(ctx, points));
  NEED(piped || c.have_points, "no points (pass them or call poba_set_points)");
  PCK(cudaMemcpyAsync(c.cams.p, cam_params, c.n_cam * 9 * 8, cudaMemcpyHostToDevice, c.stream));
  const int st = poba::linearize_device(c, false, nullptr, nullptr, nullptr, piped ? points : nullptr);
  if (piped) c.have_points = st == POBA_OK;  // the device copy now holds these points
  PTRY(st);
  if (n_invalid) *n_invalid = c.n_invalid;
  return POBA_OK;
}

int poba_linearize_explicit(poba_ctx* ctx, const double* jp, const double* jl, const double* res) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem, "no problem set");
  NEED(jp && jl && res, "null Jacobian arrays");
  PTRY(poba::linearize_device(c, true, jp, jl, res));
  return POBA_OK;
}

int poba_damp(poba_ctx* ctx, double lam, int identity) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_lin, "no linearization");
  if (!(lam >= 0)) return poba::fail(POBA_EINVAL, "lambda must be non-negative");
  return poba::damp_device(c, lam, identity ? 1 : 0);
}

int poba_series_solve(poba_ctx* ctx, double epsilon, int max_order, double* delta_p, int* order_used,
                      int* converged, double* ratios) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  if (max_order < 0) return poba::fail(POBA_EINVAL, "max_order must be non-negative");
  if (!(epsilon > 0)) return poba::fail(POBA_EINVAL, "epsilon must be positive");
  int ou = 0, cv = 0;
  PTRY(poba::series_device(c, epsilon, max_order, false, &ou, &cv));
  if (order_used) *order_used = ou;
  if (converged) *converged = cv;
  if (delta_p) {
    PCK(cudaMemcpyAsync(delta_p, c.xvec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToHost, c.stream));
  }
  if (ratios) {
    PCK(cudaMemcpyAsync(ratios, c.ratios.p, (size_t)(max_order + 1) * 8, cudaMemcpyDeviceToHost, c.stream));
  }
  PCK(cudaStreamSynchronize(c.stream));
  return POBA_OK;
}

int poba_series_apply(poba_ctx* ctx, const double* v, int order, double* out) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  if (order < 0) return poba::fail(POBA_EINVAL, "order must be non-negative");
  NEED(v && out, "null vectors");
  PCK(cudaMemcpyAsync(c.ctmp.p, v, c.n_cam * 9 * 8, cudaMemcpyHostToDevice, c.stream));
  PTRY(poba::series_apply_device(c, c.ctmp.as<double>(), order, c.ctmp2.as<double>()));
  PTRY(poba::copy_sync(c, out, c.ctmp2.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToHost));
  return POBA_OK;
}

// PoST: landmark damping diagonal override (restrict_system keeps the global D_l,
// clustering.py:118-119) and the clustered series with per-cluster stop tests
int poba_set_dl(poba_ctx* ctx, const double* d_l) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_lin, "no linearization");
  NEED(d_l, "null D_l");
  PTRY(poba::lm_upload(c, d_l, 3, c.Dl.as<double>()));
  PCK(cudaStreamSynchronize(c.stream));
  c.have_damp = c.have_solution = c.have_delta_l = false;
  return POBA_OK;
}

int poba_series_solve_clustered(poba_ctx* ctx, const int64_t* cluster_of_cam, int n_clusters, double epsilon,
                                int max_order, double* delta_p, int* order_used, int* converged) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  NEED(cluster_of_cam && n_clusters >= 1, "no clustering");
  NEED(order_used && converged, "null outputs");
  if (max_order < 0) return poba::fail(POBA_EINVAL, "max_order must be non-negative");
  if (!(epsilon > 0)) return poba::fail(POBA_EINVAL, "epsilon must be positive");
  return poba::series_clustered_device(c, cluster_of_cam, n_clusters, epsilon, max_order, delta_p, order_used,
                                       converged);
}

int poba_schur_diagonal(poba_ctx* ctx, double* blocks_81) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  PTRY(poba::schur_diag_device(c, nullptr));
  if (blocks_81) {
    std::vector<double> m45(c.n_cam * 45);
    PTRY(poba::copy_sync(c, m45.data(), c.Mbuf.p, m45.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t q = 0; q < c.n_cam; ++q)
      for (int i = 0, k = 0; i < 9; ++i)
        for (int j = i; j < 9; ++j, ++k) {
          blocks_81[q * 81 + i * 9 + j] = m45[q * 45 + k];
          blocks_81[q * 81 + j * 9 + i] = m45[q * 45 + k];
        }
  }
  return POBA_OK;
}

int poba_pcg(poba_ctx* ctx, int precond, int order, double tol, int max_iter, int resume, double* delta_p,
             int* iterations, double* final_rel, int* converged, double* rel_history) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  NEED(precond == POBA_PRECOND_SCHUR_JACOBI || precond == POBA_PRECOND_SERIES, "unknown preconditioner");
  if (precond == POBA_PRECOND_SERIES && order < 0) return poba::fail(POBA_EINVAL, "order must be non-negative");
  NEED(max_iter >= 0, "max_iter must be non-negative");
  NEED(iterations && final_rel && converged, "null outputs");
  c.have_solution = false;
  PTRY(poba::pcg_device(c, precond, order, tol, max_iter, resume != 0, delta_p, iterations, final_rel, converged,
                        rel_history));
  // the PCG iterate is the device-side delta_p for poba_back_substitute(ctx, NULL, ...)
  PCK(cudaMemcpyAsync(c.xvec.p, c.pcg_vec.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToDevice, c.stream));
  PCK(cudaStreamSynchronize(c.stream));
  c.have_solution = true;
  return POBA_OK;
}

int poba_back_substitute(poba_ctx* ctx, const double* delta_p, double* delta_l, int* nonzero) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  const double* d_dp = c.xvec.as<double>();
  if (delta_p) {
    PCK(cudaMemcpyAsync(c.ctmp.p, delta_p, c.n_cam * 9 * 8, cudaMemcpyHostToDevice, c.stream));
    d_dp = c.ctmp.as<double>();
  } else {
    NEED(c.have_solution, "no series solution on the device");
  }
  int nz = 0;
  PTRY(poba::back_substitute_device(c, d_dp, &nz, delta_l));
  if (nonzero) *nonzero = nz;
  return POBA_OK;
}

int poba_cost(poba_ctx* ctx, const double* cam_params, const double* points, int trial, double* cost,
              int64_t* n_invalid) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_problem && c.have_pixels, "no problem with pixels");
  NEED(cam_params, "null camera parameters");
  PCK(cudaMemcpyAsync(c.cams_trial.p, cam_params, c.n_cam * 9 * 8, cudaMemcpyHostToDevice, c.stream));
  PTRY(poba::cameras_prep(c, c.cams_trial.as<double>(), c.trial_prep.as<double>()));
  if (trial) NEED(c.have_delta_l, "no landmark step for the trial cost");
  double v = 0;
  int64_t bad = 0;
  if (points) {
    // explicit points: evaluate on a scratch copy, device state untouched
    DBuf saved;
    PTRY(saved.alloc(std::max<int64_t>(c.n_lm_l, 1) * 24));
    PCK(cudaMemcpyAsync(saved.p, c.points.p, c.n_lm_l * 24, cudaMemcpyDeviceToDevice, c.stream));
    PTRY(poba::lm_upload(c, points, 3, c.points.as<double>()));
    int st = poba::cost_device(c, trial != 0, &v, &bad);
    cudaMemcpyAsync(c.points.p, saved.p, c.n_lm_l * 24, cudaMemcpyDeviceToDevice, c.stream);
    cudaStreamSynchronize(c.stream);
    PTRY(st);
  } else {
    NEED(c.have_points, "no device points");
    PTRY(poba::cost_device(c, trial != 0, &v, &bad));
  }
  if (cost) *cost = v;
  if (n_invalid) *n_invalid = bad;
  return POBA_OK;
}

int poba_apply(poba_ctx* ctx, int op, const double* in, double* out) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(in && out, "null vectors");
  NEED(c.have_lin, "no linearization");
  const bool in_lm = (op == POBA_OP_W || op == POBA_OP_V_INV);
  const bool out_lm = (op == POBA_OP_WT || op == POBA_OP_V_INV);
  if (op != POBA_OP_W && op != POBA_OP_WT) NEED(c.have_damp, "no damped system");
  DBuf din, dout;
  PTRY(din.alloc((in_lm ? std::max<int64_t>(c.n_lm_l, 1) * 3 : c.n_cam * 9) * 8));
  PTRY(dout.alloc((out_lm ? std::max<int64_t>(c.n_lm_l, 1) * 3 : c.n_cam * 9) * 8));
  if (in_lm) PTRY(poba::lm_upload(c, in, 3, din.as<double>()));
  else PCK(cudaMemcpyAsync(din.p, in, c.n_cam * 9 * 8, cudaMemcpyHostToDevice, c.stream));
  PTRY(poba::apply_op_device(c, op, din.as<double>(), dout.as<double>()));
  // (the camera merge of OP_W / OP_WVW already all-reduces across ranks)
  if (out_lm) {
    PTRY(poba::lm_download(c, dout.as<double>(), 3, out));
  } else {
    PCK(cudaMemcpyAsync(out, dout.p, c.n_cam * 9 * 8, cudaMemcpyDeviceToHost, c.stream));
    PCK(cudaStreamSynchronize(c.stream));
  }
  return POBA_OK;
}

int poba_read(poba_ctx* ctx, int what, double* dst) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(dst, "null output");
  NEED(c.have_lin, "no linearization");
  std::vector<double> h;
  const int64_t nc = c.n_cam, nl = c.n_lm_l;
  auto scatter_lm = [&](const std::vector<double>& src, int width) {  // store order -> file rows
    for (int64_t j = 0; j < nl; ++j)
      std::memcpy(dst + (c.lm_lo + c.lm_order_host[j]) * width, src.data() + j * width, width * 8);
  };
  auto lm_sym = [&](const DBuf& b) -> int {
    PTRY(poba::copy_down(c, b, nl * 6 * 8, h));
    std::vector<double> full(nl * 9);
    for (int64_t j = 0; j < nl; ++j) poba::unpack3(h.data() + j * 6, full.data() + j * 9);
    scatter_lm(full, 9);
    return POBA_OK;
  };
  auto cam_sym = [&](const DBuf& b) -> int {
    PTRY(poba::copy_down(c, b, nc * 45 * 8, h));
    for (int64_t q = 0; q < nc; ++q) poba::unpack9(h.data() + q * 45, dst + q * 81);
    return POBA_OK;
  };
  const bool damped = what == POBA_READ_U || what == POBA_READ_V || what == POBA_READ_U_INV ||
                      what == POBA_READ_V_INV || what == POBA_READ_B_TILDE;
  if (damped) NEED(c.have_damp, "no damped system");
  switch (what) {
    case POBA_READ_U0: return cam_sym(c.U0);
    case POBA_READ_U: return cam_sym(c.Ud);
    case POBA_READ_U_INV: return cam_sym(c.Uinv);
    case POBA_READ_V0: return lm_sym(c.V0);
    case POBA_READ_V: return lm_sym(c.Vd);
    case POBA_READ_V_INV: return lm_sym(c.Vinv);
    case POBA_READ_B_P:
      PTRY(poba::copy_down(c, c.bp, nc * 72, h));
      std::memcpy(dst, h.data(), nc * 72);
      return POBA_OK;
    case POBA_READ_D_P:
      PTRY(poba::copy_down(c, c.Dp, nc * 72, h));
      std::memcpy(dst, h.data(), nc * 72);
      return POBA_OK;
    case POBA_READ_B_L:
      PTRY(poba::copy_down(c, c.bl, nl * 24, h));
      scatter_lm(h, 3);
      return POBA_OK;
    case POBA_READ_D_L:
      PTRY(poba::copy_down(c, c.Dl, nl * 24, h));
      scatter_lm(h, 3);
      return POBA_OK;
    case POBA_READ_B_TILDE: {
      // b_tilde = b_p - W V^-1 b_l (blocks.py:256-260), recomputed on demand
      PTRY(poba::b_tilde_device(c));
      PTRY(poba::copy_down(c, c.bt, nc * 72, h));
      std::memcpy(dst, h.data(), nc * 72);
      return POBA_OK;
    }
    case POBA_READ_STORAGE: {
      // (n_obs, 2, 13) rows in the reference's canonical order; rows of
      // observations owned by other ranks are left untouched
      PTRY(poba::build_canonical_order(c));
      const int64_t ns = c.n_slots, n = c.n_obs;
      // tile blocks: 32 metadata words, then 12 planes of 32 column pairs
      const int64_t per_tile = 12 * poba::kTile * 2;  // values per tile (after the metadata)
      std::vector<double> J((size_t)c.n_tiles * per_tile), R(ns * 2);
      if (c.precision == 32) {  // fp32 store: widen (exact) for the float64 caller
        std::vector<float> Jf((size_t)c.n_tiles * poba::kTileBlockF32 / 4);
        PTRY(poba::copy_sync(c, Jf.data(), c.J.p, Jf.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < c.n_tiles; ++t)
          for (int64_t q = 0; q < per_tile; ++q)
            J[t * per_tile + q] = (double)Jf[t * (poba::kTileBlockF32 / 4) + poba::kMetaBytes / 4 + q];
      } else {
        std::vector<double> Jd((size_t)c.n_tiles * poba::kTileBlock / 8);
        PTRY(poba::copy_sync(c, Jd.data(), c.J.p, Jd.size() * 8, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < c.n_tiles; ++t)
          std::memcpy(&J[t * per_tile], &Jd[t * (poba::kTileBlock / 8) + poba::kMetaBytes / 8], per_tile * 8);
      }
      std::vector<int> file(ns), order(n), slot_of_file(n, -1);
      PTRY(poba::copy_sync(c, R.data(), c.Rz.p, R.size() * 8, cudaMemcpyDeviceToHost));
      PTRY(poba::copy_sync(c, file.data(), c.file_s.p, ns * 4, cudaMemcpyDeviceToHost));
      PTRY(poba::copy_sync(c, order.data(), c.order.p, n * 4, cudaMemcpyDeviceToHost));
      for (int64_t q = 0; q < ns; ++q)
        if (file[q] >= 0) slot_of_file[file[q]] = (int)q;
      for (int64_t i = 0; i < n; ++i) {
        const int64_t q = slot_of_file[order[i]];
        if (q < 0) continue;
        for (int a = 0; a < 2; ++a) {
          double* row = dst + (i * 2 + a) * 13;
          for (int j = 0; j < 12; ++j) row[j] = J[(q >> 5) * per_tile + (j * poba::kTile + (q & 31)) * 2 + a];
          row[12] = R[q * 2 + a];
        }
      }
      return POBA_OK;
    }
    default:
      return poba::fail(POBA_EINVAL, "unknown read target");
  }
}

int poba_time_terms(poba_ctx* ctx, int reps, double* ms_per_term, double* ms_term_kernel, int* launches) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  NEED(reps > 0, "reps must be positive");
  return poba::time_terms_device(c, reps, ms_per_term, ms_term_kernel, launches);
}

int poba_spectral_radius(poba_ctx* ctx, const double* v0, double tol, int max_iter, double* rho, int* iterations,
                         int* converged) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  NEED(v0 && rho && iterations && converged, "null arguments");
  return poba::spectral_radius_device(c, v0, tol, max_iter, rho, iterations, converged);
}

int poba_materialize(poba_ctx* ctx, int op, int64_t limit, double* out) {
  CTX_CHECK(ctx);
  Ctx& c = ctx->c;
  NEED(c.have_damp, "no damped system");
  NEED(out, "null output");
  return poba::materialize_device(c, op, limit, out);
}

int64_t poba_launch_count(poba_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

// landmark bounds of every rank's shard (host-only; no GPU needed)
int poba_shard_bounds(int64_t n_pt, const int64_t* k_per_point, int nranks, int64_t* lm_bounds) {
  if (n_pt <= 0 || !k_per_point || !lm_bounds || nranks < 1) return poba::fail(POBA_EINVAL, "bad arguments");
  std::vector<int> k(n_pt);
  for (int64_t j = 0; j < n_pt; ++j) {
    if (k_per_point[j] < 1) return poba::fail(POBA_EINVAL, "every point must be observed at least once");
    k[j] = (int)k_per_point[j];
  }
  poba::TilePlan plan;
  poba::plan_tiles(k.data(), n_pt, plan);
  const int64_t n_obs = plan.lm_first[n_pt];
  for (int r = 0; r <= nranks; ++r) {
    const size_t t = poba::shard_cut(plan, n_obs, r, nranks);
    lm_bounds[r] = t < plan.tiles.size() ? plan.tiles[t].lm0 : n_pt;
  }
  return POBA_OK;
}

int poba_stream(poba_ctx* ctx, void** stream) {
  NEED(ctx && stream, "null argument");
  *stream = (void*)ctx->c.stream;
  return POBA_OK;
}

}  // extern "C"
