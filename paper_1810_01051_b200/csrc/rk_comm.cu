// rk_comm.cu -- the multi-GPU data plane behind the C ABI: NCCL communicators and the
// sharded scan (include/rkb200.h, "Multi-GPU").
//
// The reference splits the window range into contiguous ranges, scans them independently
// and concatenates the per-range lists in range order
// (/root/reference/pkg/src/rkmatch/parallel.py:155-172).  Here a range is a GPU (one
// process per GPU): each rank scans its shard -- its windows plus the (m-1)-byte halo
// their last bytes need -- with no traffic during the scan, and the one exchange is the
// final gather, an allgather-v over NVLink/NVSwitch:
//   1. ncclAllGather of every rank's {matches, hash_hits, collisions} (32 bytes per rank);
//   2. one grouped ncclBroadcast per rank with matches, rooted at that rank, whose receive
//      buffer on every rank is the output at the rank's prefix offset -- the positions
//      land in place, already globally ascending (rank order = range order), with no
//      padding to the largest count and no copy after the collective.
// NCCL is loaded at run time (dlopen of libnccl.so.2, i.e. the one torch already mapped
// when it is loaded), so the library still loads where NCCL is absent and only the
// rk_comm_* entry points report RK_ENCCL there.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "rk_ctx.h"

using namespace rkb;

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  int version = 0;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* path = getenv("RKB200_NCCL_LIB");
    void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      all = all && fn != nullptr;
    };
    sym(api.GetVersion, "ncclGetVersion");
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.AllGather, "ncclAllGather");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (!all) {
      api.err = "NCCL library lacks a required symbol";
      return;
    }
    api.GetVersion(&api.version);
    api.ok = true;
  });
  return api;
}

#define RK_NCCL(call)                                                                       \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return fail(RK_ENCCL, "%s failed: %s (%s:%d)", #call, nccl().GetErrorString(r_),      \
                  __FILE__, __LINE__);                                                      \
  } while (0)

}  // namespace

struct rk_comm {
  rk_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
  unsigned long long* d_cnt = nullptr;     // this rank's {matches, hash_hits, collisions, 0}
  unsigned long long* d_allcnt = nullptr;  // every rank's, rank-major
  unsigned long long* h_allcnt = nullptr;  // pinned mirror
  int64_t* d_local = nullptr;              // this rank's ordered offsets (device texts)
  uint64_t local_cap = 0;
  int64_t* d_gather = nullptr;             // whole gathered list when the caller's cap < total
  uint64_t gather_cap = 0;
  // multi-pattern shards: this rank's pairs, and every rank's gathered
  int64_t* d_moff = nullptr;
  uint32_t* d_midx = nullptr;
  uint64_t m_cap = 0;
  int64_t* d_goff = nullptr;
  uint32_t* d_gidx = nullptr;
  uint64_t g_cap = 0;
  uint64_t gathered = 0;                   // offsets of the last sharded scan in d_gather
  // batched sharded scans: per pattern, this rank's offsets and counters
  std::vector<int64_t*> b_local;
  std::vector<uint64_t> b_cap;
  unsigned long long* d_bcnt = nullptr;     // 4 x RK_BATCH_MAX_PATTERNS, this rank's
  unsigned long long* d_ballcnt = nullptr;  // every rank's, rank-major
  unsigned long long* h_ballcnt = nullptr;  // pinned mirror
  // asynchronous batches: this rank's slabs (P x slab ordered offsets), every rank's,
  // and the counters (P x 4, every rank's rank-major)
  int64_t* a_local = nullptr;
  int64_t* a_all = nullptr;
  uint64_t a_local_cap = 0, a_all_cap = 0;
  unsigned long long* a_cnt = nullptr;
  unsigned long long* a_allcnt = nullptr;
};

namespace {
struct SlabOuts {  // the kernel parameter: every pattern's output and its capacity
  int64_t* out[RK_BATCH_MAX_PATTERNS];
  uint64_t cap[RK_BATCH_MAX_PATTERNS];
};

// Block (pattern i, rank r): rank r's ordered offsets of pattern i (its slab) to their
// place in the global list, after every earlier rank's; block (i, 0) also writes pattern
// i's totals {matches, hash_hits, collisions, overflow} to counts.
__global__ void slab_compact_kernel(const int64_t* __restrict__ all,
                                    const unsigned long long* __restrict__ allcnt, uint32_t P,
                                    uint64_t slab, int nranks, SlabOuts o,
                                    unsigned long long* counts) {
  const uint32_t i = blockIdx.x;
  const int r = (int)blockIdx.y;
  uint64_t prefix = 0, total = 0, hits = 0, coll = 0;
  bool over = false;
  for (int q = 0; q < nranks; ++q) {
    const unsigned long long* c = allcnt + 4ull * ((uint64_t)q * P + i);
    if (q < r) prefix += c[0];
    total += c[0];
    hits += c[1];
    coll += c[2];
    over |= c[0] > slab;
  }
  const uint64_t cnt = allcnt[4ull * ((uint64_t)r * P + i)];
  const uint64_t n = cnt < slab ? cnt : slab;
  const int64_t* src = all + ((uint64_t)r * P + i) * slab;
  for (uint64_t j = threadIdx.x; j < n; j += blockDim.x)
    if (prefix + j < o.cap[i]) o.out[i][prefix + j] = src[j];
  if (r == 0 && threadIdx.x == 0) {
    counts[4ull * i + 0] = total;
    counts[4ull * i + 1] = hits;
    counts[4ull * i + 2] = coll;
    counts[4ull * i + 3] = over ? 1ull : 0ull;
  }
}
}  // namespace

extern "C" {

int rk_comm_get_unique_id(uint8_t* id) {
  if (!id) return fail(RK_EINVAL, "id is NULL");
  NcclApi& api = nccl();
  if (!api.ok) return fail(RK_ENCCL, "%s", api.err.c_str());
  ncclUniqueId u;
  RK_NCCL(api.GetUniqueId(&u));
  static_assert(sizeof(u) == RK_COMM_ID_BYTES, "NCCL unique id size");
  memcpy(id, &u, sizeof u);
  return RK_OK;
}

int rk_comm_init(rk_ctx_t* c, const uint8_t* id, int nranks, int rank, rk_comm_t** out) {
  if (!out) return fail(RK_EINVAL, "out is NULL");
  *out = nullptr;
  if (!c || !id) return fail(RK_EINVAL, "context or id is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(RK_EINVAL, "rank %d outside [0, %d)", rank, nranks);
  NcclApi& api = nccl();
  if (!api.ok) return fail(RK_ENCCL, "%s", api.err.c_str());
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  rk_comm* k = new rk_comm();
  k->ctx = c;
  k->nranks = nranks;
  k->rank = rank;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclResult_t r = api.CommInitRank(&k->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete k;
    return fail(RK_ENCCL, "ncclCommInitRank(rank %d of %d) failed: %s", rank, nranks,
                api.GetErrorString(r));
  }
  cudaError_t e = cudaMalloc(&k->d_cnt, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&k->d_allcnt, 4ull * nranks * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMallocHost(&k->h_allcnt, 4ull * nranks * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(k->d_cnt, 0, 4 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    api.CommDestroy(k->comm);
    cudaFree(k->d_cnt);
    cudaFree(k->d_allcnt);
    delete k;
    return fail(RK_ECUDA, "comm scratch: %s", cudaGetErrorString(e));
  }
  const char* log = getenv("RKB200_COMM_LOG");
  if (log && *log && *log != '0')
    fprintf(stderr, "[rkb200] comm rank %d/%d on device %d, NCCL %d\n", rank, nranks, c->device,
            api.version);
  *out = k;
  return RK_OK;
}

int rk_comm_destroy(rk_comm_t* k) {
  if (!k) return RK_OK;
  DeviceGuard g(k->ctx->device);
  cudaDeviceSynchronize();
  if (k->comm) nccl().CommDestroy(k->comm);
  cudaFree(k->d_cnt);
  cudaFree(k->d_allcnt);
  cudaFreeHost(k->h_allcnt);
  cudaFree(k->d_local);
  cudaFree(k->d_gather);
  for (int64_t* p : k->b_local) cudaFree(p);
  cudaFree(k->d_bcnt);
  cudaFree(k->d_ballcnt);
  cudaFree(k->a_local);
  cudaFree(k->a_all);
  cudaFree(k->a_cnt);
  cudaFree(k->a_allcnt);
  cudaFreeHost(k->h_ballcnt);
  cudaFree(k->d_moff);
  cudaFree(k->d_midx);
  cudaFree(k->d_goff);
  cudaFree(k->d_gidx);
  delete k;
  return RK_OK;
}

int rk_comm_info(rk_comm_t* k, int* nranks, int* rank, int* nccl_version) {
  if (!k) return fail(RK_EINVAL, "communicator is NULL");
  if (nranks) *nranks = k->nranks;
  if (rank) *rank = k->rank;
  if (nccl_version) *nccl_version = nccl().version;
  return RK_OK;
}

int rk_shard_range(uint64_t n, uint32_t m, int nranks, int rank, uint64_t* win_lo,
                   uint64_t* win_hi, uint64_t* byte_lo, uint64_t* byte_hi) {
  if (m < 1) return fail(RK_EINVAL, "pattern must be non-empty");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(RK_EINVAL, "rank %d outside [0, %d)", rank, nranks);
  // parallel.py:155-161: ceil(W / G) windows per range, capped at W
  const uint64_t W = n >= m ? n - m + 1 : 0;
  const uint64_t chunk = (W + (uint64_t)nranks - 1) / (uint64_t)nranks;
  const uint64_t a = std::min<uint64_t>((uint64_t)rank * chunk, W);
  const uint64_t b = std::min<uint64_t>(a + chunk, W);
  if (win_lo) *win_lo = a;
  if (win_hi) *win_hi = b;
  if (byte_lo) *byte_lo = a;
  if (byte_hi) *byte_hi = b > a ? std::min<uint64_t>(b + m - 1, n) : a;
  return RK_OK;
}

int rk_scan_sharded(rk_comm_t* k, const uint8_t* text, uint64_t len, uint64_t byte_lo,
                    const uint8_t* h_pattern, uint32_t m, uint64_t hx, uint64_t win_lo,
                    uint64_t win_hi, int64_t* d_out, uint64_t cap, uint64_t* matches,
                    uint64_t* collisions, uint64_t* hash_hits, void* stream) {
  if (!k) return fail(RK_EINVAL, "communicator is NULL");
  if (!h_pattern || m < 1) return fail(RK_EINVAL, "pattern must be non-empty");
  if (win_hi > win_lo) {
    if (win_lo < byte_lo || win_hi - byte_lo + m - 1 > len)
      return fail(RK_EINVAL, "windows [%llu, %llu) of length %u need bytes the shard [%llu, "
                  "%llu) does not hold", (unsigned long long)win_lo,
                  (unsigned long long)win_hi, m, (unsigned long long)byte_lo,
                  (unsigned long long)(byte_lo + len));
    if (!text) return fail(RK_EINVAL, "text pointer is NULL");
  }
  if (cap && !d_out) return fail(RK_EINVAL, "output pointer is NULL with cap > 0");
  rk_ctx* c = k->ctx;
  NcclApi& api = nccl();
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t start = win_hi > win_lo ? win_lo - byte_lo : 0;
  const uint64_t stop = win_hi > win_lo ? win_hi - byte_lo : 0;
  const bool on_device = stop > start && is_device_pointer(text, c->device);
  if (stop > start && !on_device) {
    cudaPointerAttributes attr;
    const bool other = cudaPointerGetAttributes(&attr, text) == cudaSuccess &&
                       attr.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    if (other)
      return fail(RK_EINVAL, "text is device memory of device %d, the communicator's is %d",
                  attr.device, c->device);
  }

  // 1. the local scan: ordered offsets (biased to global positions) + counters in d_cnt
  int64_t** local = &k->d_local;
  uint64_t* local_cap = &k->local_cap;
  if (stop > start && !on_device) {
    // host shard: staged into HBM chunk by chunk on the context's streams
    if (int r = enter(c, c->s_comp)) return r;
    if (int r = grow(&c->d_out_stage, &c->out_stage_cap, 1ull << 16, false, c->s_comp)) return r;
    if (int r = host_scan_enqueue(c, text, len, h_pattern, m, hx, start, stop, (int64_t)byte_lo,
                                  (uint64_t*)k->d_cnt))
      return r;
    local = &c->d_out_stage;
    local_cap = &c->out_stage_cap;
    if (int r = enter(c, s)) return r;  // s waits for the staged scan
  } else {
    if (int r = enter(c, s)) return r;
    if (int r = grow(&k->d_local, &k->local_cap, 1ull << 16, false, s)) return r;
    if (int r = enqueue_scan(c, text, len, h_pattern, m, hx, start, stop, k->d_local,
                             k->local_cap, (int64_t)byte_lo, s, (uint64_t*)k->d_cnt))
      return r;
  }

  // 2. every rank's counters (32 bytes per rank) to every rank
  RK_NCCL(api.AllGather(k->d_cnt, k->d_allcnt, 4, ncclUint64, k->comm, s));
  RK_CUDA(cudaMemcpyAsync(k->h_allcnt, k->d_allcnt, 4ull * k->nranks * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaStreamSynchronize(s));
  std::vector<uint64_t> cnt(k->nranks), prefix(k->nranks + 1, 0);
  uint64_t hits = 0, coll = 0;
  for (int r = 0; r < k->nranks; ++r) {
    cnt[r] = k->h_allcnt[4 * r];
    hits += k->h_allcnt[4 * r + 1];
    coll += k->h_allcnt[4 * r + 2];
    prefix[r + 1] = prefix[r] + cnt[r];
  }
  const uint64_t total = prefix[k->nranks];
  const uint64_t mine = cnt[k->rank];
  if (mine > *local_cap) {
    // more local matches than the first emission held: re-emit from the kept per-tile
    // results (never a rescan)
    if (int r = grow(local, local_cap, mine, false, s)) return r;
    if (int r = emit_last(c, *local, mine, s)) return r;
  }

  // 3. allgather-v: rank r's list broadcast from r into every rank's output at prefix[r]
  k->gathered = 0;
  if (total) {
    int64_t* recv = d_out;
    if (cap < total) {
      if (int r = grow(&k->d_gather, &k->gather_cap, total, false, s)) return r;
      recv = k->d_gather;
    }
    RK_NCCL(api.GroupStart());
    for (int r = 0; r < k->nranks; ++r) {
      if (!cnt[r]) continue;
      const void* send = r == k->rank ? (const void*)*local : (const void*)(recv + prefix[r]);
      ncclResult_t e = api.Broadcast(send, recv + prefix[r], cnt[r], ncclInt64, r, k->comm, s);
      if (e != ncclSuccess) {
        api.GroupEnd();
        return fail(RK_ENCCL, "ncclBroadcast(root %d) failed: %s", r, api.GetErrorString(e));
      }
    }
    RK_NCCL(api.GroupEnd());
    if (recv != d_out) {
      k->gathered = total;
      if (cap)
        RK_CUDA(cudaMemcpyAsync(d_out, recv, cap * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    }
  }
  if (matches) *matches = total;
  if (hash_hits) *hash_hits = hits;
  if (collisions) *collisions = coll;
  return RK_OK;
}

int rk_scan_sharded_batch(rk_comm_t* k, const uint8_t* d_text, uint64_t len, uint64_t byte_lo,
                          const uint8_t* h_patterns, const uint32_t* h_lengths,
                          const uint64_t* h_hashes, uint32_t P, const uint64_t* win_lo,
                          const uint64_t* win_hi, int64_t* const* d_outs, const uint64_t* caps,
                          uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
                          void* stream) {
  if (!k) return fail(RK_EINVAL, "communicator is NULL");
  if (P < 1 || P > RK_BATCH_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_BATCH_MAX_PATTERNS);
  if (!h_patterns || !h_lengths || !h_hashes || !win_lo || !win_hi || !d_outs || !caps ||
      !matches || !collisions || !hash_hits)
    return fail(RK_EINVAL, "NULL argument array");
  uint64_t off = 0;
  std::vector<uint64_t> pat_off(P);
  for (uint32_t i = 0; i < P; ++i) {
    const uint32_t m = h_lengths[i];
    if (m < 1) return fail(RK_EINVAL, "pattern %u is empty", i);
    pat_off[i] = off;
    off += m;
    if (win_hi[i] > win_lo[i]) {
      if (win_lo[i] < byte_lo || win_hi[i] - byte_lo + m - 1 > len)
        return fail(RK_EINVAL, "pattern %u: windows [%llu, %llu) need bytes the shard does not "
                    "hold", i, (unsigned long long)win_lo[i], (unsigned long long)win_hi[i]);
      if (!d_text) return fail(RK_EINVAL, "text pointer is NULL");
    }
    if (caps[i] && !d_outs[i]) return fail(RK_EINVAL, "pattern %u: NULL output", i);
  }
  rk_ctx* c = k->ctx;
  NcclApi& api = nccl();
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (d_text && len && !is_device_pointer(d_text, c->device))
    return fail(RK_EINVAL, "rk_scan_sharded_batch takes device texts of the context's device");
  if (int r = enter(c, s)) return r;
  if (!k->d_bcnt) {
    RK_CUDA(cudaMalloc(&k->d_bcnt, 4ull * RK_BATCH_MAX_PATTERNS * sizeof(unsigned long long)));
    RK_CUDA(cudaMalloc(&k->d_ballcnt,
                       4ull * RK_BATCH_MAX_PATTERNS * k->nranks * sizeof(unsigned long long)));
    RK_CUDA(cudaMallocHost(&k->h_ballcnt,
                           4ull * RK_BATCH_MAX_PATTERNS * k->nranks * sizeof(unsigned long long)));
  }
  if (k->b_local.size() < P) {
    k->b_local.resize(P, nullptr);
    k->b_cap.resize(P, 0);
  }
  // 1. every pattern's local scan, back to back (no host round trip between them); each
  //    keeps its ordered offsets in its own buffer (sized by the previous call's counts)
  const auto local_scan = [&](uint32_t i) -> int {
    const uint32_t m = h_lengths[i];
    const uint64_t start = win_hi[i] > win_lo[i] ? win_lo[i] - byte_lo : 0;
    const uint64_t stop = win_hi[i] > win_lo[i] ? win_hi[i] - byte_lo : 0;
    if (int r = grow(&k->b_local[i], &k->b_cap[i], 1ull << 12, false, s)) return r;
    return enqueue_scan(c, d_text, len, h_patterns + pat_off[i], m, h_hashes[i], start, stop,
                        k->b_local[i], k->b_cap[i], (int64_t)byte_lo, s,
                        (uint64_t*)(k->d_bcnt + 4ull * i));
  };
  for (uint32_t i = 0; i < P; ++i)
    if (int r = local_scan(i)) return r;
  // 2. every rank's counters of every pattern -- {matches, hash_hits, collisions, the
  //    rank's buffer size} -- in one all-gather and one host read.  A pattern with more
  //    local offsets than its buffer held on some rank makes every rank take a second
  //    round (the same decision everywhere, from the gathered sizes): that rank scans the
  //    pattern again with room (later scans reused the per-tile scratch) and the buffer
  //    keeps the size, so a steady workload pays this once.
  for (uint32_t i = 0; i < P; ++i) k->h_ballcnt[i] = k->b_cap[i];
  for (int round = 0;; ++round) {
    RK_CUDA(cudaMemcpy2DAsync(k->d_bcnt + 3, 4 * sizeof(unsigned long long), k->h_ballcnt,
                              sizeof(unsigned long long), sizeof(unsigned long long), P,
                              cudaMemcpyHostToDevice, s));
    RK_NCCL(api.AllGather(k->d_bcnt, k->d_ballcnt, 4ull * P, ncclUint64, k->comm, s));
    RK_CUDA(cudaMemcpyAsync(k->h_ballcnt, k->d_ballcnt,
                            4ull * P * k->nranks * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    RK_CUDA(cudaStreamSynchronize(s));
    bool again = false;
    for (int r = 0; r < k->nranks; ++r)
      for (uint32_t i = 0; i < P; ++i) {
        const unsigned long long* cr = k->h_ballcnt + 4ull * P * r + 4ull * i;
        again |= cr[0] > cr[3];
      }
    if (!again) break;
    if (round > 0) return fail(RK_ECUDA, "sharded batch: local offsets overflowed twice");
    std::vector<uint64_t> need(P);
    for (uint32_t i = 0; i < P; ++i) need[i] = k->h_ballcnt[4ull * P * k->rank + 4ull * i];
    for (uint32_t i = 0; i < P; ++i) {
      if (need[i] <= k->b_cap[i]) continue;
      if (int r = grow(&k->b_local[i], &k->b_cap[i], need[i], false, s)) return r;
      if (int r = local_scan(i)) return r;
    }
    for (uint32_t i = 0; i < P; ++i) k->h_ballcnt[i] = k->b_cap[i];
  }
  // 3. allgather-v of every pattern's offsets, one NCCL group for all of them (every rank
  //    takes part in every broadcast; a pattern whose list does not fit this rank's cap is
  //    received into scratch and not written)
  std::vector<uint64_t> total(P, 0);
  uint64_t spill = 0;
  for (uint32_t i = 0; i < P; ++i) {
    uint64_t hits = 0, coll = 0;
    for (int r = 0; r < k->nranks; ++r) {
      const unsigned long long* cr = k->h_ballcnt + 4ull * P * r + 4ull * i;
      total[i] += cr[0];
      hits += cr[1];
      coll += cr[2];
    }
    matches[i] = total[i];
    hash_hits[i] = hits;
    collisions[i] = coll;
    if (total[i] > caps[i]) spill += total[i];
  }
  if (spill > k->gather_cap) {
    RK_CUDA(cudaStreamSynchronize(s));
    cudaFree(k->d_gather);
    k->d_gather = nullptr;
    k->gather_cap = 0;
    RK_CUDA(cudaMalloc(&k->d_gather, spill * sizeof(int64_t)));
    k->gather_cap = spill;
  }
  k->gathered = 0;
  RK_NCCL(api.GroupStart());
  uint64_t at = 0;
  for (uint32_t i = 0; i < P; ++i) {
    int64_t* recv = d_outs[i];
    if (total[i] > caps[i]) {
      recv = k->d_gather + at;
      at += total[i];
    }
    uint64_t prefix = 0;
    for (int r = 0; r < k->nranks; ++r) {
      const uint64_t cnt = k->h_ballcnt[4ull * P * r + 4ull * i];
      if (cnt) {
        const bool me = r == k->rank;
        ncclResult_t e = api.Broadcast(me ? (const void*)k->b_local[i] : (const void*)(recv + prefix),
                                       recv + prefix, cnt, ncclInt64, r, k->comm, s);
        if (e != ncclSuccess) {
          api.GroupEnd();
          return fail(RK_ENCCL, "ncclBroadcast failed: %s", api.GetErrorString(e));
        }
      }
      prefix += cnt;
    }
  }
  RK_NCCL(api.GroupEnd());
  return RK_OK;
}

int rk_scan_sharded_batch_async(rk_comm_t* k, const uint8_t* d_text, uint64_t len,
                                uint64_t byte_lo, const uint8_t* h_patterns,
                                const uint32_t* h_lengths, const uint64_t* h_hashes, uint32_t P,
                                const uint64_t* win_lo, const uint64_t* win_hi,
                                int64_t* const* d_outs, const uint64_t* caps, uint64_t slab,
                                uint64_t* d_counts, void* stream) {
  if (!k) return fail(RK_EINVAL, "communicator is NULL");
  if (P < 1 || P > RK_BATCH_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_BATCH_MAX_PATTERNS);
  if (!h_patterns || !h_lengths || !h_hashes || !win_lo || !win_hi || !d_outs || !caps ||
      !d_counts)
    return fail(RK_EINVAL, "NULL argument array");
  if (slab < 1) return fail(RK_EINVAL, "slab must hold at least one offset");
  uint64_t off = 0;
  std::vector<uint64_t> pat_off(P);
  SlabOuts o{};
  for (uint32_t i = 0; i < P; ++i) {
    const uint32_t m = h_lengths[i];
    if (m < 1) return fail(RK_EINVAL, "pattern %u is empty", i);
    pat_off[i] = off;
    off += m;
    if (win_hi[i] > win_lo[i]) {
      if (win_lo[i] < byte_lo || win_hi[i] - byte_lo + m - 1 > len)
        return fail(RK_EINVAL, "pattern %u: windows [%llu, %llu) need bytes the shard does not "
                    "hold", i, (unsigned long long)win_lo[i], (unsigned long long)win_hi[i]);
      if (!d_text) return fail(RK_EINVAL, "text pointer is NULL");
    }
    if (caps[i] && !d_outs[i]) return fail(RK_EINVAL, "pattern %u: NULL output", i);
    o.out[i] = d_outs[i];
    o.cap[i] = caps[i];
  }
  rk_ctx* c = k->ctx;
  NcclApi& api = nccl();
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (d_text && len && !is_device_pointer(d_text, c->device))
    return fail(RK_EINVAL, "rk_scan_sharded_batch_async takes device texts of the context's device");
  if (int r = enter(c, s)) return r;
  if (!k->a_cnt) {
    RK_CUDA(cudaMalloc(&k->a_cnt, 4ull * RK_BATCH_MAX_PATTERNS * sizeof(unsigned long long)));
    RK_CUDA(cudaMalloc(&k->a_allcnt,
                       4ull * RK_BATCH_MAX_PATTERNS * k->nranks * sizeof(unsigned long long)));
  }
  if (int r = grow(&k->a_local, &k->a_local_cap, (uint64_t)P * slab, false, s)) return r;
  if (int r = grow(&k->a_all, &k->a_all_cap, (uint64_t)P * slab * k->nranks, false, s)) return r;
  // 1. the local scans, each emitting its ordered offsets into its slab
  for (uint32_t i = 0; i < P; ++i) {
    const uint32_t m = h_lengths[i];
    const uint64_t start = win_hi[i] > win_lo[i] ? win_lo[i] - byte_lo : 0;
    const uint64_t stop = win_hi[i] > win_lo[i] ? win_hi[i] - byte_lo : 0;
    if (int r = enqueue_scan(c, d_text, len, h_patterns + pat_off[i], m, h_hashes[i], start, stop,
                             k->a_local + (uint64_t)i * slab, slab, (int64_t)byte_lo, s,
                             (uint64_t*)(k->a_cnt + 4ull * i)))
      return r;
  }
  // 2. one NCCL group: every rank's counters and slabs to every rank (fixed sizes, so no
  //    host read between the scans and the exchange)
  RK_NCCL(api.GroupStart());
  ncclResult_t e = api.AllGather(k->a_cnt, k->a_allcnt, 4ull * P, ncclUint64, k->comm, s);
  if (e == ncclSuccess)
    e = api.AllGather(k->a_local, k->a_all, (uint64_t)P * slab, ncclInt64, k->comm, s);
  if (e != ncclSuccess) {
    api.GroupEnd();
    return fail(RK_ENCCL, "ncclAllGather failed: %s", api.GetErrorString(e));
  }
  RK_NCCL(api.GroupEnd());
  // 3. the global ordered lists, and the totals, on the device
  slab_compact_kernel<<<dim3(P, (unsigned)k->nranks), 256, 0, s>>>(
      k->a_all, k->a_allcnt, P, slab, k->nranks, o, (unsigned long long*)d_counts);
  RK_CUDA(cudaGetLastError());
  ++c->launches;
  return RK_OK;
}

int rk_multi_scan_sharded(rk_comm_t* k, const uint8_t* d_text, uint64_t len, uint64_t byte_lo,
                          uint64_t n_total, const uint8_t* h_patterns, const uint32_t* h_lengths,
                          uint32_t P, const uint64_t* h_hashes, uint64_t start_lo,
                          uint64_t start_hi, int64_t* d_off, uint32_t* d_idx, uint64_t cap,
                          uint64_t* pairs, void* stream) {
  if (!k || !pairs) return fail(RK_EINVAL, "communicator or pairs is NULL");
  *pairs = 0;
  if (P < 1 || P > RK_MULTI_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_MULTI_MAX_PATTERNS);
  if (!h_patterns || !h_lengths || !h_hashes) return fail(RK_EINVAL, "NULL pattern arrays");
  uint64_t max_len = 0;
  for (uint32_t i = 0; i < P; ++i) {
    if (h_lengths[i] < 1) return fail(RK_EINVAL, "pattern %u is empty", i);
    max_len = std::max<uint64_t>(max_len, h_lengths[i]);
  }
  if (byte_lo + len > n_total) return fail(RK_EINVAL, "shard beyond the text");
  if (start_hi > start_lo) {
    // every window starting in the range must fit in the held bytes (the halo) unless the
    // shard ends the text
    if (start_lo < byte_lo || (start_hi - byte_lo + max_len - 1 > len && byte_lo + len < n_total))
      return fail(RK_EINVAL, "starts [%llu, %llu) with patterns up to %llu bytes need bytes the "
                  "shard [%llu, %llu) does not hold", (unsigned long long)start_lo,
                  (unsigned long long)start_hi, (unsigned long long)max_len,
                  (unsigned long long)byte_lo, (unsigned long long)(byte_lo + len));
    if (!d_text) return fail(RK_EINVAL, "text pointer is NULL");
  }
  if (cap && (!d_off || !d_idx)) return fail(RK_EINVAL, "NULL output with cap > 0");
  rk_ctx* c = k->ctx;
  NcclApi& api = nccl();
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(c, s)) return r;

  // 1. this rank's pairs (global offsets), every start of [start_lo, start_hi) reported once
  uint64_t local = 0;
  if (k->m_cap < (1ull << 16)) {
    cudaFree(k->d_moff);
    cudaFree(k->d_midx);
    k->d_moff = nullptr;
    k->d_midx = nullptr;
    RK_CUDA(cudaMalloc(&k->d_moff, (1ull << 16) * sizeof(int64_t)));
    RK_CUDA(cudaMalloc(&k->d_midx, (1ull << 16) * sizeof(uint32_t)));
    k->m_cap = 1ull << 16;
  }
  const bool any = start_hi > start_lo && len > 0;
  if (any) {
    if (int r = multi_plan(c, h_patterns, h_lengths, P, h_hashes, s)) return r;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (int r = multi_enqueue(c, d_text, len, start_lo - byte_lo, start_hi - byte_lo,
                                (int64_t)byte_lo, k->d_moff, k->d_midx, k->m_cap, s))
        return r;
      RK_CUDA(cudaMemcpyAsync(c->h_mresult, c->d_mcount, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
      RK_CUDA(cudaStreamSynchronize(s));
      local = c->h_mresult[0];
      if (local <= k->m_cap) break;
      // more pairs than the buffer held: again with exact room (the sweep appends
      // unordered, so nothing beyond the buffer was kept)
      RK_CUDA(cudaFree(k->d_moff));
      RK_CUDA(cudaFree(k->d_midx));
      k->d_moff = nullptr;
      k->d_midx = nullptr;
      RK_CUDA(cudaMalloc(&k->d_moff, local * sizeof(int64_t)));
      RK_CUDA(cudaMalloc(&k->d_midx, local * sizeof(uint32_t)));
      k->m_cap = local;
    }
  }

  // 2. every rank's pair count, then the pairs themselves (allgather-v, offsets and indices)
  k->h_allcnt[4 * k->rank] = local;  // (scratch) this rank's count to the device slot
  RK_CUDA(cudaMemcpyAsync(k->d_cnt, &k->h_allcnt[4 * k->rank], sizeof(unsigned long long),
                          cudaMemcpyHostToDevice, s));
  RK_NCCL(api.AllGather(k->d_cnt, k->d_allcnt, 4, ncclUint64, k->comm, s));
  RK_CUDA(cudaMemcpyAsync(k->h_allcnt, k->d_allcnt, 4ull * k->nranks * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaStreamSynchronize(s));
  std::vector<uint64_t> cnt(k->nranks), prefix(k->nranks + 1, 0);
  for (int r = 0; r < k->nranks; ++r) {
    cnt[r] = k->h_allcnt[4 * r];
    prefix[r + 1] = prefix[r] + cnt[r];
  }
  const uint64_t total = prefix[k->nranks];
  *pairs = total;
  if (!total) return RK_OK;
  int64_t* goff = d_off;
  uint32_t* gidx = d_idx;
  if (cap < total) {
    if (k->g_cap < total) {
      RK_CUDA(cudaStreamSynchronize(s));
      cudaFree(k->d_goff);
      cudaFree(k->d_gidx);
      k->d_goff = nullptr;
      k->d_gidx = nullptr;
      RK_CUDA(cudaMalloc(&k->d_goff, total * sizeof(int64_t)));
      RK_CUDA(cudaMalloc(&k->d_gidx, total * sizeof(uint32_t)));
      k->g_cap = total;
    }
    goff = k->d_goff;
    gidx = k->d_gidx;
  }
  RK_NCCL(api.GroupStart());
  for (int r = 0; r < k->nranks; ++r) {
    if (!cnt[r]) continue;
    const bool me = r == k->rank;
    ncclResult_t e = api.Broadcast(me ? (const void*)k->d_moff : (const void*)(goff + prefix[r]),
                                   goff + prefix[r], cnt[r], ncclInt64, r, k->comm, s);
    if (e == ncclSuccess)
      e = api.Broadcast(me ? (const void*)k->d_midx : (const void*)(gidx + prefix[r]),
                        gidx + prefix[r], cnt[r], ncclUint32, r, k->comm, s);
    if (e != ncclSuccess) {
      api.GroupEnd();
      return fail(RK_ENCCL, "ncclBroadcast(root %d) failed: %s", r, api.GetErrorString(e));
    }
  }
  RK_NCCL(api.GroupEnd());
  // 3. (pattern index, offset) order over all ranks -- the reference's per-pattern lists
  if (int r = order_pairs(c, goff, gidx, total, n_total, P, s)) return r;
  if (goff != d_off && cap) {
    RK_CUDA(cudaMemcpyAsync(d_off, goff, cap * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    RK_CUDA(cudaMemcpyAsync(d_idx, gidx, cap * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  }
  return RK_OK;
}

int rk_comm_fetch(rk_comm_t* k, int64_t* d_out, uint64_t first, uint64_t count, void* stream) {
  if (!k) return fail(RK_EINVAL, "communicator is NULL");
  std::lock_guard<std::mutex> lk(k->ctx->mu);
  if (first > k->gathered || count > k->gathered - first)
    return fail(RK_EINVAL, "fetch [%llu, %llu) beyond the %llu offsets kept from the last "
                "sharded scan", (unsigned long long)first, (unsigned long long)(first + count),
                (unsigned long long)k->gathered);
  if (!count) return RK_OK;
  if (!d_out) return fail(RK_EINVAL, "NULL output");
  DeviceGuard g(k->ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(k->ctx, s)) return r;
  RK_CUDA(cudaMemcpyAsync(d_out, k->d_gather + first, count * sizeof(int64_t),
                          cudaMemcpyDeviceToDevice, s));
  return RK_OK;
}

}  // extern "C"
