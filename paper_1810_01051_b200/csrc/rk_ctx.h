// rk_ctx.h -- the scan context (struct rk_ctx of include/rkb200.h) and the host-side
// helpers shared by the C-ABI translation units (rk_capi.cu: scans, staging, multi-pattern;
// rk_comm.cu: NCCL communicators and the sharded scan).
#pragma once
#ifdef RK_HOST_PROFILE
#include <chrono>
#include <cstdio>
#endif
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/rkb200.h"
#include "rk_internal.h"

namespace rkb {

// Records the calling thread's error message (rk_last_error) and returns code.
int fail(int code, const char* fmt, ...);

#define RK_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return ::rkb::fail(RK_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                           \
  } while (0)

#ifdef RK_HOST_PROFILE
struct HostProf {
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit HostProf(const char* n) : name(n) {}
  ~HostProf();
};
#define RK_HPROF(n) HostProf _hp_##__LINE__(n)
#else
#define RK_HPROF(n)
#endif
struct DeviceGuard {  // (no cudaSetDevice when the caller is already on the device)
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = prev == dev || cudaSetDevice(dev) == cudaSuccess;
    if (prev == dev) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

constexpr uint64_t kStageChunk = 64ull << 20;  // host staging granularity (multiple of kTile)
#ifndef RK_RING_SLOTS
#define RK_RING_SLOTS 4
#define RK_RING_SLOT_MB 16
#endif
constexpr int kRing = RK_RING_SLOTS;                       // pinned staging slots (pageable texts)
constexpr uint64_t kRingSlot = (uint64_t)RK_RING_SLOT_MB << 20;  // bytes per pinned slot

class CopyPool;  // pageable -> pinned copy threads (rk_capi.cu)

}  // namespace rkb

using rkb::CopyPool;

// A pattern set's device layout (offsets into the context's blob) and its sweeps.
namespace rkb {
struct MultiPlan {
  struct Group {
    uint32_t m, P, tsize;
    uint64_t pats, phash, order, gidx, table, filter;
  };
  struct Sweep {
    std::vector<uint32_t> groups;  // ascending lengths
    uint32_t qmode = 0, qwords = 0;
    uint32_t qf32 = 0;     // q-gram filter of 32-bit words (several lengths) or 64-bit blocks
    uint64_t qfilter = 0;  // blob offset of the sweep's q-gram filter (qmode > 0)
    uint64_t qmap = 0;     // blob offset of its q-gram -> group-mask table
    uint32_t qmap_size = 0;
    // short sweeps (qmode == 0, lengths < 7): cuckoo table + filter, anchored q-gram length
    uint64_t stab = 0;
    TinyHash th{};
    uint32_t sq = 0;
  };
  std::vector<uint8_t> key;  // P, lengths, hashes, pattern bytes
  std::vector<Group> groups;
  std::vector<Sweep> sweeps;
};
}  // namespace rkb
using rkb::MultiPlan;

struct rk_ctx {
  int device = 0;
  int num_sms = 0;
  // Two alternating "sets" of {counters[4], block_sums[block_sums_cap]}: a scan uses
  // the current set, and its emit kernel zeroes the other one for the next scan, so a
  // scan is exactly two kernel launches (no memsets).  counters: [0] matches,
  // [1] hash_hits, [2] collisions.
  unsigned long long* d_sets = nullptr;
  unsigned long long* d_counters = nullptr;  // counters of the current set
  int cur_set = 0;
  unsigned long long* d_mcount = nullptr;    // multi-pattern pair counter
  unsigned long long* h_counters = nullptr;  // pinned mirror
  unsigned long long* d_emit_work = nullptr;  // the emit's dense-tile queue (rk_emit.cu)
  unsigned long long* d_queue = nullptr;
  uint64_t queue_cap = 0;
  uint32_t* d_tile_info = nullptr;  // per tile: matches | chunk bitmap << 16
  uint64_t tile_info_cap = 0;
  uint32_t* d_masks = nullptr;      // per tile: kTileChunks x 32 lane hit masks
  uint64_t masks_cap = 0;
  unsigned long long* d_block_sums = nullptr;  // block sums of the current set
  uint64_t block_sums_cap = 0;
  uint8_t* d_pattern = nullptr;  // pattern of the current scan (points into a cache slot)
  struct PatSlot {
    std::vector<uint8_t> bytes;
    uint8_t* d = nullptr;
    uint64_t cap = 0;
    uint8_t* h = nullptr;  // pinned source of the slot's upload (rewritten after a sync only)
    uint64_t hcap = 0;
    uint64_t last_use = 0;
  };
  std::vector<PatSlot> pat_cache = std::vector<PatSlot>(64);
  uint64_t pat_clock = 0;
  uint64_t launches = 0;
  // host staging
  uint8_t* d_stage = nullptr;
  uint64_t stage_cap = 0;
  uint8_t* h_ring[rkb::kRing] = {};
  CopyPool* copier = nullptr;  // created on the first pageable host scan
  int64_t* d_out_stage = nullptr;
  uint64_t out_stage_cap = 0;
  uint64_t host_last = 0;  // offsets held in d_out_stage by the last rk_scan_host
  cudaStream_t s_copy = nullptr, s_comp = nullptr;
  cudaEvent_t ev_copied[rkb::kRing] = {};  // ring slot free again
  cudaEvent_t ev_ready = nullptr;                 // bytes of the current chunk landed
  // multi-pattern tables
  uint8_t* d_sort = nullptr;   // scratch of the device pair sort
  uint64_t sort_cap = 0;
  uint8_t* d_mblob = nullptr;  // every length group's patterns, hashes and tables
  uint64_t mblob_cap = 0;
  uint8_t* h_mstage = nullptr;  // pinned staging of the blob
  uint64_t h_mstage_cap = 0;
  unsigned long long* h_mresult = nullptr;  // pinned (mapped): a multi scan's pair count
  MultiPlan mplan;              // the last pattern set's plan (cache key + layout)
  // The scratch above is ordered on the stream of the call that used it.  When a call
  // arrives on another stream, that stream first waits for everything queued so far on
  // the previous one (an event recorded lazily at the switch: an event between two
  // launches on one stream would cost their programmatic-dependent-launch overlap).
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  cudaEvent_t ev_switch = nullptr;
  // the last device scan's emission (rk_scan / rk_scan_async), for rk_scan_fetch
  struct LastScan {
    bool valid = false;
    bool host = false;  // staged host text (rk_scan_host): offsets into d_out_stage
    uint64_t tiles = 0, tile0 = 0;
    int64_t start_bias = 0;
  } last_scan;
  // rk_scan_host_batch: per-pattern per-tile results, counter sets and output segments of
  // the last batch (all live at once, so any pattern can be re-emitted after the counts
  // are known)
  uint32_t* d_binfo = nullptr;
  uint64_t binfo_cap = 0;
  uint32_t* d_bmasks = nullptr;
  uint64_t bmasks_cap = 0;
  int64_t* d_bspill = nullptr;  // offsets of patterns that overflowed their slot
  uint64_t bspill_cap = 0;
  unsigned long long* d_bsets = nullptr;
  uint64_t bsets_cap = 0;
  unsigned long long* h_bcounts = nullptr;  // pinned, mapped: {matches, hash_hits, collisions, 0} x P
  uint32_t h_bcounts_cap = 0;
  struct BatchSeg {
    const int64_t* d;  // the pattern's ordered offsets on the device
    uint64_t count;
  };
  std::vector<BatchSeg> batch_segs;  // the last host scan's offsets, in order (rk_scan_host_fetch)
  std::mutex mu;
};


namespace rkb {

template <class T>
int grow(T** p, uint64_t* cap, uint64_t need, bool zero, cudaStream_t s) {
  if (*cap >= need && *p) return RK_OK;
  if (*p) {
    RK_CUDA(cudaStreamSynchronize(s));
    RK_CUDA(cudaFree(*p));
    *p = nullptr;
  }
  uint64_t c = need > 64 ? need : 64;
  RK_CUDA(cudaMalloc((void**)p, c * sizeof(T)));
  if (zero) RK_CUDA(cudaMemsetAsync(*p, 0, c * sizeof(T), s));
  *cap = c;
  return RK_OK;
}

int enter(rk_ctx* c, cudaStream_t s);
int check_scan_args(const uint8_t* text, uint64_t n, const uint8_t* h_pattern, uint32_t m,
                    uint64_t start, uint64_t stop, const void* out, uint64_t cap);
int enqueue_scan(rk_ctx* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                 uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out,
                 uint64_t cap, int64_t bias, cudaStream_t s, uint64_t* d_counts = nullptr);
int emit_last(rk_ctx* c, int64_t* d_out, uint64_t cap, cudaStream_t s);
int host_scan_enqueue(rk_ctx* c, const uint8_t* h_text, uint64_t n, const uint8_t* h_pattern,
                      uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t bias,
                      uint64_t* d_counts);
bool is_device_pointer(const void* p, int device);
int multi_plan(rk_ctx* c, const uint8_t* h_patterns, const uint32_t* h_lengths, uint32_t P,
               const uint64_t* h_hashes, cudaStream_t s);
int multi_enqueue(rk_ctx* c, const uint8_t* d_text, uint64_t n, uint64_t start_lo,
                  uint64_t start_hi, int64_t bias, int64_t* d_off, uint32_t* d_idx,
                  uint64_t cap, cudaStream_t s);
int multi_order(rk_ctx* c, int64_t* d_off, uint32_t* d_idx, uint64_t cap, uint64_t n, uint32_t P,
                const unsigned long long* d_count, uint64_t* total_out, cudaStream_t s);
int order_pairs(rk_ctx* c, int64_t* d_off, uint32_t* d_idx, uint64_t k, uint64_t n, uint32_t P,
                cudaStream_t s);

}  // namespace rkb
