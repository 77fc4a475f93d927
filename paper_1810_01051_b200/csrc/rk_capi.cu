#ifdef RK_HOST_PROFILE
#include <map>
#include <string>
#endif
// rk_capi.cu -- the C ABI (include/rkb200.h): contexts, argument checking, launch
// planning for the ordered single-pattern scan, the host-text staging pipeline, the
// multi-pattern table build, and error reporting.
#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/rkb200.h"
#include "rk_ctx.h"

using namespace rkb;

namespace {
thread_local std::string g_err;
}  // namespace

int rkb::fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#ifdef RK_HOST_PROFILE
static std::map<std::string, std::pair<double, long>>& hprof_map() {
  static std::map<std::string, std::pair<double, long>> m;
  static bool reg = false;
  if (!reg) {
    reg = true;
    atexit([] {
      for (auto& kv : hprof_map())
        fprintf(stderr, "hprof %-24s %8.2f us avg over %ld\n", kv.first.c_str(),
                kv.second.first / kv.second.second, kv.second.second);
    });
  }
  return m;
}
HostProf::~HostProf() {
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  auto& e = hprof_map()[name];
  e.first += us;
  e.second += 1;
}
#endif
namespace rkb {

// Persistent host threads for the pageable -> pinned staging copy (CPU-bound: one
// thread moves ~10-14 GB/s, the DMA ~55 GB/s).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    n_ = std::min(16u, hw);  // (C2 text, 16-core box: 8 threads 31 GB/s, 12-16 42-45)
    if (const char* e = getenv("RKB200_COPY_THREADS")) n_ = std::max(1, atoi(e));
    for (unsigned i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(uint8_t* dst, const uint8_t* src, uint64_t len) {
    if (n_ <= 1 || len < (4u << 20)) {
      memcpy(dst, src, len);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = dst;
      src_ = src;
      len_ = len;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void part(unsigned i) {
    const uint64_t per = (len_ + n_ - 1) / n_;
    const uint64_t a = std::min(len_, i * per), b = std::min(len_, a + per);
    if (a < b) memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      part(i);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  unsigned n_ = 1;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  unsigned pending_ = 0;
  bool stop_ = false;
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  uint64_t len_ = 0;
};

}  // namespace rkb

namespace rkb {

PatWords pack_pattern(const uint8_t* h, uint32_t m) {
  PatWords pw{};
  for (uint32_t i = 0; i < m && i < 32; ++i) pw.w[i >> 2] |= (uint32_t)h[i] << (8 * (i & 3));
  return pw;
}

RollConsts roll_consts(uint32_t m) {
  RollConsts K;
  K.k2 = 2;
  K.k8 = 8;
  K.k16 = 16;
  K.negpow = m < 32 ? (uint32_t)(0u - (1u << m)) : 0u;
  return K;
}

// Geometry of one scan of windows [start, stop) over text at d_text.
struct Geometry {
  const uint8_t* abase;
  uint64_t amis, ja_lo, ja_hi, tile_first, num_tiles;
};

Geometry geometry(const uint8_t* d_text, uint32_t m, uint64_t start, uint64_t stop) {
  Geometry g;
  const uintptr_t p = (uintptr_t)d_text;
  g.abase = (const uint8_t*)(p & ~(uintptr_t)31);
  g.amis = p - (uintptr_t)g.abase;
  g.ja_lo = start + m - 1 + g.amis;
  g.ja_hi = stop + m - 1 + g.amis;
  g.tile_first = g.ja_lo / kTile;
  g.num_tiles = (g.ja_hi - 1) / kTile - g.tile_first + 1;
  return g;
}

uint64_t set_words(const rk_ctx* c) { return 4 + c->block_sums_cap; }

void select_set(rk_ctx* c, int k) {
  c->cur_set = k;
  c->d_counters = c->d_sets + (uint64_t)k * set_words(c);
  c->d_block_sums = c->d_counters + 4;
}

// Orders a call on stream s after all earlier work of the context (see rk_ctx::ev_switch).
int enter(rk_ctx* c, cudaStream_t s) {
  if (c->has_last && c->last_stream != s) {
    RK_CUDA(cudaEventRecord(c->ev_switch, c->last_stream));
    RK_CUDA(cudaStreamWaitEvent(s, c->ev_switch, 0));
  }
  c->last_stream = s;
  c->has_last = true;
  return RK_OK;
}

// Starts a logical scan of `tiles` tiles: per-tile buffers sized, and the next counter
// set selected (it was zeroed by the previous scan's emit, or on allocation).
int begin_scan(rk_ctx* c, uint64_t tiles, cudaStream_t s) {
  if (int r = grow(&c->d_tile_info, &c->tile_info_cap, tiles, false, s)) return r;
  if (int r = grow(&c->d_masks, &c->masks_cap, tiles * (uint64_t)(kTileChunks * 32), false, s))
    return r;
  const uint64_t nb = (tiles + kEmitTiles - 1) / kEmitTiles;
  if (!c->d_sets || c->block_sums_cap < nb) {
    if (c->d_sets) {
      RK_CUDA(cudaStreamSynchronize(s));
      RK_CUDA(cudaFree(c->d_sets));
    }
    c->block_sums_cap = std::max<uint64_t>(nb, 1024);
    RK_CUDA(cudaMalloc(&c->d_sets, 2 * set_words(c) * sizeof(unsigned long long)));
    RK_CUDA(cudaMemsetAsync(c->d_sets, 0, 2 * set_words(c) * sizeof(unsigned long long), s));
  }
  select_set(c, c->cur_set ^ 1);
  return RK_OK;
}

// Orders the offsets of a logical scan whose tiles are sequence numbers [0, tiles)
// starting at a-space tile `tile0`; copies {matches, hash_hits, collisions} to d_counts
// if given, and zeroes the other counter set for the next scan.
// Per-logical-scan device state.  Normally the context's (one scan at a time, counter
// sets alternating); a batch of scans over one staged text keeps one of these per
// pattern, so every pattern's results stay live until its offsets are emitted.
struct ScanScratch {
  unsigned long long* counters;    // [0] matches, [1] hash_hits, [2] collisions
  unsigned long long* block_sums;
  uint32_t* tile_info;
  uint32_t* masks;
  const uint8_t* pattern;          // device copy of the pattern
};

int emit(rk_ctx* c, uint64_t tiles, uint64_t tile0, int64_t start_bias, int64_t* d_out,
         uint64_t cap, cudaStream_t s, uint64_t* d_counts = nullptr,
         uint32_t* d_bitmap = nullptr, int64_t bit_bias = 0,
         const ScanScratch* x = nullptr) {
  EmitArgs e;
  e.tile_info = x ? x->tile_info : c->d_tile_info;
  e.masks = x ? x->masks : c->d_masks;
  e.block_sums = x ? x->block_sums : c->d_block_sums;
  e.num_tiles = tiles;
  e.tile0 = tile0;
  e.start_bias = start_bias;
  e.out = d_out;
  e.cap = d_out ? cap : 0;
  e.counters = x ? x->counters : c->d_counters;
  e.counts_out = (unsigned long long*)d_counts;
  // (a batch's counters are zeroed once, up front: nothing to clear for the next scan)
  e.clear = x ? nullptr : c->d_sets + (uint64_t)(c->cur_set ^ 1) * set_words(c);
  e.clear_words = x ? 0 : set_words(c);
  e.bitmap = nullptr;
  e.bit_bias = 0;
  e.work = nullptr;
  e.queue = nullptr;
  e.defer_min = 0;
  if (!d_bitmap && d_out && cap) {
    // the dense-tile queue: zeroed once, left zeroed by every emit
    uint64_t wcap = 0;
    if (!c->d_emit_work) {
      if (int r = grow(&c->d_emit_work, &wcap, 4, true, s)) return r;
    }
    if (int r = grow(&c->d_queue, &c->queue_cap, tiles, true, s)) return r;
    e.work = c->d_emit_work;
    e.queue = c->d_queue;
  }
  if (d_bitmap) {
    e.bitmap = d_bitmap;
    e.bit_bias = bit_bias;
  }
  {
    RK_HPROF("launch_emit");
    RK_CUDA(launch_emit(e, c->num_sms, s));
  }
  ++c->launches;
  return RK_OK;
}

// Counters of a scan with no windows (or an unreachable hash): zeros.
int zero_result(rk_ctx* c, uint64_t* d_counts, cudaStream_t s) {
  if (!c->d_sets) {
    if (int r = begin_scan(c, 1, s)) return r;
  }
  RK_CUDA(cudaMemsetAsync(c->d_counters, 0, 4 * sizeof(unsigned long long), s));
  if (d_counts) RK_CUDA(cudaMemsetAsync(d_counts, 0, 3 * sizeof(uint64_t), s));
  return RK_OK;
}

TextGeom text_geom(const Geometry& g, uint64_t n, uint32_t m, uint64_t seq_base) {
  TextGeom t;
  t.abase = g.abase;
  t.amis = g.amis;
  t.n = n;
  t.ja_lo = g.ja_lo;
  t.ja_hi = g.ja_hi;
  t.tile0 = g.tile_first;
  t.num_tiles = g.num_tiles;
  t.seq_base = seq_base;
  t.m = m;
  t.K = roll_consts(m);
  return t;
}

// Persistent grid: every SM full, never more warps than tiles.
int grid_for(uint64_t tiles, int num_sms, int blocks_per_sm, int warps_per_block) {
  const uint64_t max_grid = (uint64_t)num_sms * (uint64_t)blocks_per_sm;
  const uint64_t want = (tiles + warps_per_block - 1) / warps_per_block;
  return (int)std::max<uint64_t>(1, std::min(max_grid, want));
}

int launch_one(rk_ctx* c, const uint8_t* d_text, uint64_t n, uint32_t m, uint64_t hx,
               uint64_t start, uint64_t stop, uint64_t seq_base, const PatWords& pw, cudaStream_t s,
               const ScanScratch* x = nullptr) {
  const Geometry g = geometry(d_text, m, start, stop);
  ScanArgs a{};
  a.g = text_geom(g, n, m, seq_base);
  a.pattern = x ? x->pattern : c->d_pattern;
  a.hx = hx;
  a.counters = x ? x->counters : c->d_counters;
  a.block_sums = x ? x->block_sums : c->d_block_sums;
  a.tile_info = x ? x->tile_info : c->d_tile_info;
  a.masks = x ? x->masks : c->d_masks;
  a.pw = pw;
  {
    // is hx the pattern's own hash (the normal case)?  Then a window whose bytes equal the
    // pattern is a hash hit and a match (dense runs settle from the bytes alone)
    uint64_t h = 0;
    for (uint32_t i = 0; i < m && i < 32; ++i)
      h = (h << 1) + ((pw.w[i >> 2] >> (8 * (i & 3))) & 0xffu);
    a.hx_is_pattern = m <= 8 && h == hx;
  }
  // A scan with fewer tiles than the full grid has warps (e.g. C1, 1 MiB = 128 tiles
  // against 148 x 20 warps at m = 8) spreads them: every CTA slot gets ceil(tiles / slots)
  // warps, so a 1 MiB scan streams through ~128 SMs instead of 7 full CTAs.
  const uint64_t slots = (uint64_t)c->num_sms * (uint64_t)scan_blocks_per_sm(m);
  uint64_t warps = (uint64_t)scan_warps(m);
  if (g.num_tiles < slots * warps) warps = std::max<uint64_t>(1, (g.num_tiles + slots - 1) / slots);
  a.warps = (uint32_t)warps;
  RK_HPROF("launch_scan");
  RK_CUDA(launch_scan(a, grid_for(g.num_tiles, c->num_sms, scan_blocks_per_sm(m), (int)warps),
                      s));
  ++c->launches;
  return RK_OK;
}

int check_scan_args(const uint8_t* text, uint64_t n, const uint8_t* h_pattern, uint32_t m,
                    uint64_t start, uint64_t stop, const void* out, uint64_t cap) {
  if (!h_pattern || m < 1) return fail(RK_EINVAL, "pattern must be non-empty");
  if (stop > start) {
    if (!text) return fail(RK_EINVAL, "text pointer is NULL");
    if (stop + (uint64_t)m - 1 > n)
      return fail(RK_EINVAL, "window range [%llu, %llu) of length %u out of bounds for text of "
                  "length %llu", (unsigned long long)start, (unsigned long long)stop, m,
                  (unsigned long long)n);
    if (cap && !out) return fail(RK_EINVAL, "output pointer is NULL with cap > 0");
  }
  return RK_OK;
}

// m <= 24: every window hash is < 2^32, so a 64-bit hx >= 2^32 can never be hit.
bool hash_unreachable(uint32_t m, uint64_t hx) { return m <= 24 && (hx >> 32) != 0; }

// Device copy of the pattern from a small per-context cache (64 slots, LRU), so
// repeated scans with the same patterns -- a length sweep, a service loop -- issue no
// host-to-device copy and no synchronisation.  A slot is only overwritten after the
// stream has drained (the context's earlier work on other streams is ordered before s,
// see enter()), because an earlier kernel may still be reading it; the upload is an
// asynchronous copy on s from the slot's pinned buffer, so the scan is ordered after it.
int upload_pattern(rk_ctx* c, const uint8_t* h_pattern, uint32_t m, cudaStream_t s) {
  ++c->pat_clock;
  rk_ctx::PatSlot* victim = &c->pat_cache[0];
  for (auto& sl : c->pat_cache) {
    if (sl.d && sl.bytes.size() == m && memcmp(sl.bytes.data(), h_pattern, m) == 0) {
      sl.last_use = c->pat_clock;
      c->d_pattern = sl.d;
      return RK_OK;
    }
    if (sl.last_use < victim->last_use) victim = &sl;
  }
  RK_CUDA(cudaStreamSynchronize(s));
  if (int r = grow(&victim->d, &victim->cap, m, false, s)) return r;
  if (victim->hcap < m) {
    if (victim->h) RK_CUDA(cudaFreeHost(victim->h));
    victim->h = nullptr;
    victim->hcap = 0;
    RK_CUDA(cudaMallocHost(&victim->h, std::max<uint64_t>(m, 64)));
    victim->hcap = std::max<uint64_t>(m, 64);
  }
  victim->bytes.assign(h_pattern, h_pattern + m);
  victim->last_use = c->pat_clock;
  memcpy(victim->h, h_pattern, m);
  RK_CUDA(cudaMemcpyAsync(victim->d, victim->h, m, cudaMemcpyHostToDevice, s));
  c->d_pattern = victim->d;
  return RK_OK;
}

int enqueue_scan(rk_ctx* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                 uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out,
                 uint64_t cap, int64_t bias, cudaStream_t s, uint64_t* d_counts) {
  c->last_scan.valid = false;
  if (stop <= start || hash_unreachable(m, hx)) return zero_result(c, d_counts, s);
  {
    RK_HPROF("upload_pattern");
    if (int r = upload_pattern(c, h_pattern, m, s)) return r;
  }
  const Geometry g = geometry(d_text, m, start, stop);
  {
    RK_HPROF("begin_scan");
    if (int r = begin_scan(c, g.num_tiles, s)) return r;
  }
  {
    RK_HPROF("launch_one");
    if (int r = launch_one(c, d_text, n, m, hx, start, stop, 0, pack_pattern(h_pattern, m), s))
      return r;
  }
  RK_HPROF("emit");
  c->last_scan.valid = true;
  c->last_scan.host = false;
  c->last_scan.tiles = g.num_tiles;
  c->last_scan.tile0 = g.tile_first;
  c->last_scan.start_bias = bias - (int64_t)g.amis - (int64_t)m + 1;
  return emit(c, g.num_tiles, g.tile_first, c->last_scan.start_bias, d_out, cap, s, d_counts);
}

int read_counters(rk_ctx* c, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
                  cudaStream_t s) {
  RK_CUDA(cudaMemcpyAsync(c->h_counters, c->d_counters, 3 * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaStreamSynchronize(s));
  if (matches) *matches = c->h_counters[0];
  if (hash_hits) *hash_hits = c->h_counters[1];
  if (collisions) *collisions = c->h_counters[2];
  return RK_OK;
}

// Re-runs the ordered emission of the context's last scan (device or staged host text)
// into d_out with room for cap offsets: the scan's per-tile results and block sums are
// still in the current counter set (nothing rescans).
int emit_last(rk_ctx* c, int64_t* d_out, uint64_t cap, cudaStream_t s) {
  if (!c->last_scan.valid) return fail(RK_EINVAL, "no scan to re-emit");
  return emit(c, c->last_scan.tiles, c->last_scan.tile0, c->last_scan.start_bias, d_out, cap, s);
}

bool is_device_pointer(const void* p, int device) {
  cudaPointerAttributes attr;
  const bool dev = cudaPointerGetAttributes(&attr, p) == cudaSuccess &&
                   (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) &&
                   attr.device == device;
  cudaGetLastError();
  return dev;
}

// The staging pipeline of a HOST text (rk_scan_host, rk_scan_sharded): windows [start,
// stop) of h_text (n bytes) are scanned as their bytes land in HBM.  The bytes [start,
// stop + m - 1) go to c->d_stage in kStageChunk pieces by cudaMemcpyAsync on s_copy
// (pinned text: straight from it; pageable: through the pinned ring, filled by the copy
// threads), and the windows ending in each piece are scanned on s_comp as soon as it has
// landed, while the next piece is in flight.  The ordered offsets (+ bias) go to
// c->d_out_stage (first out_stage_cap of them; emit_last re-emits more), the counters
// to c->d_counters (and d_counts if given).  Enqueued only: the caller holds c->mu, has
// entered s_comp, and has sized d_out_stage.
int host_scan_enqueue(rk_ctx* c, const uint8_t* h_text, uint64_t n, const uint8_t* h_pattern,
                      uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t bias,
                      uint64_t* d_counts) {
  cudaStream_t sc = c->s_comp, sk = c->s_copy;
  c->last_scan.valid = false;
  if (stop <= start || hash_unreachable(m, hx)) return zero_result(c, d_counts, sc);
  // bytes the windows need: [start, stop + m - 1)
  const uint64_t b_lo = start, b_hi = stop + m - 1;
  if (int r = grow(&c->d_stage, &c->stage_cap, n, false, sc)) return r;
  if (int r = upload_pattern(c, h_pattern, m, sc)) return r;

  cudaPointerAttributes attr;
  const bool pinned = cudaPointerGetAttributes(&attr, h_text) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (!pinned && !c->h_ring[0]) {
    for (auto& h : c->h_ring) RK_CUDA(cudaMallocHost(&h, kRingSlot));
    c->copier = new CopyPool();
  }

  // The staging buffer is cudaMalloc'ed (256-byte aligned), so a-space == text index.
  const Geometry gall = geometry(c->d_stage, m, start, stop);
  if (int r = begin_scan(c, gall.num_tiles, sc)) return r;
  const PatWords pw = pack_pattern(h_pattern, m);

  // chunk k covers end positions [k*C, (k+1)*C) and needs bytes < (k+1)*C; its copy on
  // s_copy overlaps the scan of chunk k-1 on s_comp.
  const uint64_t ja_lo = gall.ja_lo, ja_hi = gall.ja_hi;
  const uint64_t k0 = ja_lo / kStageChunk, k1 = (ja_hi - 1) / kStageChunk;
  uint64_t copied = b_lo;  // bytes [b_lo, copied) are enqueued
  int slot = 0;
  for (uint64_t k = k0; k <= k1; ++k) {
    const uint64_t e_lo = std::max(ja_lo, k * kStageChunk);
    const uint64_t e_hi = std::min(ja_hi, (k + 1) * kStageChunk);
    const uint64_t need = std::min(b_hi, (k + 1) * kStageChunk);
    if (need > copied) {
      const uint64_t len = need - copied;
      if (pinned) {
        RK_CUDA(cudaMemcpyAsync(c->d_stage + copied, h_text + copied, len,
                                cudaMemcpyHostToDevice, sk));
      } else {
        // pageable: multi-threaded CPU copy into a pinned ring slot, then DMA; a slot
        // is reused only after the DMA issued from it kRing steps ago has finished
        for (uint64_t off = 0; off < len; off += kRingSlot) {
          const uint64_t l = std::min<uint64_t>(kRingSlot, len - off);
          RK_CUDA(cudaEventSynchronize(c->ev_copied[slot]));
          c->copier->copy(c->h_ring[slot], h_text + copied + off, l);
          RK_CUDA(cudaMemcpyAsync(c->d_stage + copied + off, c->h_ring[slot], l,
                                  cudaMemcpyHostToDevice, sk));
          RK_CUDA(cudaEventRecord(c->ev_copied[slot], sk));
          slot = (slot + 1) % kRing;
        }
      }
      copied = need;
      RK_CUDA(cudaEventRecord(c->ev_ready, sk));
      RK_CUDA(cudaStreamWaitEvent(sc, c->ev_ready, 0));
    }
    const uint64_t ws = e_lo - (m - 1), we = e_hi - (m - 1);  // windows ending in the chunk
    const Geometry gk = geometry(c->d_stage, m, ws, we);
    if (int r = launch_one(c, c->d_stage, n, m, hx, ws, we, gk.tile_first - gall.tile_first, pw,
                           sc))
      return r;
  }
  c->last_scan.valid = true;
  c->last_scan.host = true;
  c->last_scan.tiles = gall.num_tiles;
  c->last_scan.tile0 = gall.tile_first;
  c->last_scan.start_bias = bias - (int64_t)m + 1;  // staging buffer: a-space == text index
  return emit(c, gall.num_tiles, gall.tile_first, c->last_scan.start_bias, c->d_out_stage,
              c->out_stage_cap, sc, d_counts);
}

}  // namespace rkb

// Builds (or reuses) the device tables of a pattern set: every length group's patterns,
// hashes, key table and filter, plus one q-gram filter per sweep, in one device blob.
// The plan is cached per context: repeating a search with the same set uploads nothing.
int rkb::multi_plan(rk_ctx* c, const uint8_t* h_patterns, const uint32_t* h_lengths, uint32_t P,
               const uint64_t* h_hashes, cudaStream_t s) {
  std::vector<uint8_t> key(sizeof(uint32_t) + P * (sizeof(uint32_t) + sizeof(uint64_t)));
  uint64_t total = 0;
  for (uint32_t i = 0; i < P; ++i) total += h_lengths[i];
  memcpy(key.data(), &P, 4);
  memcpy(key.data() + 4, h_lengths, 4ull * P);
  memcpy(key.data() + 4 + 4ull * P, h_hashes, 8ull * P);
  key.insert(key.end(), h_patterns, h_patterns + total);
  if (c->d_mblob && key == c->mplan.key) return RK_OK;

  MultiPlan plan;
  std::vector<uint64_t> first_byte(P + 1, 0);
  for (uint32_t i = 0; i < P; ++i) first_byte[i + 1] = first_byte[i] + h_lengths[i];
  std::map<uint32_t, std::vector<uint32_t>> by_len;
  for (uint32_t i = 0; i < P; ++i) by_len[h_lengths[i]].push_back(i);

  std::vector<uint8_t> blob;
  auto reserve = [&blob](uint64_t bytes) {
    const uint64_t off = (blob.size() + 15) & ~(uint64_t)15;
    blob.resize(off + bytes, 0);
    return off;
  };
  for (const auto& [m, members] : by_len) {
    MultiPlan::Group b{};
    b.m = m;
    b.P = (uint32_t)members.size();
    std::vector<std::pair<uint32_t, uint32_t>> keyed(b.P);
    for (uint32_t i = 0; i < b.P; ++i) keyed[i] = {(uint32_t)h_hashes[members[i]], i};
    std::stable_sort(keyed.begin(), keyed.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    std::vector<uint32_t> order(b.P);
    std::vector<std::pair<uint32_t, uint32_t>> runs;  // (key, first << 13 | count)
    for (uint32_t i = 0; i < b.P;) {
      uint32_t j = i;
      while (j < b.P && keyed[j].first == keyed[i].first) {
        order[j] = keyed[j].second;
        ++j;
      }
      runs.push_back({keyed[i].first, (i << 13) | (j - i)});
      i = j;
    }
    b.tsize = 64;
    while (b.tsize < 2 * runs.size()) b.tsize <<= 1;
    b.pats = reserve((uint64_t)b.P * m);
    b.phash = reserve((uint64_t)b.P * sizeof(uint64_t));
    b.order = reserve((uint64_t)b.P * sizeof(uint32_t));
    b.gidx = reserve((uint64_t)b.P * sizeof(uint32_t));
    b.table = reserve((uint64_t)b.tsize * sizeof(uint2));
    b.filter = reserve(kMultiFilterWords * sizeof(uint32_t));
    uint8_t* base = blob.data();
    for (uint32_t i = 0; i < b.P; ++i) {
      memcpy(base + b.pats + (uint64_t)i * m, h_patterns + first_byte[members[i]], m);
      memcpy(base + b.phash + 8ull * i, &h_hashes[members[i]], 8);
      memcpy(base + b.gidx + 4ull * i, &members[i], 4);
    }
    memcpy(base + b.order, order.data(), 4ull * b.P);
    uint2* table = reinterpret_cast<uint2*>(base + b.table);
    uint32_t* filter = reinterpret_cast<uint32_t*>(base + b.filter);
    for (uint32_t t = 0; t < b.tsize; ++t) table[t] = make_uint2(0u, kMultiEmpty);
    for (const auto& r : runs) {
      uint32_t slot = (r.first * 0x9E3779B1u) & (b.tsize - 1);
      while (table[slot].y != kMultiEmpty) slot = (slot + 1) & (b.tsize - 1);
      table[slot] = make_uint2(r.first, r.second);
      const uint32_t bit = (r.first * 0x9E3779B1u) >> 16;
      filter[bit >> 5] |= 1u << (bit & 31);
    }
    plan.groups.push_back(b);
  }

  // sweeps: the lengths 4..6 of the set in one anchored short sweep, 1..3 in one
  // per-window short sweep, lengths >= 7 in runs of kMultiMaxGroups sharing one q-gram
  // filter
  size_t gi = 0;
  std::vector<uint32_t> short_sets[2];  // [0] lengths 1..3, [1] lengths 4..6
  for (; gi < plan.groups.size() && plan.groups[gi].m < 7; ++gi)
    short_sets[plan.groups[gi].m >= 4].push_back((uint32_t)gi);
  for (const auto& members : short_sets) {
    if (members.empty()) continue;
    MultiPlan::Sweep sw{};
    sw.groups = members;
    const uint32_t m_min = plan.groups[members.front()].m;
    sw.sq = m_min >= 4 ? (uint32_t)short_gram_q((int)m_min) : 0u;
    // every pattern of the sweep: (tagged key, caller index)
    struct Entry {
      uint32_t lo, hb, len, idx;
    };
    std::vector<Entry> es;
    for (uint32_t g : members) {
      const MultiPlan::Group& b = plan.groups[g];
      for (uint32_t i = 0; i < b.P; ++i) {
        Entry e{0, 0, b.m, 0};
        const uint8_t* pb = blob.data() + b.pats + (uint64_t)i * b.m;
        memcpy(&e.lo, pb, std::min<uint32_t>(b.m, 4));
        if (b.m > 4) memcpy(&e.hb, pb + 4, b.m - 4);
        memcpy(&e.idx, blob.data() + b.gidx + 4ull * i, 4);
        es.push_back(e);
      }
    }
    std::vector<uint64_t> slots;
    TinyHash th{};
    bool ok = false;
    for (uint32_t size = 64; !ok && size <= kTinySlotsMax; size <<= 1) {
      if (size < 2 * es.size()) continue;
      uint32_t lg = 0;
      while ((1u << lg) < size) ++lg;
      for (uint32_t seed = 0; !ok && seed < 64; ++seed) {
        th.c1 = (0x9E3779B1u + 0x6A09E667u * seed) | 1u;
        th.c2 = 0x85EBCA77u ^ (0xBB67AE85u * seed);
        th.c3 = (0xC2B2AE3Du + 0x3C6EF372u * seed) | 1u;
        th.shift = 32 - lg;
        th.size = size;
        slots.assign(size, ~0ull);
        ok = true;
        for (size_t i = 0; i < es.size() && ok; ++i) {
          uint64_t cur = short_key(es[i].lo, es[i].hb, es[i].len) | ((uint64_t)es[i].idx << 51);
          uint32_t s1, s2;
          const auto slots_of = [&](uint64_t v) {
            const uint32_t lo = (uint32_t)v, hb = (uint32_t)(v >> 32) & 0xffffu;
            const uint32_t len = (uint32_t)(v >> 48) & 7u;
            tiny_slots(tiny_key_hash(lo, short_tag(hb, len), th), th, s1, s2);
          };
          slots_of(cur);
          uint32_t at = s1;
          for (int kick = 0; kick < 500; ++kick) {
            std::swap(cur, slots[at]);
            if (cur == ~0ull) break;
            slots_of(cur);
            at = (at == s1) ? s2 : s1;
            if (kick == 499) ok = false;
          }
        }
      }
    }
    if (!ok) return fail(RK_ECUDA, "cannot build the short-pattern table");
    sw.th = th;
    sw.stab = reserve((uint64_t)th.size * 8 + kShortFilterWords * 4);
    memcpy(blob.data() + sw.stab, slots.data(), (uint64_t)th.size * 8);
    uint32_t* filt = reinterpret_cast<uint32_t*>(blob.data() + sw.stab + (uint64_t)th.size * 8);
    const uint32_t fbits = short_filter_bits(sw.sq);
    const auto set_bits = [&](uint32_t x) {
      const uint32_t h = short_filter_hash(x);
      filt[short_filter_word(h)] |= short_filter_bit_set(h, fbits);
    };
    for (const Entry& e : es) {
      if (sw.sq) {
        // the anchored q-grams p[j:j+q], j = 0, 1 (q + 1 <= m)
        uint8_t pb[8] = {};
        memcpy(pb, &e.lo, 4);
        memcpy(pb + 4, &e.hb, 2);
        for (int j = 0; j < 2; ++j) {
          uint32_t gram = 0;
          memcpy(&gram, pb + j, sw.sq);
          set_bits(gram);
        }
        if (short_refined(sw.sq)) set_bits(e.lo ^ kShortKeySalt);  // the 4-byte prefix
      } else {
        set_bits(tiny_key_hash(e.lo, short_tag(0u, e.len), th));
      }
    }
    plan.sweeps.push_back(sw);
  }
  for (; gi < plan.groups.size(); gi += kMultiMaxGroups) {
    const size_t g_end = std::min(plan.groups.size(), gi + kMultiMaxGroups);
    MultiPlan::Sweep sw{};
    for (size_t k = gi; k < g_end; ++k) sw.groups.push_back((uint32_t)k);
    const uint32_t m_min = plan.groups[gi].m;
    // (s, q = 4 * qwords) from the shortest length (q + s - 1 <= m_min) and the
    // alphabet: rich alphabets (>= 20 distinct pattern bytes) filter well with 8-byte
    // q-grams every 8 bytes; small ones (DNA) need longer q-grams
    bool seen[256] = {};
    uint32_t distinct = 0;
    for (size_t k = gi; k < g_end; ++k)
      for (uint64_t i = 0; i < (uint64_t)plan.groups[k].P * plan.groups[k].m; ++i) {
        const uint8_t byte = blob[plan.groups[k].pats + i];
        if (!seen[byte]) {
          seen[byte] = true;
          ++distinct;
        }
      }
    if (m_min >= 23 && distinct < 20) sw.qmode = 8, sw.qwords = 4;
    else if (m_min >= 15 && distinct < 20) sw.qmode = 4, sw.qwords = 3;
    else if (m_min >= 15) sw.qmode = 8, sw.qwords = 2;
    else if (m_min >= 11) sw.qmode = 4, sw.qwords = 2;
    else sw.qmode = 4, sw.qwords = 1;
    sw.qfilter = reserve(kQFilterWords * sizeof(uint32_t));
    // several lengths: 32-bit filter words (fewer bank conflicts, measured +10% on 64 mixed
    // lengths); one length: 64-bit blocks (fewer false positives, +3% on C3)
    sw.qf32 = (g_end - gi) > 1 ? 1u : 0u;
    std::unordered_map<uint32_t, uint64_t> groups_of;  // q-gram hash -> group mask
    for (size_t k = gi; k < g_end; ++k)
      for (uint32_t i = 0; i < plan.groups[k].P; ++i) {
        const uint8_t* p = blob.data() + plan.groups[k].pats + (uint64_t)i * plan.groups[k].m;
        for (uint32_t j = 0; j < sw.qmode; ++j) {
          uint32_t w[4] = {0, 0, 0, 0};
          memcpy(w, p + j, 4 * sw.qwords);
          uint32_t h = 0;
          switch (sw.qwords) {
            case 4: h = qgram_hash<4>(w); break;
            case 3: h = qgram_hash<3>(w); break;
            case 2: h = qgram_hash<2>(w); break;
            default: h = qgram_hash<1>(w); break;
          }
          uint32_t* qf = reinterpret_cast<uint32_t*>(blob.data() + sw.qfilter);
          if (sw.qf32) {
            qf[h >> kQWordShift] |= (1u << (h & 31)) | (1u << ((h >> 5) & 31)) | (1u << ((h >> 10) & 31));
          } else {
            uint32_t* blk = qf + 2 * (h >> kQBlockShift);
            blk[0] |= (1u << (h & 31)) | (1u << ((h >> 5) & 31));
            blk[1] |= (1u << ((h >> 10) & 31)) | (1u << ((h >> 15) & 31));
          }
          groups_of[h] |= 1ull << (k - gi);
        }
      }
    sw.qmap_size = 64;
    while (sw.qmap_size < 2 * groups_of.size()) sw.qmap_size <<= 1;
    sw.qmap = reserve((uint64_t)sw.qmap_size * sizeof(uint4));
    uint4* qmap = reinterpret_cast<uint4*>(blob.data() + sw.qmap);
    for (const auto& [h, mask] : groups_of) {
      uint32_t slot = (h * 0x9E3779B1u) & (sw.qmap_size - 1);
      while (qmap[slot].z | qmap[slot].w) slot = (slot + 1) & (sw.qmap_size - 1);
      qmap[slot] = make_uint4(h, 0u, (uint32_t)mask, (uint32_t)(mask >> 32));
    }
    plan.sweeps.push_back(sw);
  }

  // one pinned-staged upload of the whole blob
  if (int r = grow(&c->d_mblob, &c->mblob_cap, (uint64_t)blob.size(), false, s)) return r;
  if (c->h_mstage_cap < blob.size()) {
    RK_CUDA(cudaStreamSynchronize(s));
    if (c->h_mstage) cudaFreeHost(c->h_mstage);
    c->h_mstage = nullptr;
    RK_CUDA(cudaMallocHost(&c->h_mstage, blob.size()));
    c->h_mstage_cap = blob.size();
  } else {
    RK_CUDA(cudaStreamSynchronize(s));  // the staging buffer may still feed a previous upload
  }
  memcpy(c->h_mstage, blob.data(), blob.size());
  RK_CUDA(cudaMemcpyAsync(c->d_mblob, c->h_mstage, blob.size(), cudaMemcpyHostToDevice, s));
  plan.key = std::move(key);
  c->mplan = std::move(plan);
  return RK_OK;
}

namespace rkb {

// Launches the sweeps of a PatternSet over the device text (patterns already planned into
// c->mplan): every (window start, caller index) pair whose start lies in [start_lo,
// start_hi) is appended, unordered, to d_off (start + bias) / d_idx, the count to
// c->d_mcount.  Enqueued only.
int multi_enqueue(rk_ctx* c, const uint8_t* d_text, uint64_t n, uint64_t start_lo,
                  uint64_t start_hi, int64_t bias, int64_t* d_off, uint32_t* d_idx,
                  uint64_t cap, cudaStream_t s) {
  const MultiPlan& plan = c->mplan;
  RK_CUDA(cudaMemsetAsync(c->d_mcount, 0, sizeof(unsigned long long), s));
  const uint8_t* dev = c->d_mblob;
  auto group_of = [&](const MultiPlan::Group& b, uint64_t amis) {
    MultiGroup G{};
    G.pats = dev + b.pats;
    G.phash = reinterpret_cast<const uint64_t*>(dev + b.phash);
    G.order = reinterpret_cast<const uint32_t*>(dev + b.order);
    G.gidx = reinterpret_cast<const uint32_t*>(dev + b.gidx);
    G.table = reinterpret_cast<const uint2*>(dev + b.table);
    G.filter = reinterpret_cast<const uint32_t*>(dev + b.filter);
    // window starts the sweep may report: [start_lo, min(n - m + 1, start_hi))
    const uint64_t hi = b.m <= n ? std::min<uint64_t>(n - b.m + 1, start_hi) : 0;
    G.ys_hi = amis + std::max<uint64_t>(hi, start_lo);
    G.m = b.m;
    G.tsize = b.tsize;
    G.P = b.P;
    return G;
  };
  for (const MultiPlan::Sweep& sw : plan.sweeps) {
    // (lengths longer than the text stay in the sweep -- group bits are positions in
    // it -- with an empty window range)
    const uint32_t m_min = plan.groups[sw.groups.front()].m;
    if (m_min > n) continue;
    const uint64_t nw = n - m_min + 1;
    Geometry gg = geometry(d_text, m_min, 0, nw);
    MultiArgs p{};
    p.qmode = sw.qmode;
    p.qwords = sw.qwords;
    p.qf32 = sw.qf32;
    if (sw.qmode) {
      // tiles over the anchors e (q-gram ends): [first start + q - 1, last start of the
      // shortest length + q - 1 + s), clamped to the text
      const uint64_t q = 4ull * sw.qwords;
      gg.ja_lo = gg.amis + q - 1;
      gg.ja_hi = std::min<uint64_t>(gg.amis + nw - 1 + q - 1 + sw.qmode, gg.amis + n);
      gg.tile_first = gg.ja_lo / kTile;
      gg.num_tiles = (gg.ja_hi - 1) / kTile - gg.tile_first + 1;
      p.qfilter = reinterpret_cast<const uint32_t*>(dev + sw.qfilter);
      p.qmap = reinterpret_cast<const uint4*>(dev + sw.qmap);
      p.qmap_size = sw.qmap_size;
    } else {
      p.stab = dev + sw.stab;
      p.th = sw.th;
      p.sq = sw.sq;
      if (sw.sq) {
        // anchored short sweep: tiles over the anchors (q-gram ends, every 2 bytes) of the
        // window starts [amis, amis + nw); window validity is checked on the starts
        const uint64_t q = sw.sq;
        gg.ja_lo = gg.amis + q - 1;
        gg.ja_hi = std::min<uint64_t>(gg.amis + nw - 1 + q - 1 + 2, gg.amis + n);
        gg.tile_first = gg.ja_lo / kTile;
        gg.num_tiles = (gg.ja_hi - 1) / kTile - gg.tile_first + 1;
      }
      // (per-window short sweep: tiles over the window ends of the shortest length)
    }
    p.G = (uint32_t)sw.groups.size();
    for (size_t k = 0; k < sw.groups.size(); ++k)
      p.grp[k] = group_of(plan.groups[sw.groups[k]], gg.amis);
    p.g = text_geom(gg, n, m_min, 0);
    p.ys_lo = gg.amis + start_lo;
    p.out_bias = bias;
    p.out_off = d_off;
    p.out_idx = d_idx;
    p.cap = cap;
    p.counters = c->d_mcount;
    multi_set_append(p);
    const uint64_t grid = std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)c->num_sms * multi_blocks_per_sm(p),
                              (gg.num_tiles + kMultiWarps - 1) / kMultiWarps));
    RK_CUDA(launch_multi(p, (int)grid, s));
    ++c->launches;
  }

  return RK_OK;
}

// Orders k pairs of d_off / d_idx (k known on the host) by (caller index, offset) -- the
// reference's per-pattern ascending lists: one block in shared memory up to kSmallSort
// pairs, else the device radix sort.  Offsets < n, indices < P.
int order_pairs(rk_ctx* c, int64_t* d_off, uint32_t* d_idx, uint64_t k, uint64_t n, uint32_t P,
                cudaStream_t s) {
  if (k > kSmallSort) {
    const size_t need = sort_pairs_scratch(k);
    if (int r = grow(&c->d_sort, &c->sort_cap, (uint64_t)need, false, s)) return r;
    RK_CUDA(sort_pairs(d_off, d_idx, k, n, P, c->d_sort, c->sort_cap, s));
  } else if (k > 1) {
    RK_CUDA(small_sort_pairs(d_off, d_idx, nullptr, k, k, n, nullptr, s));
  }
  return RK_OK;
}

// The same for pairs whose count is on the device (d_count): the one-block sort reads it
// there and writes it to the pinned result word (mapped, no copy); the host waits once,
// and only a set above kSmallSort pairs needs the radix sort after that.  *total_out
// receives the pair count (which may exceed cap: only cap were written).
int multi_order(rk_ctx* c, int64_t* d_off, uint32_t* d_idx, uint64_t cap, uint64_t n, uint32_t P,
                const unsigned long long* d_count, uint64_t* total_out, cudaStream_t s) {
  c->h_mresult[0] = 0;
  RK_CUDA(small_sort_pairs(d_off, d_idx, d_count, 0, cap, n, c->h_mresult, s));
  RK_CUDA(cudaStreamSynchronize(s));
  const uint64_t total = *(volatile unsigned long long*)c->h_mresult;
  *total_out = total;
  const uint64_t k = std::min(total, cap);
  return k > kSmallSort ? order_pairs(c, d_off, d_idx, k, n, P, s) : RK_OK;
}

}  // namespace rkb

extern "C" {

const char* rk_version(void) { return "rkb200 0.1.0 sm_100a"; }

const char* rk_last_error(void) { return g_err.c_str(); }

int rk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rk_ctx_create(int device, rk_ctx_t** out) {
  if (!out) return fail(RK_EINVAL, "out is NULL");
  *out = nullptr;
  int ndev = rk_device_count();
  if (device < 0 || device >= ndev)
    return fail(RK_ECUDA, "CUDA device %d not available (%d visible)", device, ndev);
  DeviceGuard g(device);
  if (!g.ok) return fail(RK_ECUDA, "cudaSetDevice(%d) failed", device);
  cudaDeviceProp prop;
  RK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(RK_ECUDA, "device %d is sm_%d%d; librkb200 is built for sm_100a", device,
                prop.major, prop.minor);
  rk_ctx* c = new rk_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  RK_CUDA(cudaMalloc(&c->d_mcount, sizeof(unsigned long long)));
  RK_CUDA(cudaMallocHost(&c->h_counters, 4 * sizeof(unsigned long long)));
  RK_CUDA(cudaMallocHost(&c->h_mresult, 4 * sizeof(unsigned long long)));
  RK_CUDA(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
  RK_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
  for (auto& e : c->ev_copied) RK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RK_CUDA(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  RK_CUDA(cudaEventCreateWithFlags(&c->ev_switch, cudaEventDisableTiming));
  *out = c;
  return RK_OK;
}

int rk_ctx_destroy(rk_ctx_t* c) {
  if (!c) return RK_OK;
  DeviceGuard g(c->device);
  cudaDeviceSynchronize();
  cudaFree(c->d_sets);
  cudaFree(c->d_mcount);
  cudaFreeHost(c->h_counters);
  cudaFree(c->d_tile_info);
  cudaFree(c->d_emit_work);
  cudaFree(c->d_queue);
  cudaFree(c->d_masks);
  for (auto& sl : c->pat_cache) {
    cudaFree(sl.d);
    cudaFreeHost(sl.h);
  }
  cudaEventDestroy(c->ev_switch);
  cudaFree(c->d_stage);
  cudaFree(c->d_out_stage);
  for (auto* h : c->h_ring) cudaFreeHost(h);
  delete c->copier;
  for (auto e : c->ev_copied) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_ready);
  cudaStreamDestroy(c->s_copy);
  cudaStreamDestroy(c->s_comp);
  cudaFree(c->d_binfo);
  cudaFree(c->d_bspill);
  cudaFree(c->d_bmasks);
  cudaFree(c->d_bsets);
  cudaFreeHost(c->h_bcounts);
  cudaFree(c->d_mblob);
  cudaFree(c->d_sort);
  cudaFreeHost(c->h_mstage);
  cudaFreeHost(c->h_mresult);
  delete c;
  return RK_OK;
}

uint64_t rk_launch_count(rk_ctx_t* c) { return c ? c->launches : 0; }

int rk_scan_async(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                  uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out,
                  uint64_t cap, int64_t out_bias, uint64_t* d_counts, void* stream) {
  RK_HPROF("rk_scan_async total");
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (int r = check_scan_args(d_text, n, h_pattern, m, start, stop, d_out, cap)) return r;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(c, s)) return r;
  return enqueue_scan(c, d_text, n, h_pattern, m, hx, start, stop, d_out, cap, out_bias, s,
                      d_counts);
}

int rk_scan_bitmap(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                   uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, uint32_t* d_bitmap,
                   uint64_t* d_counts, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (int r = check_scan_args(d_text, n, h_pattern, m, start, stop, nullptr, 0)) return r;
  if (stop > start && !d_bitmap) return fail(RK_EINVAL, "bitmap pointer is NULL");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(c, s)) return r;
  c->last_scan.valid = false;
  if (stop > start)
    RK_CUDA(cudaMemsetAsync(d_bitmap, 0, ((stop - start + 31) / 32) * sizeof(uint32_t), s));
  if (stop <= start || hash_unreachable(m, hx)) return zero_result(c, d_counts, s);
  if (int r = upload_pattern(c, h_pattern, m, s)) return r;
  const Geometry gm = geometry(d_text, m, start, stop);
  if (int r = begin_scan(c, gm.num_tiles, s)) return r;
  if (int r = launch_one(c, d_text, n, m, hx, start, stop, 0, pack_pattern(h_pattern, m), s))
    return r;
  // bit of window start x = (end - m + 1 - amis) - start
  const int64_t bit_bias = -(int64_t)gm.amis - (int64_t)m + 1 - (int64_t)start;
  return emit(c, gm.num_tiles, gm.tile_first, 0, nullptr, 0, s, d_counts, d_bitmap, bit_bias);
}

int rk_scan_result(rk_ctx_t* c, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
                   void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  if (int r = enter(c, (cudaStream_t)stream)) return r;
  return read_counters(c, matches, collisions, hash_hits, (cudaStream_t)stream);
}

int rk_scan(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern, uint32_t m,
            uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out, uint64_t cap,
            uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (int r = check_scan_args(d_text, n, h_pattern, m, start, stop, d_out, cap)) return r;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(c, s)) return r;
  if (stop <= start || hash_unreachable(m, hx)) {
    if (int r = enqueue_scan(c, d_text, n, h_pattern, m, hx, start, stop, d_out, cap, 0, s))
      return r;
    return read_counters(c, matches, collisions, hash_hits, s);
  }
  // The emit kernel writes {matches, hash_hits, collisions} straight into the pinned
  // counter block (host memory mapped through UVA): no device-to-host copy sits between
  // the last kernel and the wait (C1, 1 MiB: the synchronous call is launch-bound).
  unsigned long long* hc = c->h_counters;
  if (int r = enqueue_scan(c, d_text, n, h_pattern, m, hx, start, stop, d_out, cap, 0, s,
                           (uint64_t*)hc))
    return r;
  RK_CUDA(cudaStreamSynchronize(s));
  if (matches) *matches = hc[0];
  if (hash_hits) *hash_hits = hc[1];
  if (collisions) *collisions = hc[2];
  return RK_OK;
}

int rk_scan_host(rk_ctx_t* c, const uint8_t* h_text, uint64_t n, const uint8_t* h_pattern,
                 uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* h_out,
                 uint64_t cap, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (int r = check_scan_args(h_text, n, h_pattern, m, start, stop, h_out, cap)) return r;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t sc = c->s_comp;
  if (int r = enter(c, sc)) return r;
  c->host_last = 0;
  if (stop <= start || hash_unreachable(m, hx)) {
    c->last_scan.valid = false;
    if (int r = zero_result(c, nullptr, sc)) return r;
    return read_counters(c, matches, collisions, hash_hits, sc);
  }
  if (int r = grow(&c->d_out_stage, &c->out_stage_cap, std::max<uint64_t>(cap, 1ull << 16), false,
                   sc))
    return r;
  if (int r = host_scan_enqueue(c, h_text, n, h_pattern, m, hx, start, stop, 0, nullptr)) return r;
  uint64_t mt = 0, co = 0, hh = 0;
  if (int r = read_counters(c, &mt, &co, &hh, sc)) return r;
  if (mt > c->out_stage_cap) {
    // more offsets than the staging output held: re-emit from the kept masks (no rescan)
    if (int r = grow(&c->d_out_stage, &c->out_stage_cap, mt, false, sc)) return r;
    if (int r = emit_last(c, c->d_out_stage, mt, sc)) return r;
  }
  c->host_last = mt;
  c->batch_segs.assign(1, rk_ctx::BatchSeg{c->d_out_stage, mt});
  const uint64_t nout = std::min(mt, cap);
  if (nout) {
    RK_CUDA(cudaMemcpyAsync(h_out, c->d_out_stage, nout * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            sc));
    RK_CUDA(cudaStreamSynchronize(sc));
  }
  if (matches) *matches = mt;
  if (collisions) *collisions = co;
  if (hash_hits) *hash_hits = hh;
  return RK_OK;
}

int rk_scan_host_batch(rk_ctx_t* c, const uint8_t* h_text, uint64_t n, const uint8_t* h_patterns,
                       const uint32_t* h_lengths, const uint64_t* h_hashes, uint32_t P,
                       int64_t* h_out, uint64_t cap, uint64_t* matches, uint64_t* collisions,
                       uint64_t* hash_hits) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (P < 1 || P > RK_BATCH_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_BATCH_MAX_PATTERNS);
  if (!h_patterns || !h_lengths || !h_hashes || !matches || !collisions || !hash_hits)
    return fail(RK_EINVAL, "NULL pattern or result arrays");
  for (uint32_t i = 0; i < P; ++i)
    if (h_lengths[i] < 1) return fail(RK_EINVAL, "pattern %u is empty", i);
  if (n && !h_text) return fail(RK_EINVAL, "text pointer is NULL");
  if (cap && !h_out) return fail(RK_EINVAL, "output pointer is NULL with cap > 0");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  cudaStream_t sc = c->s_comp, sk = c->s_copy;
  if (int r = enter(c, sc)) return r;
  c->host_last = 0;
  c->batch_segs.clear();
  c->last_scan.valid = false;

  // per pattern: its windows [0, n - m + 1) as a-space geometry of the staging buffer,
  // its scratch slices and device pattern copy
  struct Job {
    uint32_t m;
    uint64_t hx, nw;
    Geometry gall;
    uint64_t info_off, set_off, nb;
    const uint8_t* pat;
    PatWords pw;
    bool live;
  };
  std::vector<Job> jobs(P);
  uint64_t info_words = 0, set_words_all = 0, max_m = 0, pat_off = 0;
  for (uint32_t i = 0; i < P; ++i) {
    Job& j = jobs[i];
    j.m = h_lengths[i];
    j.hx = h_hashes[i];
    j.pat = h_patterns + pat_off;
    pat_off += j.m;
    j.nw = n >= j.m ? n - j.m + 1 : 0;
    j.live = j.nw > 0 && !hash_unreachable(j.m, j.hx);
    if (!j.live) continue;
    max_m = std::max<uint64_t>(max_m, j.m);
    j.gall = geometry(nullptr, j.m, 0, j.nw);  // the staging buffer is 256-byte aligned
    j.info_off = info_words;
    info_words += j.gall.num_tiles;
    j.nb = (j.gall.num_tiles + kEmitTiles - 1) / kEmitTiles;
    j.set_off = set_words_all;
    set_words_all += 4 + j.nb;
    j.pw = pack_pattern(j.pat, j.m);
  }
  // every pattern's device copy first (the cache may sync the stream to reuse a slot:
  // before any of this call's copies are queued)
  std::vector<const uint8_t*> dpat(P, nullptr);
  for (uint32_t i = 0; i < P; ++i) {
    if (!jobs[i].live) continue;
    if (int r = upload_pattern(c, jobs[i].pat, jobs[i].m, sc)) return r;
    dpat[i] = c->d_pattern;
  }
  if (c->h_bcounts_cap < P) {
    RK_CUDA(cudaStreamSynchronize(sc));
    if (c->h_bcounts) RK_CUDA(cudaFreeHost(c->h_bcounts));
    c->h_bcounts = nullptr;
    RK_CUDA(cudaMallocHost(&c->h_bcounts, 4ull * RK_BATCH_MAX_PATTERNS * sizeof(unsigned long long)));
    c->h_bcounts_cap = RK_BATCH_MAX_PATTERNS;
  }
  memset(c->h_bcounts, 0, 4ull * P * sizeof(unsigned long long));
  if (!info_words) {
    for (uint32_t i = 0; i < P; ++i) matches[i] = collisions[i] = hash_hits[i] = 0;
    return RK_OK;
  }
  if (int r = grow(&c->d_stage, &c->stage_cap, n, false, sc)) return r;
  if (int r = grow(&c->d_binfo, &c->binfo_cap, info_words, false, sc)) return r;
  if (int r = grow(&c->d_bmasks, &c->bmasks_cap, info_words * (uint64_t)(kTileChunks * 32), false,
                   sc))
    return r;
  if (int r = grow(&c->d_bsets, &c->bsets_cap, set_words_all, false, sc)) return r;
  constexpr uint64_t kSlot = 1ull << 16;  // offsets per pattern emitted before the counts are known
  if (int r = grow(&c->d_out_stage, &c->out_stage_cap, kSlot * P, false, sc)) return r;
  RK_CUDA(cudaMemsetAsync(c->d_bsets, 0, set_words_all * sizeof(unsigned long long), sc));
  std::vector<ScanScratch> xs(P);
  for (uint32_t i = 0; i < P; ++i) {
    if (!jobs[i].live) continue;
    xs[i].counters = c->d_bsets + jobs[i].set_off;
    xs[i].block_sums = xs[i].counters + 4;
    xs[i].tile_info = c->d_binfo + jobs[i].info_off;
    xs[i].masks = c->d_bmasks + jobs[i].info_off * (uint64_t)(kTileChunks * 32);
    xs[i].pattern = dpat[i];
  }
  cudaPointerAttributes attr;
  const bool pinned = cudaPointerGetAttributes(&attr, h_text) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (!pinned && !c->h_ring[0]) {
    for (auto& h : c->h_ring) RK_CUDA(cudaMallocHost(&h, kRingSlot));
    c->copier = new CopyPool();
  }

  // the text crosses PCIe ONCE: chunk k's bytes land on s_copy while every pattern's
  // windows ending in chunk k-1 are scanned on s_comp (the just-landed chunk is read from
  // L2 by the later patterns)
  const uint64_t k1 = (n - 1) / kStageChunk;
  uint64_t copied = 0;
  int slot = 0;
  for (uint64_t k = 0; k <= k1; ++k) {
    const uint64_t need = std::min(n, (k + 1) * kStageChunk);
    if (need > copied) {
      const uint64_t len = need - copied;
      if (pinned) {
        RK_CUDA(cudaMemcpyAsync(c->d_stage + copied, h_text + copied, len,
                                cudaMemcpyHostToDevice, sk));
      } else {
        for (uint64_t off = 0; off < len; off += kRingSlot) {
          const uint64_t l = std::min<uint64_t>(kRingSlot, len - off);
          RK_CUDA(cudaEventSynchronize(c->ev_copied[slot]));
          c->copier->copy(c->h_ring[slot], h_text + copied + off, l);
          RK_CUDA(cudaMemcpyAsync(c->d_stage + copied + off, c->h_ring[slot], l,
                                  cudaMemcpyHostToDevice, sk));
          RK_CUDA(cudaEventRecord(c->ev_copied[slot], sk));
          slot = (slot + 1) % kRing;
        }
      }
      copied = need;
      RK_CUDA(cudaEventRecord(c->ev_ready, sk));
      RK_CUDA(cudaStreamWaitEvent(sc, c->ev_ready, 0));
    }
    for (uint32_t i = 0; i < P; ++i) {
      const Job& j = jobs[i];
      if (!j.live) continue;
      const uint64_t e_lo = std::max(j.gall.ja_lo, k * kStageChunk);
      const uint64_t e_hi = std::min(j.gall.ja_hi, (k + 1) * kStageChunk);
      if (e_hi <= e_lo) continue;
      const uint64_t ws = e_lo - (j.m - 1), we = e_hi - (j.m - 1);
      const Geometry gk = geometry(c->d_stage, j.m, ws, we);
      if (int r = launch_one(c, c->d_stage, n, j.m, j.hx, ws, we,
                             gk.tile_first - j.gall.tile_first, j.pw, sc, &xs[i]))
        return r;
    }
  }
  // every pattern's ordered offsets into its slot; the counts land in mapped pinned memory
  for (uint32_t i = 0; i < P; ++i) {
    const Job& j = jobs[i];
    if (!j.live) continue;
    if (int r = emit(c, j.gall.num_tiles, j.gall.tile_first, -(int64_t)j.m + 1,
                     c->d_out_stage + kSlot * i, kSlot, sc, (uint64_t*)(c->h_bcounts + 4 * i),
                     nullptr, 0, &xs[i]))
      return r;
  }
  RK_CUDA(cudaStreamSynchronize(sc));
  uint64_t total = 0, spill = 0;
  for (uint32_t i = 0; i < P; ++i) {
    matches[i] = c->h_bcounts[4 * i];
    hash_hits[i] = c->h_bcounts[4 * i + 1];
    collisions[i] = c->h_bcounts[4 * i + 2];
    total += matches[i];
    if (matches[i] > kSlot) spill += (matches[i] + 31) & ~31ull;
  }
  // patterns with more offsets than their slot: re-emitted whole, from their kept
  // per-tile results, into a spill region after the slots (never a rescan)
  std::vector<const int64_t*> seg(P, nullptr);
  if (spill) {
    // (a separate buffer: growing d_out_stage would drop the slots' contents)
    if (int r = grow(&c->d_bspill, &c->bspill_cap, spill, false, sc)) return r;
    uint64_t at = 0;
    for (uint32_t i = 0; i < P; ++i) {
      if (matches[i] <= kSlot) continue;
      const Job& j = jobs[i];
      if (int r = emit(c, j.gall.num_tiles, j.gall.tile_first, -(int64_t)j.m + 1,
                       c->d_bspill + at, matches[i], sc, nullptr, nullptr, 0, &xs[i]))
        return r;
      seg[i] = c->d_bspill + at;
      at += (matches[i] + 31) & ~31ull;  // segments stay 256-byte aligned
    }
  }
  for (uint32_t i = 0; i < P; ++i) {
    if (!seg[i]) seg[i] = c->d_out_stage + kSlot * i;
    c->batch_segs.push_back(rk_ctx::BatchSeg{seg[i], matches[i]});
  }
  c->host_last = total;
  // the first cap offsets (pattern after pattern) to the host
  uint64_t done = 0;
  for (uint32_t i = 0; i < P && done < cap; ++i) {
    const uint64_t k = std::min<uint64_t>(matches[i], cap - done);
    if (k)
      RK_CUDA(cudaMemcpyAsync(h_out + done, seg[i], k * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              sc));
    done += k;
  }
  RK_CUDA(cudaStreamSynchronize(sc));
  return RK_OK;
}

int rk_scan_host_fetch(rk_ctx_t* c, int64_t* h_out, uint64_t first, uint64_t count) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  std::lock_guard<std::mutex> lk(c->mu);
  if (first > c->host_last || count > c->host_last - first)
    return fail(RK_EINVAL, "fetch [%llu, %llu) beyond the %llu offsets of the last host scan",
                (unsigned long long)first, (unsigned long long)(first + count),
                (unsigned long long)c->host_last);
  if (!count) return RK_OK;
  if (!h_out) return fail(RK_EINVAL, "NULL output");
  DeviceGuard g(c->device);
  if (int r = enter(c, c->s_comp)) return r;
  // the offsets are one segment per pattern (a single one after rk_scan_host)
  uint64_t base = 0, done = 0;
  for (const auto& sg : c->batch_segs) {
    if (done == count) break;
    const uint64_t lo = std::max(first + done, base), hi = std::min(first + count, base + sg.count);
    if (lo < hi) {
      RK_CUDA(cudaMemcpyAsync(h_out + done, sg.d + (lo - base), (hi - lo) * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, c->s_comp));
      done += hi - lo;
    }
    base += sg.count;
  }
  RK_CUDA(cudaStreamSynchronize(c->s_comp));
  return RK_OK;
}

int rk_scan_fetch(rk_ctx_t* c, int64_t* d_out, uint64_t cap, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (cap && !d_out) return fail(RK_EINVAL, "output pointer is NULL with cap > 0");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->last_scan.valid || c->last_scan.host)
    return fail(RK_EINVAL, "rk_scan_fetch: the context's last call was not a device scan "
                "with matches to re-emit");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int r = enter(c, s)) return r;
  return emit_last(c, d_out, cap, s);
}

int rk_window_hashes(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, uint32_t m, uint64_t start,
                     uint64_t stop, uint64_t* d_out, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (m < 1) return fail(RK_EINVAL, "window length must be >= 1");
  if (stop == start) return RK_OK;
  if (stop < start || stop - 1 + m > n)
    return fail(RK_EINVAL, "window range [%llu, %llu) of length %u out of bounds for text of "
                "length %llu", (unsigned long long)start, (unsigned long long)stop, m,
                (unsigned long long)n);
  if (!d_text || !d_out) return fail(RK_EINVAL, "NULL pointer");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  RK_CUDA(launch_window_hashes(d_text, n, m, start, stop, d_out, (cudaStream_t)stream));
  ++c->launches;
  return RK_OK;
}

int rk_generate(rk_ctx_t* c, uint8_t* d_out, uint64_t count, uint64_t seed, uint64_t skip,
                const uint8_t* h_alphabet, uint32_t k, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (!h_alphabet || k < 1 || k > 256) return fail(RK_EINVAL, "alphabet must have 1..256 symbols");
  if (count && !d_out) return fail(RK_EINVAL, "NULL output");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard g(c->device);
  RK_CUDA(launch_generate(d_out, count, seed, skip, h_alphabet, k, (cudaStream_t)stream));
  ++c->launches;
  return RK_OK;
}

int rk_multi_scan(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_patterns,
                  uint32_t P, uint32_t m, const uint64_t* h_hashes, int64_t* d_off,
                  uint32_t* d_idx, uint64_t cap, uint64_t* pairs, void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (m < 1) return fail(RK_EINVAL, "patterns must be non-empty");
  if (P < 1 || P > RK_MULTI_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_MULTI_MAX_PATTERNS);
  std::vector<uint32_t> lengths(P, m);
  return rk_multi_scan_mixed(c, d_text, n, h_patterns, lengths.data(), P, h_hashes, d_off, d_idx,
                             cap, pairs, stream);
}

int rk_multi_scan_mixed(rk_ctx_t* c, const uint8_t* d_text, uint64_t n, const uint8_t* h_patterns,
                        const uint32_t* h_lengths, uint32_t P, const uint64_t* h_hashes,
                        int64_t* d_off, uint32_t* d_idx, uint64_t cap, uint64_t* pairs,
                        void* stream) {
  if (!c) return fail(RK_EINVAL, "context is NULL");
  if (P < 1 || P > RK_MULTI_MAX_PATTERNS)
    return fail(RK_EINVAL, "pattern count %u outside [1, %d]", P, RK_MULTI_MAX_PATTERNS);
  if (!h_patterns || !h_lengths || !h_hashes) return fail(RK_EINVAL, "NULL pattern arrays");
  for (uint32_t i = 0; i < P; ++i)
    if (h_lengths[i] < 1) return fail(RK_EINVAL, "pattern %u is empty", i);
  if (cap && (!d_off || !d_idx)) return fail(RK_EINVAL, "NULL output with cap > 0");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  *pairs = 0;
  if (int r = enter(c, s)) return r;
  uint64_t max_len = 0, min_len = ~0ull;
  for (uint32_t i = 0; i < P; ++i) {
    max_len = std::max<uint64_t>(max_len, h_lengths[i]);
    min_len = std::min<uint64_t>(min_len, h_lengths[i]);
  }
  if (min_len > n) return RK_OK;  // no pattern has a window
  if (!d_text) return fail(RK_EINVAL, "text pointer is NULL");
  if (int r = multi_plan(c, h_patterns, h_lengths, P, h_hashes, s)) return r;
  if (int r = multi_enqueue(c, d_text, n, 0, n, 0, d_off, d_idx, cap, s)) return r;
  return multi_order(c, d_off, d_idx, cap, n, P, c->d_mcount, pairs, s);
}

}  // extern "C"
