// rk_emit.cu -- ordered emission of match offsets (the ordered concatenation of
// /root/reference/pkg/src/rkmatch/parallel.py:168-172, done on the device).
//
// The scan kernel never waits on other tiles: it leaves, per 8 KiB tile, its match
// count and chunk bitmap (tile_info), the per-lane hit masks of the chunks that matched
// (masks), and per-256-tile sums (block_sums).  This kernel turns that into the ordered
// int64 offsets: each block adds up the counts before its span of tiles, scans its tile
// counts, and each warp expands the masks of its tiles with matches into window starts
// written at their final positions -- ascending, deterministic, no sort, no text
// re-read.  For sparse matches this is a few microseconds per GiB.
//
// Dense outputs (every window matching, BASELINE config C5) are write-bound: a chunk's
// offsets are staged in shared memory (padded so the lane-strided fill is nearly
// conflict-free) and written back coalesced; a chunk whose 1024 windows all match is
// written directly as an arithmetic run of 32-byte stores.  Tiles with >= kDeferMin
// matches are not expanded by the block whose span holds them but queued, and expanded
// by whichever warps are free once their own spans are done (dynamic balance: a static
// split writes at the pace of the slowest SM).
#include <algorithm>

#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

constexpr int kEmitWarps = kEmitTiles / 32;
#ifndef RK_EMIT_MAX_GROUPS
#define RK_EMIT_MAX_GROUPS 4
#endif
constexpr uint64_t kEmitMaxGroups = RK_EMIT_MAX_GROUPS;  // x kEmitTiles: a block's largest span
#ifndef RK_EMIT_LD
#define RK_EMIT_LD(p) (*(p))
#endif
constexpr int kPadded = kChunk + kChunk / 32;  // 1056 slots: +1 per 32

__device__ __forceinline__ int padded(int i) { return i + (i >> 5); }

__device__ __forceinline__ void st_global_v4(int64_t* p, int64_t a) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(a + 1),
               "l"(a + 2), "l"(a + 3)
               : "memory");
}

// Writes the arithmetic run v0, v0 + 1, ..., v0 + kChunk - 1 to o[0, kChunk) (o 8-byte
// aligned): up to 3 scalar stores reach a 32-byte boundary, the body goes out as 32-byte
// stores (STG.256, 1 KiB per warp instruction), then up to 3 scalar stores.  A run's start
// is rarely aligned: C5's first chunk has 1021 matches, which shifts every later run.
__device__ __forceinline__ void store_run(int64_t* o, int64_t v0, int lane) {
  const int head = (int)(((32u - ((uint32_t)(uintptr_t)o & 31u)) & 31u) >> 3);
  if (lane < head) o[lane] = v0 + lane;
  int64_t* ob = o + head;
  const int64_t vb = v0 + head;
  const int body = (kChunk - head) & ~3;
#pragma unroll 2
  for (int i = 4 * lane; i < body; i += 128) st_global_v4(ob + i, vb + i);
  if (lane < kChunk - head - body) ob[body + lane] = vb + body + lane;
}

// Loads the hit masks of tile tseq's flagged chunks (one round of independent loads).
__device__ __forceinline__ void fetch_masks(const EmitArgs& e, uint64_t tseq, uint32_t flags,
                                            int lane, uint32_t (&dst)[kTileChunks]) {
  const uint32_t* tm = e.masks + tseq * (kTileChunks * 32);
#pragma unroll
  for (int c = 0; c < kTileChunks; ++c) dst[c] = ((flags >> c) & 1u) ? tm[c * 32 + lane] : 0u;
}

// Writes tile tseq's match offsets (hit masks hms of its flagged chunks) at out[run, ...).
// The emit's code is kept small (rolled chunk loop): it runs beside the next scan's CTAs,
// and a 3x larger emit (this expansion unrolled, inlined in both phases) cost that scan
// 0.7% on the C2 sweep -- instruction-cache pressure, measured.
__device__ __forceinline__ void expand_tile(const EmitArgs& e, uint64_t tseq, uint32_t flags,
                                        uint64_t run, const uint32_t (&hms)[kTileChunks],
                                        int64_t* stage, int lane) {
  const int64_t tile_a = (int64_t)((e.tile0 + tseq) * (uint64_t)kTile);
  uint32_t h[kTileChunks];
#pragma unroll
  for (int c = 0; c < kTileChunks; ++c) h[c] = hms[c];
  // a rolled loop over the chunks (the masks rotate through h[0]: registers, not a local
  // array) keeps the kernel's code small
#pragma unroll 1
  for (int c = 0; c < kTileChunks; ++c) {
    uint32_t hm = h[0];
#pragma unroll
    for (int i = 0; i + 1 < kTileChunks; ++i) h[i] = h[i + 1];
    if (!((flags >> c) & 1u)) continue;
    const int64_t chunk0 = tile_a + c * kChunk + e.start_bias;  // value of window 0
    if (__all_sync(kFull, hm == 0xffffffffu)) {
      // all 1024 windows match: a contiguous arithmetic run
      const uint64_t lim = e.cap > run ? e.cap - run : 0;
      int64_t* o = e.out + run;
      if (run + kChunk <= e.cap && ((uintptr_t)o & 7u) == 0) {
        store_run(o, chunk0, lane);
      } else {
        for (int i = lane; i < kChunk; i += 32)
          if ((uint64_t)i < lim) e.out[run + i] = chunk0 + i;
      }
      run += kChunk;
      continue;
    }
    const uint32_t n = __popc(hm);
    const uint32_t i2 = warp_incl_scan(n, lane);
    const uint32_t tot = __shfl_sync(kFull, i2, 31);
    // stage this chunk's offsets in order, then write them back coalesced
    int r = (int)(i2 - n);
    const int64_t v0 = chunk0 + lane * kR;
    while (hm) {
      const int k = __ffs(hm) - 1;
      hm &= hm - 1;
      stage[padded(r++)] = v0 + k;
    }
    __syncwarp();
    const uint64_t lim = e.cap > run ? e.cap - run : 0;
    for (int i = lane; i < (int)tot; i += 32)
      if ((uint64_t)i < lim) e.out[run + i] = stage[padded(i)];
    __syncwarp();
    run += tot;
  }
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int kQueueTileBits = 22;
#ifdef RK_DEBUG_CHECKS
#define RK_DCHECK(c) \
  do {               \
    if (!(c)) __trap(); \
  } while (0)
#else
#define RK_DCHECK(c) \
  do {               \
  } while (0)
#endif

// Expands the hit masks of the warp's tiles with matches -- lane j's tile is tw + j ts,
// info its tile_info, excl its exclusive match prefix -- into ordered offsets.
__device__ __forceinline__ void emit_group(const EmitArgs& e, uint64_t tw, uint32_t ts,
                                           uint32_t info, uint64_t excl, int64_t* stage,
                                           int lane) {
  const uint32_t cnt = info & 0xffffu;
  unsigned todo = __ballot_sync(kFull, cnt != 0);
  if (!todo) return;
  if (e.bitmap) {
    // bitmap mode (MatchResult.to_bitmap): each lane ORs its 32 hit bits into place
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t tseq = tw + (uint64_t)j * ts;
      uint32_t flags = __shfl_sync(kFull, info, j) >> 16;
      const int64_t tile_a = (int64_t)((e.tile0 + tseq) * (uint64_t)kTile);
      const uint32_t* tm = e.masks + tseq * (kTileChunks * 32);
      while (flags) {
        const int c = __ffs(flags) - 1;
        flags &= flags - 1;
        const uint32_t hm = tm[c * 32 + lane];
        if (hm) {
          // hm only has bits of valid windows, so every nonzero part lands in the bitmap
          const int64_t bit = tile_a + c * kChunk + lane * kR + e.bit_bias;
          const int64_t word = bit >> 5;  // floor, also for the first (partial) word
          const int sh = (int)(bit & 31);
          const uint32_t lo = hm << sh, hi = sh ? hm >> (32 - sh) : 0u;
          if (lo) atomicOr(&e.bitmap[word], lo);
          if (hi) atomicOr(&e.bitmap[word + 1], hi);
        }
      }
    }
    return;
  }
  // the hit masks of a tile come in one round of independent loads, issued while the
  // previous tile is being expanded (not one load latency per chunk)
  uint32_t hms[kTileChunks], nxt[kTileChunks];
  int jn = __ffs(todo) - 1;
  fetch_masks(e, tw + (uint64_t)jn * ts, __shfl_sync(kFull, info, jn) >> 16, lane, nxt);
  while (todo) {
    const int j = jn;
    todo &= todo - 1;
#pragma unroll
    for (int c = 0; c < kTileChunks; ++c) hms[c] = nxt[c];
    jn = todo ? __ffs(todo) - 1 : -1;
    const uint32_t fl_next = __shfl_sync(kFull, info, jn < 0 ? 0 : jn) >> 16;
    if (jn >= 0) fetch_masks(e, tw + (uint64_t)jn * ts, fl_next, lane, nxt);
    const uint32_t flags = __shfl_sync(kFull, info, j) >> 16;
    expand_tile(e, tw + (uint64_t)j * ts, flags, __shfl_sync(kFull, excl, j), hms, stage, lane);
  }
}

// Second phase (scans with dense tiles only): once a block has finished its span, its
// warps take queued dense tiles one at a time from a ticket counter until the queue is
// drained and every block has finished its span.  Dense output is write-bound, and
// statically assigned spans run at the pace of the slowest SM (measured: 6.2 TB/s for a
// static split of a 2 GiB write against 7.3 for dynamic tickets, tools/write_fronts.cu).
// Waiting for the other blocks needs them all resident: the grid is one wave of one CTA
// per SM (launch_emit), and all of them have started before anything else may be
// scheduled behind them (programmatic launch triggers once every CTA has run).  Entries
// are zeroed after use and the last block out resets the counters.
__device__ __forceinline__ unsigned long long claim_ticket(const EmitArgs& e, int lane) {
  unsigned long long t = 0;
  if (lane == 0) t = atomicAdd(&e.work[0], 1ull);
  return __shfl_sync(kFull, t, 0);
}

// Entry t once published, or 0 when the queue is drained and every block has
// finished its span (blocking: lane 0 spins on the entry and the done count).
__device__ __forceinline__ unsigned long long wait_entry(const EmitArgs& e, unsigned long long t,
                                                         int lane) {
  unsigned long long ex = 0;
  if (lane == 0) {
    unsigned long long t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
      if (t < e.num_tiles) ex = ld_relaxed(&e.queue[t]);
      if (ex) break;
      if (ld_acquire(&e.work[2]) == gridDim.x && t >= ld_acquire(&e.work[1])) break;
      if ((spins & 1023u) == 0) {
        // a producer missing for 60 s (other work can hold SMs for a while, never that
        // long): fail loudly instead of hanging
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (!t0) t0 = now;
        if (now - t0 > 60ull * 1000000000ull) __trap();
      }
      __nanosleep(100);
    }
  }
  return __shfl_sync(kFull, ex, 0);
}

// Entry t if already published, else 0 (non-blocking probe).
__device__ __forceinline__ unsigned long long probe_entry(const EmitArgs& e, unsigned long long t,
                                                          int lane) {
  unsigned long long ex = 0;
  if (lane == 0 && t < e.num_tiles) ex = ld_relaxed(&e.queue[t]);
  return __shfl_sync(kFull, ex, 0);
}

struct QueuedTile {
  uint64_t tseq;
  uint32_t flags;
  uint32_t hms[kTileChunks];
};

constexpr unsigned long long kQueueFull = 1ull << 63;  // every window of the tile matches

__device__ __forceinline__ void load_entry(const EmitArgs& e, unsigned long long ex, int lane,
                                           QueuedTile& q) {
  q.tseq = ex & ((1ull << kQueueTileBits) - 1);
  RK_DCHECK(q.tseq < e.num_tiles);
  if (ex & kQueueFull) {  // known from the entry: no tile_info or mask loads
    q.flags = (1u << kTileChunks) - 1u;
#pragma unroll
    for (int c = 0; c < kTileChunks; ++c) q.hms[c] = ~0u;
    return;
  }
  q.flags = e.tile_info[q.tseq] >> 16;
  fetch_masks(e, q.tseq, q.flags, lane, q.hms);
}

__device__ __forceinline__ void drain_queue(const EmitArgs& e, int64_t* stage, int lane) {
  // software-pipelined: the next ticket is claimed, and its entry loaded if already
  // published, before the current tile is expanded (a tile's claim-and-load chain is a
  // few microseconds of latency against ~10 of writing it)
  unsigned long long t = claim_ticket(e, lane);
  unsigned long long ex = wait_entry(e, t, lane);
  QueuedTile cur, nxt;
  if (ex) load_entry(e, ex, lane, cur);
  while (ex) {
    const unsigned long long t2 = claim_ticket(e, lane);
    unsigned long long ex2 = probe_entry(e, t2, lane);
    if (ex2) load_entry(e, ex2, lane, nxt);
    __syncwarp();
    if (lane == 0) e.queue[t] = 0ull;  // consumed: the queue is left zeroed
    expand_tile(e, cur.tseq, cur.flags, ((ex & ~kQueueFull) >> kQueueTileBits) - 1, cur.hms, stage,
                lane);
    if (!ex2) {
      ex2 = wait_entry(e, t2, lane);
      if (ex2) load_entry(e, ex2, lane, nxt);
    }
    t = t2;
    ex = ex2;
    cur = nxt;
  }
}

// Block b handles the tiles [b S, (b + 1) S), S = e.tiles_per_block <= 1024, each thread
// 4 consecutive ones (the block's starting offset is block_sums over the groups before
// its span plus the counts of the tiles of its first group that precede it; one block-wide
// scan orders the rest).  Sparse tiles are expanded in place; dense ones are queued for
// the balanced second phase.
__global__ void __launch_bounds__(kEmitTiles) rk_emit_kernel(const EmitArgs e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scan's writes are visible
  asm volatile("griddepcontrol.launch_dependents;");  // the next scan may be scheduled
  extern __shared__ __align__(16) int64_t stage_all[];
  __shared__ unsigned long long red[kEmitWarps];
  __shared__ uint32_t wsum[kEmitWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* stage = stage_all + warp * kPadded;
  const uint64_t S = e.tiles_per_block;
  const uint64_t t_begin = (uint64_t)blockIdx.x * S;
  const uint64_t t_end = t_begin + S < e.num_tiles ? t_begin + S : e.num_tiles;

  // Thread tid owns the Q consecutive tiles from tq (a span is at most Q x 256 tiles):
  // all tile_info loads are issued at once and one block-wide scan orders them -- one
  // barrier per emit instead of two per 256 tiles (the emit sits on the critical path
  // between two scans of a sweep: C2 1.487 -> 1.480 ms per step)
  constexpr int Q = (int)kEmitMaxGroups;
  const uint64_t tq = t_begin + (uint64_t)tid * Q;
  uint32_t inf[Q];
  uint32_t tsum = 0;
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    const uint64_t seq = tq + k;
    inf[k] = seq < t_end ? RK_EMIT_LD(&e.tile_info[seq]) : 0u;
    tsum += inf[k] & 0xffffu;
  }
  const uint64_t gb = t_begin / kEmitTiles;
  unsigned long long pre = 0;
  for (uint64_t i = tid; i < gb; i += kEmitTiles) pre += RK_EMIT_LD(&e.block_sums[i]);
  // the balanced phase runs when the scan saw a warp match a dense tile's worth
  // (counters[3]; every block reads the same flag, so all agree)
  const bool defer = e.defer_min && e.counters[3] != 0;
  if (gb * kEmitTiles + tid < t_begin) pre += RK_EMIT_LD(&e.tile_info[gb * kEmitTiles + tid]) & 0xffffu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(kFull, pre, o);
  const uint32_t inc = warp_incl_scan(tsum, lane);
  if (lane == 0) red[warp] = pre;
  if (lane == 31) wsum[warp] = inc;
  for (uint64_t i = (uint64_t)blockIdx.x * kEmitTiles + tid; i < e.clear_words;
       i += (uint64_t)gridDim.x * kEmitTiles)
    e.clear[i] = 0ull;
  __syncthreads();
  unsigned long long base = 0;
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kEmitWarps; ++w) {
    base += red[w];
    if (w < warp) wpre += wsum[w];
  }
#ifdef RK_EMIT_DEBUG
  if (tid == 0) RK_EMIT_DEBUG[blockIdx.x] = base;
#endif
  uint64_t ex[Q];
  ex[0] = base + wpre + inc - tsum;
#pragma unroll
  for (int k = 1; k < Q; ++k) ex[k] = ex[k - 1] + (inf[k - 1] & 0xffffu);
  if (defer) {
    // dense tiles to the queue, in tile order (lane-major, then k: ascending tiles), so
    // consecutive tickets write neighbouring output
    uint32_t dm = 0;
#pragma unroll
    for (int k = 0; k < Q; ++k) dm |= ((inf[k] & 0xffffu) >= kDeferMin ? 1u : 0u) << k;
    const uint32_t d = __popc(dm);
    const uint32_t dinc = warp_incl_scan(d, lane);
    const uint32_t dtot = __shfl_sync(kFull, dinc, 31);
    if (dtot) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(&e.work[1], (unsigned long long)dtot);
      at = __shfl_sync(kFull, at, 0) + dinc - d;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        if ((dm >> k) & 1u) {
          RK_DCHECK(at < e.num_tiles && tq + k < e.num_tiles);
          const bool full = inf[k] == ((uint32_t)kTile | (((1u << kTileChunks) - 1u) << 16));
          st_relaxed(&e.queue[at], ((ex[k] + 1) << kQueueTileBits) | (tq + k) |
                                       (full ? kQueueFull : 0ull));
          ++at;
          inf[k] = 0u;  // not expanded here
        }
      }
    }
  }
  if (t_end == e.num_tiles && tq <= e.num_tiles - 1 && e.num_tiles - 1 < tq + Q) {
    // the last tile's thread: the totals
    const uint64_t total = ex[0] + tsum;
    e.counters[0] = total;
    if (e.counts_out) {
      e.counts_out[0] = total;
      e.counts_out[1] = e.counters[1];
      e.counts_out[2] = e.counters[2];
    }
  }
  // (a rolled loop -- the tiles' words rotate through inf[0] / ex[0] -- keeps the emit's
  // code small: it runs beside the next scan's CTAs)
#pragma unroll 1
  for (int k = 0; k < Q; ++k) {
    emit_group(e, t_begin + (uint64_t)warp * 32 * Q + k, Q, inf[0], ex[0], stage, lane);
#pragma unroll
    for (int j = 0; j + 1 < Q; ++j) {
      inf[j] = inf[j + 1];
      ex[j] = ex[j + 1];
    }
  }
  if (defer) {
    __syncthreads();  // this block's queue entries are all published
    if (tid == 0) {
      __threadfence();
      atomicAdd(&e.work[2], 1ull);
    }
    drain_queue(e, stage, lane);
    __syncthreads();  // this block's warps are out of the queue
    if (tid == 0 && atomicAdd(&e.work[3], 1ull) == gridDim.x - 1) {
      e.work[0] = 0;  // the last block out: a clean queue for the next emit
      e.work[1] = 0;
      e.work[2] = 0;
      e.work[3] = 0;
    }
  }
}

// The emit grid is launched as a programmatic dependent of the scan, so its CTAs are
// placed as scan CTAs retire: with a small footprint several would pile onto the first SMs
// to free up (a dense emit then ran on a third of the SMs, 2.4x slower).  Reserving more
// than half an SM's shared memory keeps it to one CTA per SM.
#ifndef RK_EMIT_CTAS
#define RK_EMIT_CTAS 1  // emit CTAs per SM (the grid is a whole number of waves of these)
#endif
#ifndef RK_EMIT_MIN_SMEM_KB
#define RK_EMIT_MIN_SMEM_KB (228 / (RK_EMIT_CTAS + 1) + 1)
#endif
constexpr size_t kEmitMinSmem = RK_EMIT_MIN_SMEM_KB * 1024;
size_t emit_smem_bytes() {
  const size_t b = (size_t)kEmitWarps * kPadded * sizeof(int64_t);
  return b < kEmitMinSmem ? kEmitMinSmem : b;
}

cudaError_t launch_emit(EmitArgs e, int num_sms, cudaStream_t s) {
  const uint64_t sms = (num_sms > 0 ? (uint64_t)num_sms : 1) * RK_EMIT_CTAS;
  const uint64_t tiles = e.num_tiles > 0 ? e.num_tiles : 1;
  // the dense-tile queue (offsets mode, when the caller provides its buffers; used by the
  // kernel only if the scan saw a dense tile) needs all blocks resident: one wave
  e.defer_min = (kDeferMin > 0 && !e.bitmap && e.work && e.queue) ? kDeferMin : 0;
  // Whole waves of one block per SM, each block's span at most kEmitMaxGroups x 256 tiles
  // and at least 32 (one warp's worth), equal spans: a scan of up to 148 x 4 groups (1.16
  // GiB) is one wave, which the queue needs (measured against spans of whole groups with
  // helper blocks for the queue: the same C5, 0.3% faster on the C2 sweep).
  const uint64_t per_wave = sms * kEmitMaxGroups * kEmitTiles;
  uint64_t blocks = std::min<uint64_t>(sms * ((tiles + per_wave - 1) / per_wave), (tiles + 31) / 32);
  e.tiles_per_block = (tiles + blocks - 1) / blocks;
  blocks = (tiles + e.tiles_per_block - 1) / e.tiles_per_block;
  if (blocks > sms || tiles >= (1ull << kQueueTileBits)) e.defer_min = 0;  // one wave
  static bool attr[kMaxDevices] = {};  // the smem opt-in is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices || !attr[dev]) {
    cudaError_t err = cudaFuncSetAttribute(rk_emit_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)emit_smem_bytes());
    if (err != cudaSuccess) return err;
    if (dev < kMaxDevices) attr[dev] = true;
  }
  // programmatic dependent launch: the emit grid is scheduled as the scan's CTAs retire
  // and waits (griddepcontrol.wait) for the scan's results, instead of paying a full
  // launch gap after the scan drains
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kEmitTiles);
  cfg.dynamicSmemBytes = emit_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = RK_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, rk_emit_kernel, e);
}

}  // namespace rkb
