// rk_emit.cu -- ordered emission of match offsets (the ordered concatenation of
// /root/reference/pkg/src/rkmatch/parallel.py:168-172, done on the device).
//
// The scan kernel never waits on other tiles: it leaves, per 8 KiB tile, its match
// count and chunk bitmap (tile_info), the per-lane hit masks of the chunks that matched
// (masks), and per-256-tile sums (block_sums).  This kernel turns that into the ordered
// int64 offsets: block b adds up block_sums[0..b), scans its 256 tile counts, and each
// warp expands the masks of its tiles with matches into window starts written at their
// final positions -- ascending, deterministic, no sort, no text re-read.  For sparse
// matches this is a few microseconds per GiB.
//
// Dense outputs (every window matching, BASELINE config C5) are write-bound: a chunk's
// offsets are staged in shared memory (padded so the lane-strided fill is nearly
// conflict-free) and written back as contiguous, coalesced 16-byte stores; a chunk whose
// 1024 windows all match is written directly as an arithmetic run.
#include <algorithm>

#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

constexpr int kEmitWarps = kEmitTiles / 32;
constexpr int kPadded = kChunk + kChunk / 32;  // 1056 slots: +1 per 32

__device__ __forceinline__ int padded(int i) { return i + (i >> 5); }

__device__ __forceinline__ void st_global_v2(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// Expands the hit masks of the tiles with matches among group g's 256 tiles (info = this
// thread's tile_info, excl = its exclusive match prefix) into ordered offsets.
__device__ __forceinline__ void emit_group(const EmitArgs& e, uint64_t g, uint32_t info,
                                           uint64_t excl, int64_t* stage, int lane, int warp) {
  const uint32_t cnt = info & 0xffffu;
  unsigned todo = __ballot_sync(kFull, cnt != 0);
  if (!todo) return;
  if (e.bitmap) {
    // bitmap mode (MatchResult.to_bitmap): each lane ORs its 32 hit bits into place
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t tseq = g * kEmitTiles + warp * 32 + j;
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
  auto fetch = [&](int j, uint32_t(&dst)[kTileChunks]) {
    const uint64_t tseq = g * kEmitTiles + warp * 32 + j;
    const uint32_t fl = __shfl_sync(kFull, info, j) >> 16;
    const uint32_t* tm = e.masks + tseq * (kTileChunks * 32);
#pragma unroll
    for (int c = 0; c < kTileChunks; ++c) dst[c] = ((fl >> c) & 1u) ? tm[c * 32 + lane] : 0u;
  };
  int jn = __ffs(todo) - 1;
  fetch(jn, nxt);
  while (todo) {
    const int j = jn;
    todo &= todo - 1;
#pragma unroll
    for (int c = 0; c < kTileChunks; ++c) hms[c] = nxt[c];
    jn = todo ? __ffs(todo) - 1 : -1;
    if (jn >= 0) fetch(jn, nxt);
    const uint64_t tseq = g * kEmitTiles + warp * 32 + j;
    uint32_t flags = __shfl_sync(kFull, info, j) >> 16;
    uint64_t run = __shfl_sync(kFull, excl, j);
    const int64_t tile_a = (int64_t)((e.tile0 + tseq) * (uint64_t)kTile);
#pragma unroll
    for (int c = 0; c < kTileChunks; ++c) {
      if (!((flags >> c) & 1u)) continue;
      uint32_t hm = hms[c];
      const int64_t chunk0 = tile_a + c * kChunk + e.start_bias;  // value of window 0
      if (__all_sync(kFull, hm == 0xffffffffu)) {
        // all 1024 windows match: a contiguous arithmetic run
        const uint64_t lim = e.cap > run ? e.cap - run : 0;
        int64_t* o = e.out + run;
        if (run + kChunk <= e.cap && ((uintptr_t)o & 15u) == 0) {  // 16-byte stores
#pragma unroll 4
          for (int i = 2 * lane; i < kChunk; i += 64) st_global_v2(o + i, chunk0 + i, chunk0 + i + 1);
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
}

// Block b handles the groups (of kEmitTiles tiles) [b G, (b + 1) G), G = e.groups_per_block,
// so that a sparse emit is one wave of blocks; the next group's tile_info is loaded while
// the current one is scanned and expanded.
__global__ void __launch_bounds__(kEmitTiles) rk_emit_kernel(const EmitArgs e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scan's writes are visible
  asm volatile("griddepcontrol.launch_dependents;");  // the next scan may be scheduled
  extern __shared__ __align__(16) int64_t stage_all[];
  __shared__ unsigned long long red[kEmitWarps];
  __shared__ uint32_t wsum[kEmitWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* stage = stage_all + warp * kPadded;
  const uint64_t G = e.groups_per_block;
  const uint64_t g0 = (uint64_t)blockIdx.x * G;
  const uint64_t groups = (e.num_tiles + kEmitTiles - 1) / kEmitTiles;
  const uint64_t g_end = g0 + G < groups ? g0 + G : groups;

  auto load_info = [&](uint64_t g) -> uint32_t {
    const uint64_t seq = g * kEmitTiles + tid;
    return (g < g_end && seq < e.num_tiles) ? e.tile_info[seq] : 0u;
  };
  uint32_t info = load_info(g0);  // issued with the prefix loads below
  unsigned long long pre = 0;
  for (uint64_t i = tid; i < g0; i += kEmitTiles) pre += e.block_sums[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(kFull, pre, o);
  if (lane == 0) red[warp] = pre;
  for (uint64_t i = (uint64_t)blockIdx.x * kEmitTiles + tid; i < e.clear_words;
       i += (uint64_t)gridDim.x * kEmitTiles)
    e.clear[i] = 0ull;
  __syncthreads();
  unsigned long long base = 0;
#pragma unroll
  for (int w = 0; w < kEmitWarps; ++w) base += red[w];

  for (uint64_t g = g0; g < g_end; ++g) {
    const uint32_t next = load_info(g + 1);
    const uint32_t cnt = info & 0xffffu;
    const uint32_t inc = warp_incl_scan(cnt, lane);
    __syncthreads();  // wsum of the previous group has been read
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0, gtot = 0;
#pragma unroll
    for (int w = 0; w < kEmitWarps; ++w) {
      if (w < warp) wpre += wsum[w];
      gtot += wsum[w];
    }
    const uint64_t excl = base + wpre + inc - cnt;
    const uint64_t seq = g * kEmitTiles + tid;
    if (seq == e.num_tiles - 1) {
      e.counters[0] = excl + cnt;
      if (e.counts_out) {
        e.counts_out[0] = excl + cnt;
        e.counts_out[1] = e.counters[1];
        e.counts_out[2] = e.counters[2];
      }
    }
    emit_group(e, g, info, excl, stage, lane, warp);
    base += gtot;
    info = next;
  }
}

// The emit grid is launched as a programmatic dependent of the scan, so its CTAs are
// placed as scan CTAs retire: with a small footprint several would pile onto the first SMs
// to free up (a dense emit then ran on a third of the SMs, 2.4x slower).  Reserving more
// than half an SM's shared memory keeps it to one CTA per SM.
#ifndef RK_EMIT_MIN_SMEM_KB
#define RK_EMIT_MIN_SMEM_KB 116
#endif
constexpr size_t kEmitMinSmem = RK_EMIT_MIN_SMEM_KB * 1024;
#ifndef RK_EMIT_MAX_GROUPS
#define RK_EMIT_MAX_GROUPS 4
#endif
constexpr uint64_t kEmitMaxGroups = RK_EMIT_MAX_GROUPS;  // groups of kEmitTiles per block
size_t emit_smem_bytes() {
  const size_t b = (size_t)kEmitWarps * kPadded * sizeof(int64_t);
  return b < kEmitMinSmem ? kEmitMinSmem : b;
}

cudaError_t launch_emit(EmitArgs e, int num_sms, cudaStream_t s) {
  // one wave of blocks (one per SM, see below) when the scan is up to num_sms groups x G
  const uint64_t groups = (e.num_tiles + kEmitTiles - 1) / kEmitTiles;
  const uint64_t sms = num_sms > 0 ? (uint64_t)num_sms : 1;
  e.groups_per_block = std::max<uint64_t>(1, std::min<uint64_t>(kEmitMaxGroups, (groups + sms - 1) / sms));
  const uint64_t blocks = (groups + e.groups_per_block - 1) / e.groups_per_block;
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
