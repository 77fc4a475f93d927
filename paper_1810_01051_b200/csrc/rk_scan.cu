// rk_scan.cu -- single-pattern exact scan for sm_100a (the reference's _scan_range,
// /root/reference/pkg/src/rkmatch/_scan.py:28-50, plus the ordered merge of
// parallel.py:155-172), fused into one pass:
//
//   LDG.256 stream (1 KiB per warp step, 4 steps in flight)
//     -> exact 32-bit rolling hash per window (dp4a-folded seed, 1 shift-add per byte)
//     -> compare with low32(hx)  (candidates are ~2^-32 of windows on random text)
//     -> candidates: 64-bit hash + byte verify -> match / collision counters
//     -> per-tile hit masks in shared memory
//     -> decoupled look-back over 16 KiB tiles -> ordered int64 window starts.
//
// Each warp owns whole tiles (dynamic ticket), so the output is globally ascending
// without a sort, and the text is read from HBM exactly once.
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

template <int M>
__device__ __forceinline__ bool valid_end(const ScanArgs& a, int64_t ja) {
  return ja >= (int64_t)a.ja_lo && ja < (int64_t)a.ja_hi;
}

// 64-bit hash of the window whose last byte is at text index je (global memory).
__device__ __noinline__ uint64_t hash_window_global(const ScanArgs& a, int64_t je) {
  const uint8_t* text = a.abase + a.amis;
  const int64_t span = a.m < 64 ? (int64_t)a.m : 64;
  uint64_t h = 0;
  for (int64_t i = je - span + 1; i <= je; ++i) h = (h << 1) + (uint64_t)text[i];
  return h;
}

__device__ __noinline__ bool verify_global(const ScanArgs& a, int64_t x) {
  const uint8_t* text = a.abase + a.amis + x;
  for (uint32_t i = 0; i < a.m; ++i)
    if (text[i] != a.pattern[i]) return false;
  return true;
}

// Fast pass over one chunk: returns true if any window of this lane's 32 end positions
// has low32(hash) == T.  `carry*` hold the previous chunk's lane-31 state.
template <int M>
__device__ __forceinline__ bool fast_chunk(const Vec32& v, uint32_t T, int lane, uint32_t& carryS,
                                           uint32_t (&carryW)[8]) {
  bool any = false;
  if constexpr (M >= 32) {
    const uint32_t F = fold32(v.w);  // = S at this lane's last byte
    const uint32_t up = __shfl_up_sync(kFull, F, 1);
    const uint32_t top = __shfl_sync(kFull, F, 31);
    uint32_t S = lane == 0 ? carryS : up;
    carryS = top;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      S = 2u * S + bsel(v.w[k >> 2], k & 3);
      any |= (S == T);
    }
  } else {
    constexpr int w0 = (32 - M) >> 2;
    uint32_t lb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i >= w0) {
        const uint32_t up = __shfl_up_sync(kFull, v.w[i], 1);
        const uint32_t top = __shfl_sync(kFull, v.w[i], 31);
        lb[i] = lane == 0 ? carryW[i] : up;
        carryW[i] = top;
      } else {
        lb[i] = 0;
      }
    }
    uint32_t L = fold_tail<M>(lb);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int ii = 32 + k, io = 32 + k - M;
      const uint32_t in = bsel(v.w[k >> 2], k & 3);
      const uint32_t out = io < 32 ? bsel(lb[io >> 2], io & 3) : bsel(v.w[(io - 32) >> 2], io & 3);
      (void)ii;
      L = 2u * L + in - (out << M);
      any |= (L == T);
    }
  }
  return any;
}

struct SlowOut {
  uint32_t hm;    // hit bits (window end = J + k)
  uint32_t hits;  // hash hits (matches + collisions)
};

// Slow pass over one chunk that had a candidate: exact per-window decisions.
template <int M>
__device__ __forceinline__ SlowOut slow_chunk(const ScanArgs& a, int64_t J) {
  SlowOut r{0u, 0u};
  const Vec32 v = load_edge(a, J);
  const Vec32 lbv = load_edge(a, J - 32);
  const uint32_t T = (uint32_t)a.hx;
  if constexpr (M >= 32) {
    uint32_t S = fold32(lbv.w);
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      S = 2u * S + bsel(v.w[k >> 2], k & 3);
      if (S == T && valid_end<M>(a, J + k)) {
        const int64_t je = J + k - (int64_t)a.amis;  // text index of the last byte
        if (hash_window_global(a, je) == a.hx) {
          ++r.hits;
          if (verify_global(a, je - (int64_t)a.m + 1)) r.hm |= 1u << k;
        }
      }
    }
  } else {
    uint32_t L = fold_tail<M>(lbv.w);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int io = 32 + k - M;
      const uint32_t in = bsel(v.w[k >> 2], k & 3);
      const uint32_t out =
          io < 32 ? bsel(lbv.w[io >> 2], io & 3) : bsel(v.w[(io - 32) >> 2], io & 3);
      L = 2u * L + in - (out << M);
      if (L == T && valid_end<M>(a, J + k)) {
        // window bytes are positions [33+k-M, 32+k] of lbv ++ v
        bool hit = true;
        if constexpr (M > 24) {
          uint64_t h = 0;
#pragma unroll
          for (int i = 0; i < M; ++i) {
            const int p = 33 + k - M + i;
            const uint32_t b = p < 32 ? bsel(lbv.w[p >> 2], p & 3) : bsel(v.w[(p - 32) >> 2], p & 3);
            h = (h << 1) + b;
          }
          hit = (h == a.hx);
        }
        if (hit) {
          ++r.hits;
          bool eq = true;
#pragma unroll
          for (int i = 0; i < M; ++i) {
            const int p = 33 + k - M + i;
            const uint32_t b = p < 32 ? bsel(lbv.w[p >> 2], p & 3) : bsel(v.w[(p - 32) >> 2], p & 3);
            eq &= (b == bsel(a.pw.w[i >> 2], i & 3));
          }
          if (eq) r.hm |= 1u << k;
        }
      }
    }
  }
  return r;
}

template <int M>
__device__ __forceinline__ void scan_tile(const ScanArgs& a, uint64_t t, int lane,
                                          uint32_t* __restrict__ smask) {
  const int64_t tile_a = (int64_t)((a.tile0 + t) * (uint64_t)kTile);
  const bool interior =
      tile_a - 32 >= (int64_t)a.amis && tile_a + kTile <= (int64_t)(a.amis + a.n);
  const uint32_t T = (uint32_t)a.hx;

  // state carried into chunk 0's lane 0: the 32 bytes before the tile
  uint32_t carryS = 0;
  uint32_t carryW[8];
  {
    const Vec32 prev = load_edge(a, tile_a - 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) carryW[i] = prev.w[i];
    if constexpr (M >= 32) carryS = fold32(prev.w);
  }

  const uint8_t* lane_base = a.abase + tile_a + lane * kR;
  Vec32 buf[kPrefetch];
#pragma unroll
  for (int i = 0; i < kPrefetch; ++i)
    buf[i] = interior ? ldg256(lane_base + i * kChunk) : load_edge(a, tile_a + i * kChunk + lane * kR);

  uint32_t cand = 0;
#pragma unroll 1
  for (int c0 = 0; c0 < kTileChunks; c0 += kPrefetch) {
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i) {
      const int c = c0 + i;
      const Vec32 v = buf[i];
      if (c + kPrefetch < kTileChunks) {
        buf[i] = interior ? ldg256(lane_base + (c + kPrefetch) * kChunk)
                          : load_edge(a, tile_a + (c + kPrefetch) * kChunk + lane * kR);
      }
      const bool any = fast_chunk<M>(v, T, lane, carryS, carryW);
      if (__any_sync(kFull, any)) cand |= 1u << c;
    }
  }

  // exact pass over the (rare) chunks with candidates
  uint32_t hitflags = 0, my_matches = 0, my_hits = 0;
  while (cand) {
    const int c = __ffs(cand) - 1;
    cand &= cand - 1;
    const SlowOut r = slow_chunk<M>(a, tile_a + c * kChunk + lane * kR);
    my_hits += r.hits;
    my_matches += __popc(r.hm);
    if (__ballot_sync(kFull, r.hm != 0)) {
      smask[c * 32 + lane] = r.hm;
      hitflags |= 1u << c;
    }
  }

  const uint64_t agg = warp_sum_u64(my_matches);
  const uint64_t hits = warp_sum_u64(my_hits);
  if (lane == 0 && hits) {
    atomicAdd(&a.counters[1], (unsigned long long)hits);
    atomicAdd(&a.counters[2], (unsigned long long)(hits - agg));
  }
  const uint64_t excl = lookback(a.status, a.seq_base + t, a.epoch, agg, lane);
  if (a.last_launch && t == a.num_tiles - 1 && lane == 0) a.counters[0] = excl + agg;

  // ordered emission of this tile's window starts
  uint64_t run = excl;
  const int64_t start_bias = a.out_bias - (int64_t)a.amis - (int64_t)a.m + 1;
  while (hitflags) {
    const int c = __ffs(hitflags) - 1;
    hitflags &= hitflags - 1;
    uint32_t hm = smask[c * 32 + lane];
    const uint32_t cnt = __popc(hm);
    const uint32_t inc = warp_incl_scan(cnt, lane);
    const uint32_t tot = __shfl_sync(kFull, inc, 31);
    uint64_t pos = run + inc - cnt;
    const int64_t J = tile_a + c * kChunk + lane * kR;
    while (hm) {
      const int k = __ffs(hm) - 1;
      hm &= hm - 1;
      if (pos < a.cap) a.out[pos] = J + k + start_bias;
      ++pos;
    }
    run += tot;
  }
}

template <int M>
__global__ void __launch_bounds__(kBlock) rk_scan_kernel(const ScanArgs a) {
  __shared__ uint32_t smask[kWarpsPerBlock][kTileChunks * 32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(kFull, t, 0) - a.ticket_base;
    if (t >= a.num_tiles) break;
    scan_tile<M>(a, t, lane, smask[warp]);
  }
}

// ------------------------------------------------------------------ host launchers
template <int M>
static cudaError_t launch_m(const ScanArgs& a, int grid, cudaStream_t s) {
  rk_scan_kernel<M><<<grid, kBlock, 0, s>>>(a);
  return cudaGetLastError();
}

template <int M>
static int occupancy_m() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rk_scan_kernel<M>, kBlock, 0);
  return b > 0 ? b : 1;
}

using LaunchFn = cudaError_t (*)(const ScanArgs&, int, cudaStream_t);
using OccFn = int (*)();

template <int... Ms>
struct Table {
  static constexpr LaunchFn launch[sizeof...(Ms)] = {&launch_m<Ms>...};
  static constexpr OccFn occ[sizeof...(Ms)] = {&occupancy_m<Ms>...};
};
using ScanTable = Table<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                        21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32>;

static int variant_of(uint32_t m) { return m >= 32 ? 31 : (int)m - 1; }

int scan_blocks_per_sm(uint32_t m) {
  static int cache[32] = {0};
  const int v = variant_of(m);
  if (!cache[v]) cache[v] = ScanTable::occ[v]();
  return cache[v];
}

cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t s) {
  return ScanTable::launch[variant_of(a.m)](a, grid, s);
}

}  // namespace rkb
