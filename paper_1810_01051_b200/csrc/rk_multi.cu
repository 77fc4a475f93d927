// rk_multi.cu -- multi-pattern scan over one equal-length group of a PatternSet
// (/root/reference/pkg/src/rkmatch/matcher.py:139-153: per length, hash every window,
// look the hash up in the set's hash index, byte-verify every pattern carrying it).
//
// The reference's O(P) compare per window becomes one shared-memory probe:
//   * a 2^16-bit filter (8 KiB smem) keyed by a multiplicative hash of low32(window hash)
//     rejects ~98% of windows at P = 1024 with one LDS;
//   * survivors probe an open-addressing table (smem) of the distinct low32 keys, whose
//     entries point at the run of patterns sharing that key (several patterns may share
//     a hash, e.g. "ac"/"ba", tests/test_matcher.py:139-146);
//   * each such pattern is confirmed by its 64-bit hash (m > 24) and by its bytes.
// Hits are appended with warp ballot/popc and one atomic per warp; the host orders them
// by (pattern index, offset), which is exactly the reference's per-pattern ascending lists.
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

constexpr int kFilterBits = 1 << 16;
constexpr uint32_t kEmpty = 0xffffffffu;

struct MultiArgs {
  const uint8_t* abase;
  uint64_t amis;
  uint64_t n;
  const uint8_t* pats;        // P * m bytes, deduplicated, index order
  const uint64_t* phash;      // 64-bit hash per pattern
  const uint32_t* filter;     // kFilterBits / 32 words
  const uint2* table;         // tsize entries: {key, (first << 13) | count}, val kEmpty = free
  const uint32_t* order;      // pattern indices grouped by key
  uint64_t ja_lo, ja_hi;
  uint64_t tile0, num_tiles, ticket_base;
  int64_t* out_off;
  uint32_t* out_idx;
  uint64_t cap;
  unsigned long long* ticket;
  unsigned long long* counters;  // [0] = pairs found
  uint32_t m, P, tsize;
};

__device__ __forceinline__ uint32_t mhash(uint32_t key) { return key * 0x9E3779B1u; }

__device__ __forceinline__ bool filter_test(const uint32_t* __restrict__ f, uint32_t L) {
  const uint32_t b = mhash(L) >> 16;
  return (f[b >> 5] >> (b & 31)) & 1u;
}

template <int M>
__device__ __forceinline__ bool multi_fast_chunk(const Vec32& v, const uint32_t* f, int lane,
                                                 uint32_t& carryS, uint32_t (&carryW)[8]) {
  bool any = false;
  if constexpr (M >= 32) {
    const uint32_t F = fold32(v.w);
    const uint32_t up = __shfl_up_sync(kFull, F, 1);
    const uint32_t top = __shfl_sync(kFull, F, 31);
    uint32_t S = lane == 0 ? carryS : up;
    carryS = top;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      S = 2u * S + bsel(v.w[k >> 2], k & 3);
      any |= filter_test(f, S);
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
      const int io = 32 + k - M;
      const uint32_t in = bsel(v.w[k >> 2], k & 3);
      const uint32_t out = io < 32 ? bsel(lb[io >> 2], io & 3) : bsel(v.w[(io - 32) >> 2], io & 3);
      L = 2u * L + in - (out << M);
      any |= filter_test(f, L);
    }
  }
  return any;
}

__device__ __noinline__ uint64_t multi_hash_global(const MultiArgs& a, int64_t je) {
  const uint8_t* text = a.abase + a.amis;
  const int64_t span = a.m < 64 ? (int64_t)a.m : 64;
  uint64_t h = 0;
  for (int64_t i = je - span + 1; i <= je; ++i) h = (h << 1) + (uint64_t)text[i];
  return h;
}

// Returns the matching pattern index for the window ending at a-position ja with
// low32 hash L, or -1.  Deduplicated patterns of one length are distinct, so at most
// one pattern can byte-match a window.
__device__ __noinline__ int multi_resolve(const MultiArgs& a, const uint2* __restrict__ tbl,
                                          uint32_t L, int64_t ja) {
  uint32_t slot = mhash(L) & (a.tsize - 1);
  for (;;) {
    const uint2 e = tbl[slot];
    if (e.y == kEmpty) return -1;
    if (e.x == L) {
      const uint32_t first = e.y >> 13, cnt = e.y & 0x1fff;
      const int64_t je = ja - (int64_t)a.amis;
      const int64_t x = je - (int64_t)a.m + 1;
      const uint8_t* w = a.abase + a.amis + x;
      uint64_t h = 0;
      bool have_h = false;
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t idx = a.order[first + q];
        if (a.m > 24) {
          if (!have_h) {
            h = multi_hash_global(a, je);
            have_h = true;
          }
          if (h != a.phash[idx]) continue;
        }
        const uint8_t* p = a.pats + (uint64_t)idx * a.m;
        bool eq = true;
        for (uint32_t i = 0; i < a.m; ++i)
          if (w[i] != p[i]) {
            eq = false;
            break;
          }
        if (eq) return (int)idx;
      }
      return -1;
    }
    slot = (slot + 1) & (a.tsize - 1);
  }
}

template <int M>
__device__ __forceinline__ void multi_slow_chunk(const MultiArgs& a, const uint2* tbl,
                                                 const uint32_t* f, int64_t J, int lane,
                                                 const ScanArgs& ea) {
  const Vec32 v = load_edge(ea, J);
  const Vec32 lbv = load_edge(ea, J - 32);
  uint32_t L;
  if constexpr (M >= 32) L = fold32(lbv.w);
  else L = fold_tail<M>(lbv.w);
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    if constexpr (M >= 32) {
      L = 2u * L + bsel(v.w[k >> 2], k & 3);
    } else {
      const int io = 32 + k - M;
      const uint32_t in = bsel(v.w[k >> 2], k & 3);
      const uint32_t out =
          io < 32 ? bsel(lbv.w[io >> 2], io & 3) : bsel(v.w[(io - 32) >> 2], io & 3);
      L = 2u * L + in - (out << M);
    }
    const int64_t ja = J + k;
    int idx = -1;
    if (ja >= (int64_t)a.ja_lo && ja < (int64_t)a.ja_hi && filter_test(f, L))
      idx = multi_resolve(a, tbl, L, ja);
    const unsigned hit = __ballot_sync(kFull, idx >= 0);
    if (hit) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)__popc(hit));
      base = __shfl_sync(kFull, base, 0);
      if (idx >= 0) {
        const uint64_t pos = base + __popc(hit & ((1u << lane) - 1u));
        if (pos < a.cap) {
          a.out_off[pos] = ja - (int64_t)a.amis - (int64_t)a.m + 1;
          a.out_idx[pos] = (uint32_t)idx;
        }
      }
    }
  }
}

template <int M>
__global__ void __launch_bounds__(kBlock) rk_multi_kernel(const MultiArgs a) {
  __shared__ uint32_t sfilter[kFilterBits / 32];
  extern __shared__ uint2 stable[];
  for (int i = threadIdx.x; i < kFilterBits / 32; i += blockDim.x) sfilter[i] = a.filter[i];
  for (uint32_t i = threadIdx.x; i < a.tsize; i += blockDim.x) stable[i] = a.table[i];
  __syncthreads();

  // the edge-safe loader works on ScanArgs; reuse it with the text fields
  ScanArgs ea{};
  ea.abase = a.abase;
  ea.amis = a.amis;
  ea.n = a.n;

  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1ull);
    t = __shfl_sync(kFull, t, 0) - a.ticket_base;
    if (t >= a.num_tiles) break;

    const int64_t tile_a = (int64_t)((a.tile0 + t) * (uint64_t)kTile);
    const bool interior =
        tile_a - 32 >= (int64_t)a.amis && tile_a + kTile <= (int64_t)(a.amis + a.n);
    uint32_t carryS = 0, carryW[8];
    {
      const Vec32 prev = load_edge(ea, tile_a - 32);
#pragma unroll
      for (int i = 0; i < 8; ++i) carryW[i] = prev.w[i];
      if constexpr (M >= 32) carryS = fold32(prev.w);
    }
    const uint8_t* lane_base = a.abase + tile_a + lane * kR;
    Vec32 buf[kPrefetch];
#pragma unroll
    for (int i = 0; i < kPrefetch; ++i)
      buf[i] = interior ? ldg256(lane_base + i * kChunk)
                        : load_edge(ea, tile_a + i * kChunk + lane * kR);
    uint32_t cand = 0;
#pragma unroll 1
    for (int c0 = 0; c0 < kTileChunks; c0 += kPrefetch) {
#pragma unroll
      for (int i = 0; i < kPrefetch; ++i) {
        const int c = c0 + i;
        const Vec32 v = buf[i];
        if (c + kPrefetch < kTileChunks)
          buf[i] = interior ? ldg256(lane_base + (c + kPrefetch) * kChunk)
                            : load_edge(ea, tile_a + (c + kPrefetch) * kChunk + lane * kR);
        const bool any = multi_fast_chunk<M>(v, sfilter, lane, carryS, carryW);
        if (__any_sync(kFull, any)) cand |= 1u << c;
      }
    }
    while (cand) {
      const int c = __ffs(cand) - 1;
      cand &= cand - 1;
      multi_slow_chunk<M>(a, stable, sfilter, tile_a + c * kChunk + lane * kR, lane, ea);
    }
  }
}

template <int M>
static cudaError_t launch_multi_m(const MultiArgs& a, int grid, cudaStream_t s) {
  const size_t smem = (size_t)a.tsize * sizeof(uint2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rk_multi_kernel<M>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  rk_multi_kernel<M><<<grid, kBlock, smem, s>>>(a);
  return cudaGetLastError();
}

using MultiLaunchFn = cudaError_t (*)(const MultiArgs&, int, cudaStream_t);
template <int... Ms>
struct MultiTable {
  static constexpr MultiLaunchFn launch[sizeof...(Ms)] = {&launch_multi_m<Ms>...};
};
using MTable = MultiTable<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                          21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32>;

cudaError_t launch_multi(const MultiArgs& a, int grid, cudaStream_t s) {
  return MTable::launch[a.m >= 32 ? 31 : (int)a.m - 1](a, grid, s);
}

}  // namespace rkb

// ------------------------------------------------------------------ host helpers
namespace rkb {
cudaError_t launch_multi_plan(const MultiHostPlan& p, int grid, cudaStream_t s) {
  MultiArgs a;
  a.abase = p.abase;
  a.amis = p.amis;
  a.n = p.n;
  a.pats = p.pats;
  a.phash = p.phash;
  a.filter = p.filter;
  a.table = p.table;
  a.order = p.order;
  a.ja_lo = p.ja_lo;
  a.ja_hi = p.ja_hi;
  a.tile0 = p.tile0;
  a.num_tiles = p.num_tiles;
  a.ticket_base = p.ticket_base;
  a.out_off = p.out_off;
  a.out_idx = p.out_idx;
  a.cap = p.cap;
  a.ticket = p.ticket;
  a.counters = p.counters;
  a.m = p.m;
  a.P = p.P;
  a.tsize = p.tsize;
  return launch_multi(a, grid, s);
}
}  // namespace rkb
