// rk_multi_impl.cuh -- multi-pattern scan over one equal-length group of a PatternSet
// (/root/reference/pkg/src/rkmatch/matcher.py:139-153: per length, hash every window,
// look the hash up in the set's hash index, byte-verify every pattern carrying it).
//
// Same streaming engine as the single-pattern scan (TMA ring, exact 32-bit roll); the
// reference's O(P) compare per window becomes shared-memory lookups:
//   * a 2^16-bit filter (8 KiB smem) keyed by a multiplicative hash of low32(window hash)
//     rejects ~98% of windows at P = 1024 with one LDS;
//   * survivors probe an open-addressing table (smem) of the distinct low32 keys, whose
//     entries point at the run of patterns sharing that key (several patterns may share
//     a hash, e.g. "ac"/"ba", tests/test_matcher.py:139-146);
//   * each such pattern is confirmed by its 64-bit hash (m > 24) and by its bytes.
// Hits are appended with warp ballot/popc and one atomic per warp; the host orders them
// by (pattern index, offset), which is exactly the reference's per-pattern ascending lists.
#pragma once
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

__device__ __forceinline__ uint32_t mhash(uint32_t key) { return key * 0x9E3779B1u; }

__device__ __forceinline__ bool filter_test(const uint32_t* __restrict__ f, uint32_t L) {
  const uint32_t b = mhash(L) >> 16;
  return (f[b >> 5] >> (b & 31)) & 1u;
}

static __device__ __noinline__ uint64_t multi_hash_global(const uint8_t* text, uint32_t m,
                                                         int64_t je) {
  const int64_t span = m < 64 ? (int64_t)m : 64;
  uint64_t h = 0;
  for (int64_t i = je - span + 1; i <= je; ++i) h = (h << 1) + (uint64_t)text[i];
  return h;
}

// Index of the pattern the window ending at text index je (low32 hash L) matches, or -1.
// Deduplicated patterns of one length are distinct, so at most one can byte-match.
static __device__ __noinline__ int multi_resolve(const uint8_t* text, const uint8_t* pats,
                                                 const uint64_t* phash, const uint32_t* order,
                                                 const uint2* __restrict__ tbl, uint32_t tsize,
                                                 uint32_t m, uint32_t L, int64_t je) {
  uint32_t slot = mhash(L) & (tsize - 1);
  for (;;) {
    const uint2 e = tbl[slot];
    if (e.y == kMultiEmpty) return -1;
    if (e.x == L) {
      const uint32_t first = e.y >> 13, cnt = e.y & 0x1fff;
      const uint8_t* w = text + je - (int64_t)m + 1;
      uint64_t h = 0;
      bool have_h = false;
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t idx = order[first + q];
        if (m > 24) {
          if (!have_h) {
            h = multi_hash_global(text, m, je);
            have_h = true;
          }
          if (h != phash[idx]) continue;
        }
        const uint8_t* p = pats + (uint64_t)idx * m;
        bool eq = true;
        for (uint32_t i = 0; i < m; ++i)
          if (w[i] != p[i]) {
            eq = false;
            break;
          }
        if (eq) return (int)idx;
      }
      return -1;
    }
    slot = (slot + 1) & (tsize - 1);
  }
}

template <int M>
__device__ __forceinline__ void multi_slow_chunk(const MultiArgs& a, const uint2* tbl,
                                                 const uint32_t* f, int64_t J, int lane) {
  const TextGeom& g = a.g;
  const Vec32 v = load_edge(g, J);
  const Vec32 lbv = load_edge(g, J - 32);
  const uint8_t* text = g.abase + g.amis;
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
    if (g.valid_end(ja) && filter_test(f, L))
      idx = multi_resolve(text, a.pats, a.phash, a.order, tbl, a.tsize, g.m, L,
                          ja - (int64_t)g.amis);
    const unsigned hit = __ballot_sync(kFull, idx >= 0);
    if (hit) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)__popc(hit));
      base = __shfl_sync(kFull, base, 0);
      if (idx >= 0) {
        const uint64_t pos = base + __popc(hit & ((1u << lane) - 1u));
        if (pos < a.cap) {
          a.out_off[pos] = ja - (int64_t)g.amis - (int64_t)g.m + 1;
          a.out_idx[pos] = (uint32_t)idx;
        }
      }
    }
  }
}

template <int M>
__global__ void __launch_bounds__(kBlock) rk_multi_kernel(const MultiArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  WarpRing* rings = reinterpret_cast<WarpRing*>(smem);
  uint32_t* sfilter = reinterpret_cast<uint32_t*>(smem + sizeof(WarpRing) * kWarpsPerBlock);
  uint2* stable = reinterpret_cast<uint2*>(sfilter + kMultiFilterWords);
  for (int i = threadIdx.x; i < kMultiFilterWords; i += blockDim.x) sfilter[i] = a.filter[i];
  for (uint32_t i = threadIdx.x; i < a.tsize; i += blockDim.x) stable[i] = a.table[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  WarpRing* R = rings + warp;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * kWarpsPerBlock;
  const uint64_t w = (uint64_t)blockIdx.x * kWarpsPerBlock + warp;
  const auto pred = [sfilter](uint32_t L) { return filter_test(sfilter, L); };
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    uint32_t cand = fast_tile<M>(a.g, R, S, t, lane, pred);
    const int64_t ta = a.g.tile_a(t);
    while (cand) {
      const int c = __ffs(cand) - 1;
      cand &= cand - 1;
      multi_slow_chunk<M>(a, stable, sfilter, ta + c * kChunk + lane * kR, lane);
    }
  }
}

template <int M>
cudaError_t launch_multi_m(const MultiArgs& a, int grid, cudaStream_t s) {
  const size_t smem = multi_smem_bytes(a.tsize);
  cudaError_t e = cudaFuncSetAttribute(rk_multi_kernel<M>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  rk_multi_kernel<M><<<grid, kBlock, smem, s>>>(a);
  return cudaGetLastError();
}

template <int M>
int multi_occupancy_m(uint32_t tsize) {
  const size_t smem = multi_smem_bytes(tsize);
  cudaFuncSetAttribute(rk_multi_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rk_multi_kernel<M>, kBlock, smem);
  return b > 0 ? b : 1;
}

}  // namespace rkb
