// rk_multi_impl.cuh -- multi-pattern scan of a PatternSet (/root/reference/pkg/src/rkmatch/
// matcher.py:125-157: per length, hash every window, look the hash up in the set's hash
// index, byte-verify every pattern carrying it) -- here all lengths >= 7 of a set share
// ONE sweep over the text, the reference's per-length passes being the
// special case of one length group.
//
// The exact test is the reference's: a window matches pattern i iff its Rabin hash
// equals hash_full(pattern i) and its bytes equal the pattern.  Per length group, hashes
// are looked up in a table of the distinct low-32 keys whose entries point at the run of
// patterns sharing the key (several patterns may share a hash, e.g. "ac"/"ba",
// tests/test_matcher.py:139-146); the 64-bit hash (m > 24) and the bytes confirm.
//
// Which windows get that test is decided by a filter that never rejects a match:
//   * q-gram sampling (every length >= 7): anchors are the positions e with
//     e + 1 = 0 mod s.  Every occurrence of a pattern p at y contains exactly one anchored
//     q-gram: the q bytes ending at the first anchor e >= y + q - 1, which are p[j:j+q]
//     with j = e-q+1-y < s (so q + s - 1 <= m; (s, q) follow the group's shortest
//     length).  All such pattern q-grams go into a 64 KiB blocked Bloom filter (one
//     64-bit block, 4 bits, per q-gram) in shared memory; the fast pass tests one word-aligned q-gram per s bytes straight
//     from the loaded words (no rolling hash).  A q-gram that hits makes its s window
//     starts candidates; s lanes of the warp check them at once against every length
//     group (exact hash + table + bytes), and since each window has one anchor nothing
//     is reported twice.  (s, q) is chosen on the host from the lengths and the pattern
//     alphabet: q up to 16 bytes so that low-entropy texts (DNA: 4^q q-grams) still filter.
//   * m < 7 (one length per launch): the window is its own exact key, looked up in a cuckoo
//     table of the patterns in shared memory (rk_multi_tiny_kernel).
// Hits are appended with warp ballot/popc and one atomic per warp; the host orders them
// by (pattern index, offset), which is exactly the reference's per-pattern ascending lists.
#pragma once
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

#ifndef RK_MULTI_UNROLL
#define RK_MULTI_UNROLL false
#endif
constexpr int kMultiBlock = 32 * kMultiWarps;
using MultiRing = WarpRingT<kMultiStageChunks>;

__device__ __forceinline__ uint32_t mhash(uint32_t key) { return key * 0x9E3779B1u; }

__device__ __forceinline__ bool filter_test(const uint32_t* __restrict__ f, uint32_t L) {
  const uint32_t b = mhash(L) >> 16;
  return (f[b >> 5] >> (b & 31)) & 1u;
}

template <int QW>
__device__ __forceinline__ bool qfilter_test(const uint32_t* __restrict__ f, const uint32_t* w) {
  const uint32_t h = qgram_hash<QW>(w);
  const uint2 x = reinterpret_cast<const uint2*>(f)[h >> 19];
  // rotates take the position mod 32: four SHF and two LOP3, no masking
  const uint32_t r = __funnelshift_r(x.x, x.x, h) & __funnelshift_r(x.x, x.x, h >> 5) &
                     __funnelshift_r(x.y, x.y, h >> 10) & __funnelshift_r(x.y, x.y, h >> 15);
  return (r & 1u) != 0u;
}

// Anchored q-gram tests of one lane (window-end anchors e = J + s*t + s - 1, the q-gram
// being the QW words ending at e inside lb ++ v); bit t set when anchor t passes.
template <int S, int QW>
__device__ __forceinline__ uint32_t qgram_tests(const uint32_t* f, const Vec32& v,
                                                const uint32_t (&lb)[8]) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    w[i] = lb[i];
    w[8 + i] = v.w[i];
  }
  uint32_t qm = 0;
#pragma unroll
  for (int t = 0; t < 32 / S; ++t) {
    constexpr int kw = S / 4;              // words per step
    const int end_w = 8 + (t + 1) * kw;    // one past the q-gram's last word
    qm |= (uint32_t)qfilter_test<QW>(f, &w[end_w - QW]) << t;
  }
  return qm;
}

static __device__ __noinline__ uint64_t multi_hash_global(const uint8_t* text, uint32_t m,
                                                         int64_t je) {
  const int64_t span = m < 64 ? (int64_t)m : 64;
  uint64_t h = 0;
  for (int64_t i = je - span + 1; i <= je; ++i) h = (h << 1) + (uint64_t)text[i];
  return h;
}

// Caller's index of the pattern of group G that the window ending at text index je (low32
// hash L) matches, or -1.  Deduplicated patterns of one length are distinct, so at most
// one can byte-match.  (Fields by value: a reference into the kernel parameters would
// force them into local memory.)
static __device__ __noinline__ int multi_resolve(const uint8_t* text, const uint8_t* pats,
                                                 const uint64_t* phash, const uint32_t* order,
                                                 const uint32_t* gidx,
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
        if (eq) return (int)gidx[idx];
      }
      return -1;
    }
    slot = (slot + 1) & (tsize - 1);
  }
}

__device__ __forceinline__ int group_resolve(const MultiGroup& G, const uint8_t* text, uint32_t L,
                                             int64_t je) {
  return multi_resolve(text, G.pats, G.phash, G.order, G.gidx, G.table, G.tsize, G.m, L, je);
}

// Appends (window start, pattern) for the lanes with idx >= 0: one atomic per warp.
__device__ __forceinline__ void multi_append(const MultiArgs& a, int idx, int64_t y, int lane) {
  const unsigned hit = __ballot_sync(kFull, idx >= 0);
  if (hit) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)__popc(hit));
    base = __shfl_sync(kFull, base, 0);
    if (idx >= 0) {
      const uint64_t pos = base + __popc(hit & ((1u << lane) - 1u));
      if (pos < a.cap) {
        a.out_off[pos] = y;
        a.out_idx[pos] = (uint32_t)idx;
      }
    }
  }
}

// Length groups (bit i = grp[i]) with a pattern whose sampled q-grams include the one
// hashing to h: an open-addressing table {key, -, mask lo, mask hi} built with the filter.
__device__ __forceinline__ uint64_t qgram_groups(const MultiArgs& a, uint32_t h) {
  uint32_t slot = mhash(h) & (a.qmap_size - 1);
  for (;;) {
    const uint4 e = a.qmap[slot];
    if ((e.z | e.w) == 0u) return 0;  // empty: no pattern has this q-gram
    if (e.x == h) return ((uint64_t)e.w << 32) | e.z;
    slot = (slot + 1) & (a.qmap_size - 1);
  }
}

// Exact check of the window(s) starting at a-position ya against the length groups in
// gmask (lanes with active == false only take part in the warp collectives).
__device__ __forceinline__ void multi_check_window(const MultiArgs& a, int64_t ya, bool active,
                                                   int lane, uint64_t gmask) {
  const TextGeom& g = a.g;
  const uint8_t* text = g.abase + g.amis;
  const int64_t y = ya - (int64_t)g.amis;  // text index of the first byte
  for (; gmask; gmask &= gmask - 1) {
    const uint32_t gi = __ffsll((long long)gmask) - 1;
    const uint32_t m = a.grp[gi].m;
    int idx = -1;
    if (active && ya >= (int64_t)a.ys_lo && ya < (int64_t)a.grp[gi].ys_hi) {
      const int64_t je = y + (int64_t)m - 1;  // text index of the last byte
      const uint32_t span = m < 32 ? m : 32;  // low 32 bits of the hash: last <= 32 bytes
      uint32_t L = 0;
      for (uint32_t i = 0; i < span; ++i) L = 2u * L + text[je - span + 1 + i];
      if (filter_test(a.grp[gi].filter, L)) idx = group_resolve(a.grp[gi], text, L, je);
    }
    multi_append(a, idx, y, lane);
  }
}

// The SS windows of anchor e (their q-gram ends at e and passed the filter), checked by
// lanes 0..SS-1 against the length groups holding that q-gram.
template <int SS, int QW>
__device__ __forceinline__ void qgram_candidate(const MultiArgs& a, int64_t e, int lane) {
  constexpr int q = 4 * QW;
  if (e < (int64_t)a.g.ja_lo || e >= (int64_t)a.g.ja_hi) return;  // no window (uniform)
  // which length groups hold this q-gram (the filter only says "some pattern")
  uint64_t gmask = 1;
  if (a.G > 1) {
    const uint32_t* qw = reinterpret_cast<const uint32_t*>(a.g.abase + e - q + 1);
    uint32_t w[QW];
#pragma unroll
    for (int i = 0; i < QW; ++i) w[i] = qw[i];
    gmask = qgram_groups(a, qgram_hash<QW>(w));
  }
  // the window whose q-gram starts j = lane bytes in
  if (gmask) multi_check_window(a, e - q + 1 - lane, lane < SS, lane, gmask);
}

// One tile of anchored q-grams (one per SS bytes, ending at e = J + SS*t + SS - 1); a
// q-gram that passes the filter makes its SS windows candidates, checked by SS lanes at once.
template <int SS, int QW>
__device__ __forceinline__ void qgram_tile(const MultiArgs& a, MultiRing* R, Stream& S,
                                           uint32_t t, int lane, const uint32_t* sfilter) {
  constexpr int q = 4 * QW;
  // the anchored q-grams only reach into the 32 bytes before the lane's when a q-gram is
  // longer than the sampling step (QW words > SS / 4): otherwise skip loading them
  constexpr int kStreamM = QW > SS / 4 ? 31 : 0;
  stream_tile<kStreamM, RK_MULTI_UNROLL>(
      a.g, R, S, t, lane,
      [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t&, int64_t J, int) {
        const uint32_t qm = qgram_tests<SS, QW>(sfilter, v, lb);
        unsigned lanes = __ballot_sync(kFull, qm != 0);
        while (lanes) {
          const int src = __ffs(lanes) - 1;
          lanes &= lanes - 1;
          uint32_t ms = __shfl_sync(kFull, qm, src);
          const int64_t Js = __shfl_sync(kFull, J, src);
          while (ms) {
            const int tt = __ffs(ms) - 1;
            ms &= ms - 1;
            // the window whose anchor this is: its q-gram starts j = lane bytes in
            qgram_candidate<SS, QW>(a, Js + (int64_t)SS * tt + SS - 1, lane);
          }
        }
      });
}

// m < 7: a window is at most 6 bytes, so it is its own exact key.  The set's patterns sit
// in a cuckoo table in shared memory -- slot = key bytes | pattern index << 48, every
// key in one of its two slots -- so a window is looked up with two 8-byte loads and no
// loop or branch: the reference's "hash equal, then bytes equal" (matcher.py:147-153)
// collapses into one exact comparison, since a window of this length IS its hash input.
// (The rolling-hash filter of the longer lengths would pass most windows here: a 5-byte
// hash takes ~3000 values over printable ASCII.)
__device__ __forceinline__ unsigned long long ld_shared_u64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

// Blocked Bloom filter of the keys: 2048 blocks of 64 bits, 4 bits per key (2 per half),
// one LDS.64 per window; ~5e-5 false positives per window at 1024 patterns, so a group
// of 8 windows rarely leaves the fast path.
__device__ __forceinline__ uint32_t tiny_filter_test(uint32_t bitmap, uint32_t f) {
  unsigned long long x = ld_shared_u64(bitmap + 8 * (f >> kTinyFilterShift));
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const uint32_t p = f ^ (f >> 13);  // bit positions from mixed bits, each mod 32
  return __funnelshift_r(xl, xl, p) & __funnelshift_r(xl, xl, p >> 5) &
         __funnelshift_r(xh, xh, p >> 10) & __funnelshift_r(xh, xh, p >> 15) & 1u;
}

// The 32 windows go in four groups of 8: one filter probe each and one predicate per
// group; a group with a filter hit looks its passing windows up in the cuckoo table.
template <int M>
__device__ __forceinline__ void tiny_chunk(const MultiArgs& a, const Vec32& v,
                                           const uint32_t (&lb)[8], int64_t J, uint32_t vmask,
                                           uint32_t slots, uint32_t bitmap, const TinyHash& th) {
  constexpr uint32_t K0 = M >= 4 ? 0xffffffffu : ((1u << (8 * M)) - 1u);
  constexpr uint32_t K1 = M > 4 ? ((1u << (8 * (M - 4))) - 1u) : 0u;
#pragma unroll
  for (int grp = 0; grp < 4; ++grp) {
    uint32_t lo[8], hi[8], f[8], pass = 0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int s0 = 33 + grp * 8 + kk - M;  // first byte of the window, in lb ++ v
      lo[kk] = w64(lb, v, s0) & K0;
      hi[kk] = M > 4 ? (w64(lb, v, s0 + 4) & K1) : 0u;
      f[kk] = tiny_key_hash(lo[kk], hi[kk], th);
      pass |= tiny_filter_test(bitmap, f[kk]) << kk;
    }
    pass &= vmask >> (grp * 8);
    if (pass & 0xffu) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if ((pass >> kk) & 1u) {
          uint32_t s1, s2;
          tiny_slots(f[kk], th, s1, s2);
          const unsigned long long key = ((unsigned long long)hi[kk] << 32) | lo[kk];
          const unsigned long long e1 = ld_shared_u64(slots + 8 * s1) ^ key;
          const unsigned long long e2 = ld_shared_u64(slots + 8 * s2) ^ key;
          // a hit leaves only the index (< 2^12) in the top 16 bits; empty slots are ~0
          const bool h1 = (e1 & 0xffffffffffffull) == 0 && (e1 >> 48) < 0xffffull;
          const bool h2 = (e2 & 0xffffffffffffull) == 0 && (e2 >> 48) < 0xffffull;
          if (h1 || h2) {
            const unsigned long long pos = atomicAdd(&a.counters[0], 1ull);
            if (pos < a.cap) {
              a.out_off[pos] = J + grp * 8 + kk - M + 1 - (int64_t)a.g.amis;
              a.out_idx[pos] = (uint32_t)((h1 ? e1 : e2) >> 48);
            }
          }
        }
      }
    }
  }
}

// 8 bytes of the text at a-space position p (the bytes of a candidate window): from the
// TMA stage in shared memory when staged (cur = shared address of a-space position c0),
// else from global memory with bounds checks (edge tiles, the end of a chunk).
__device__ __forceinline__ uint2 tiny_window_bytes(const TextGeom& g, uint32_t cur, int64_t c0,
                                                   int64_t p) {
  // the stage holds the chunk's 32-byte lookback and its 1 KiB (a window may end up to 2
  // bytes past the chunk: those bytes are the next chunk's, which the stage only holds
  // when the chunk is not its last)
  if (cur && p - c0 + 12 <= 32 + kChunk) {
    const uint32_t addr = cur + (uint32_t)(p - c0);
    const uint32_t al = addr & ~3u, r = 8u * (addr & 3u);
    const uint32_t x0 = lds_u32(al), x1 = lds_u32(al + 4), x2 = lds_u32(al + 8);
    return make_uint2(__funnelshift_r(x0, x1, r), __funnelshift_r(x1, x2, r));
  }
  const int64_t lo = (int64_t)g.amis, hi = (int64_t)(g.amis + g.n);
  return make_uint2(edge_word(g.abase, lo, hi, p), edge_word(g.abase, lo, hi, p + 4));
}

// m in [kTinyAnchorFrom, 6]: one anchored q-gram per 2 bytes (anchors at odd lane offsets
// k, the q-gram being the q bytes ending at J + k) is tested against a blocked Bloom
// filter (2 bits in one 64-bit block, one LDS.64) of the patterns' anchored q-grams
// (p[0:q], p[1:q+1]; ~0.1% false positives at 1024 patterns); a passing anchor makes its two
// window starts (J + k - q + 1 - j, j = 0, 1) candidates, looked up exactly in the cuckoo
// table.  Each window has exactly one anchor, so nothing is reported twice.
template <int M>
__device__ __forceinline__ void tiny_anchor_chunk(const MultiArgs& a, const Vec32& v,
                                                  const uint32_t (&lb)[8], int64_t J,
                                                  uint32_t cur, int lane, uint32_t slots,
                                                  uint32_t bitmap, const TinyHash& th) {
  constexpr int Q = tiny_gram_q(M);
  constexpr uint32_t QK = Q >= 4 ? 0xffffffffu : ((1u << (8 * Q)) - 1u);
  constexpr uint32_t K0 = M >= 4 ? 0xffffffffu : ((1u << (8 * M)) - 1u);
  constexpr uint32_t K1 = M > 4 ? ((1u << (8 * (M - 4))) - 1u) : 0u;
  uint32_t pass = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int k = 2 * t + 1;  // the anchor is window end J + k
    const uint32_t h = (w64(lb, v, 33 + k - Q) & QK) * kGramMul;
    const unsigned long long x = ld_shared_u64(bitmap + 8u * (h >> 21));
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    pass |= (__funnelshift_r(xl, xl, h >> 16) & __funnelshift_r(xh, xh, h >> 11) & 1u) << t;
  }
  if (!pass) return;
  const int64_t c0 = J - kR * lane - 32;  // a-space position of the chunk's lookback start
  do {
    const int t = __ffs(pass) - 1;
    pass &= pass - 1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t ya = J + 2 * t + 2 - Q - j;  // candidate window start, a-space
      if (ya < (int64_t)a.ys_lo || ya >= (int64_t)a.grp[0].ys_hi) continue;
      const uint2 w = tiny_window_bytes(a.g, cur, c0, ya);
      const uint32_t lo = w.x & K0, hi = w.y & K1;
      const uint32_t f = tiny_key_hash(lo, hi, th);
      uint32_t s1, s2;
      tiny_slots(f, th, s1, s2);
      const unsigned long long key = ((unsigned long long)hi << 32) | lo;
      const unsigned long long e1 = ld_shared_u64(slots + 8 * s1) ^ key;
      const unsigned long long e2 = ld_shared_u64(slots + 8 * s2) ^ key;
      const bool h1 = (e1 & 0xffffffffffffull) == 0 && (e1 >> 48) < 0xffffull;
      const bool h2 = (e2 & 0xffffffffffffull) == 0 && (e2 >> 48) < 0xffffull;
      if (h1 || h2) {
        const unsigned long long pos = atomicAdd(&a.counters[0], 1ull);
        if (pos < a.cap) {
          a.out_off[pos] = ya - (int64_t)a.g.amis;
          a.out_idx[pos] = (uint32_t)((h1 ? e1 : e2) >> 48);
        }
      }
    }
  } while (pass);
}

template <int M>
__global__ void __launch_bounds__(kMultiBlock) rk_multi_tiny_kernel(const __grid_constant__ MultiArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  MultiRing* rings = reinterpret_cast<MultiRing*>(smem);
  uint8_t* tab = smem + sizeof(MultiRing) * kMultiWarps;
  const TinyHash th = a.grp[0].tiny_hash;
  const uint32_t n16 = (th.size * 8u + kTinyFilterBytes) / 16u;  // slots, then the filter
  const uint4* src = reinterpret_cast<const uint4*>(a.grp[0].tiny);
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(tab)[i] = src[i];
  __syncthreads();
  const uint32_t slots = smem_u32(tab);
  const uint32_t bitmap = slots + th.size * 8u;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  MultiRing* R = rings + warp;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * kMultiWarps;
  const uint64_t w = (uint64_t)blockIdx.x * kMultiWarps + warp;
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    const int64_t ta = a.g.tile_a(t);
    const bool full = ta >= (int64_t)a.g.ja_lo && ta + kTile <= (int64_t)a.g.ja_hi;
    stream_tile<M, false>(a.g, R, S, t, lane,
                          [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t&, int64_t J, int) {
                            if constexpr (M >= kTinyAnchorFrom) {
                              tiny_anchor_chunk<M>(a, v, lb, J, S.cur, lane, slots, bitmap, th);
                            } else {
                              tiny_chunk<M>(a, v, lb, J, full ? 0xffffffffu : valid_mask(a.g, J),
                                            slots, bitmap, th);
                            }
                          });
  }
}

template <class K>
int multi_occupancy(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kMultiBlock, smem);
  return b > 0 ? b : 1;
}

// (Attr is a per-kernel tag so each kernel opts in to > 48 KiB of smem once per device.)
template <class Attr, class K>
cudaError_t multi_launch_kernel(K kernel, const MultiArgs& a, int grid, size_t smem,
                                cudaStream_t s) {
  static bool attr[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDevices) attr[dev] = true;
  }
  kernel<<<grid, kMultiBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rkb
