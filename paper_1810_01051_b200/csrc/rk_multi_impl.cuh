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
//   * m < 7 (lengths 4..6 in one sweep, 1..3 in another): the window is its own exact key,
//     looked up in a cuckoo table of the patterns in shared memory (rk_multi_short_kernel).
// Hits are appended with warp ballot/popc and one atomic per warp; the host orders them
// by (pattern index, offset), which is exactly the reference's per-pattern ascending lists.
#pragma once
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

#ifndef RK_MULTI_UNROLL
#define RK_MULTI_UNROLL false
#endif
#ifndef RK_MULTI_STAGED_TESTS
#define RK_MULTI_STAGED_TESTS 1  // q-gram tests unrolled per TMA stage, candidates afterwards
#endif
constexpr int kMultiBlock = 32 * kMultiWarps;
using MultiRing = WarpRingT<kMultiStageChunks>;

__device__ __forceinline__ uint32_t mhash(uint32_t key) { return key * 0x9E3779B1u; }

__device__ __forceinline__ bool filter_test(const uint32_t* __restrict__ f, uint32_t L) {
  const uint32_t b = mhash(L) >> 16;
  return (f[b >> 5] >> (b & 31)) & 1u;
}

// F32: the filter's layout -- one 32-bit word per q-gram with three bits (one LDS.32),
// or one 64-bit block with four (one LDS.64; fewer false positives).  The host picks per
// sweep (MultiPlan::Sweep::qf32): measured C3 (one length) 5245 GB/s with 64-bit blocks
// against 5080 with words, 64 mixed lengths 3626 against 4000.
template <int QW, bool F32>
__device__ __forceinline__ bool qfilter_test(const uint32_t* __restrict__ f, const uint32_t* w) {
  const uint32_t h = qgram_hash<QW>(w);
  if constexpr (F32) {
    const uint32_t x = f[h >> kQWordShift];
    return (__funnelshift_r(x, x, h) & __funnelshift_r(x, x, h >> 5) &
            __funnelshift_r(x, x, h >> 10) & 1u) != 0u;
  } else {
    const uint2 x = reinterpret_cast<const uint2*>(f)[h >> kQBlockShift];
    // rotates take the position mod 32: four SHF and two LOP3, no masking
    const uint32_t r = __funnelshift_r(x.x, x.x, h) & __funnelshift_r(x.x, x.x, h >> 5) &
                       __funnelshift_r(x.y, x.y, h >> 10) & __funnelshift_r(x.y, x.y, h >> 15);
    return (r & 1u) != 0u;
  }
}

// Anchored q-gram tests of one lane (window-end anchors e = J + s*t + s - 1, the q-gram
// being the QW words ending at e inside lb ++ v); bit t set when anchor t passes.
template <int S, int QW, bool F32>
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
    qm |= (uint32_t)qfilter_test<QW, F32>(f, &w[end_w - QW]) << t;
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
// This warp's append buffer (after the kernel's rings): a count, then append_cap offsets
// and append_cap indices.
__device__ __forceinline__ uint8_t* append_buf(const MultiArgs& a) {
  extern __shared__ __align__(16) uint8_t smem_dyn[];
  return smem_dyn + sizeof(MultiRing) * kMultiWarps +
         (threadIdx.x >> 5) * multi_append_stride(a.append_cap);
}

__device__ __forceinline__ void multi_append_init(const MultiArgs& a, int lane) {
  if (a.append_cap && lane == 0) *reinterpret_cast<uint32_t*>(append_buf(a)) = 0u;
  __syncwarp();
}

// Writes the warp's buffered pairs out: one atomic reserves their slots, then coalesced
// stores (warp-uniform call).
__device__ __forceinline__ void multi_flush(const MultiArgs& a, int lane) {
  if (!a.append_cap) return;
  uint8_t* b = append_buf(a);
  __syncwarp();
  const uint32_t n = *reinterpret_cast<volatile uint32_t*>(b);
  if (!n) return;
  const int64_t* boff = reinterpret_cast<const int64_t*>(b + 16);
  const uint32_t* bidx = reinterpret_cast<const uint32_t*>(b + 16 + 8u * a.append_cap);
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)n);
  base = __shfl_sync(kFull, base, 0);
  for (uint32_t i = lane; i < n; i += 32) {
    const uint64_t pos = base + i;
    if (pos < a.cap) {
      a.out_off[pos] = boff[i] + a.out_bias;
      a.out_idx[pos] = bidx[i];
    }
  }
  __syncwarp();
  if (lane == 0) *reinterpret_cast<uint32_t*>(b) = 0u;
  __syncwarp();
}

// Appends the lanes' pairs (idx >= 0) -- warp-uniform call -- with one atomic per warp per
// round, or (Buffered) into the warp's shared-memory buffer, flushed with one atomic per
// append_cap pairs: dense output (all 'a' against {aaaa, aaaaa, aaaaaa}) made one atomic
// per round serialise on one address.  The buffered path is out of line: inlined into the
// fast pass it cost registers (spills) in the sparse common case.
static __device__ __noinline__ void multi_append_buffered(const MultiArgs& a, int idx, int64_t y,
                                                   int lane, unsigned hit) {
  const uint32_t k = __popc(hit);
  const uint32_t rank = __popc(hit & ((1u << lane) - 1u));
  uint8_t* b = append_buf(a);
  uint32_t n = *reinterpret_cast<volatile uint32_t*>(b);
  if (n + k > a.append_cap) {
    multi_flush(a, lane);
    n = 0;
  }
  if (idx >= 0) {
    reinterpret_cast<int64_t*>(b + 16)[n + rank] = y;
    reinterpret_cast<uint32_t*>(b + 16 + 8u * a.append_cap)[n + rank] = (uint32_t)idx;
  }
  __syncwarp();
  if (lane == 0) *reinterpret_cast<uint32_t*>(b) = n + k;
  __syncwarp();
}

template <bool Buffered = false>
__device__ __forceinline__ void multi_append(const MultiArgs& a, int idx, int64_t y, int lane) {
  const unsigned hit = __ballot_sync(kFull, idx >= 0);
  if (!hit) return;
  if (Buffered && a.append_cap) {
    multi_append_buffered(a, idx, y, lane, hit);
    return;
  }
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&a.counters[0], (unsigned long long)__popc(hit));
  base = __shfl_sync(kFull, base, 0);
  if (idx >= 0) {
    const uint64_t pos = base + __popc(hit & ((1u << lane) - 1u));
    if (pos < a.cap) {
      a.out_off[pos] = y + a.out_bias;
      a.out_idx[pos] = (uint32_t)idx;
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

// The candidates of one chunk (qm = the lane's passing anchors, J = its first position):
// each anchor's SS windows are checked by SS lanes at once (warp-uniform call).
template <int SS, int QW>
__device__ __forceinline__ void qgram_settle(const MultiArgs& a, uint32_t qm, int64_t J, int lane) {
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
}

// One tile of anchored q-grams (one per SS bytes, ending at e = J + SS*t + SS - 1); a
// q-gram that passes the filter makes its SS windows candidates, checked by SS lanes at
// once.  Staged tiles run each TMA stage's chunks through the filter tests unrolled, with
// nothing else in that code, and settle the (rare) candidates after the stage's tests.
template <int SS, int QW, bool F32>
__device__ __forceinline__ void qgram_tile(const MultiArgs& a, MultiRing* R, Stream& S,
                                           uint32_t t, int lane, const uint32_t* sfilter) {
  // the anchored q-grams only reach into the 32 bytes before the lane's when a q-gram is
  // longer than the sampling step (QW words > SS / 4): otherwise skip loading them
  constexpr int kStreamM = QW > SS / 4 ? 31 : 0;
  constexpr int SC = kMultiStageChunks;
  const TextGeom& g = a.g;
  const int64_t ta = g.tile_a(t);
#if RK_MULTI_STAGED_TESTS
  if (t >= S.int_lo && t < S.int_hi) {
#pragma unroll 1
    for (int s = 0; s < kTileChunks / SC; ++s) {
      mbar_wait(&R->bar[S.cslot], S.cphase);
      const uint8_t* st = R->buf[S.cslot];
      uint32_t qm[SC], anyq = 0;
#pragma unroll
      for (int j = 0; j < SC; ++j) {
        const Vec32 v = lds32(st + 32 + j * kChunk + lane * kR);
        uint32_t lb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if constexpr (kStreamM > 0) {
          const Vec32 l = lds32(st + j * kChunk + lane * kR);
#pragma unroll
          for (int i = 0; i < 8; ++i) lb[i] = l.w[i];
        }
        qm[j] = qgram_tests<SS, QW, F32>(sfilter, v, lb);
        anyq |= qm[j];
      }
      if (__any_sync(kFull, anyq != 0)) {
#pragma unroll 1
        for (int j = 0; j < SC; ++j) {
          uint32_t q = qm[0];
#pragma unroll
          for (int jj = 1; jj < SC; ++jj) q = j == jj ? qm[jj] : q;
          qgram_settle<SS, QW>(a, q, ta + (int64_t)(s * SC + j) * kChunk + lane * kR, lane);
        }
      }
      // the slot's bytes are consumed: hand it back to the producer
      S.cslot = (S.cslot + 1) & (kStages - 1);
      S.cphase ^= (S.cslot == 0);
      --S.pending;
      __syncwarp();
      stream_issue(R, S, lane);
    }
    return;
  }
#endif
  stream_tile<kStreamM, RK_MULTI_UNROLL>(
      g, R, S, t, lane,
      [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t&, int64_t J, int) {
        qgram_settle<SS, QW>(a, qgram_tests<SS, QW, F32>(sfilter, v, lb), J, lane);
      });
}

// ---------------------------------------------------------------------------------
// Lengths < 7: a window of length L <= 6 is its own exact key, so the reference's
// "hash equal, then bytes equal" (matcher.py:147-153) collapses into one exact lookup of
// (bytes, L) in the sweep's cuckoo table in shared memory (two 8-byte loads, no loop).
// (The rolling-hash filter of the longer lengths would pass most windows here: a 5-byte
// hash takes ~3000 values over printable ASCII.)  Which windows are looked up:
//   * anchored sweep (every length of the set in 4..6): one q-gram per 2 bytes (anchors
//     at odd lane offsets k, the q-gram being the q bytes ending at J + k) is tested
//     against the sweep's Bloom filter of the patterns' anchored q-grams; a passing anchor
//     makes its two window starts candidates for every length of the sweep.  Each window
//     has exactly one anchor, so nothing is reported twice.
//   * per-window sweep (lengths 1..3): every window end, for every length, tests its key
//     against the filter of the patterns' keys.
// The fast pass only builds each lane's pass mask; candidates are then settled in warp
// rounds -- every lane with a pending candidate takes its next one -- and appended with
// one ballot and ONE atomic per warp per round (multi_append), so dense output (all 'a'
// against {aaaa, aaaaa, aaaaaa}) costs a warp-wide append per round, not an atomic per
// match.
__device__ __forceinline__ unsigned long long ld_shared_u64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

// 1 iff the entry x's three bits are set in the sweep's filter (rk_internal.h)
template <int Q>
__device__ __forceinline__ uint32_t short_filter_test(uint32_t filt, uint32_t x) {
  const uint32_t h = short_filter_hash(x);
  const uint32_t w = lds_u32(filt + 4u * short_filter_word(h));
  // rotates take the bit positions mod 32
  if constexpr (short_filter_bits(Q) == 3) {
    return __funnelshift_r(w, w, h) & __funnelshift_r(w, w, h >> 5) &
           __funnelshift_r(w, w, h >> 10) & 1u;
  } else {
    return __funnelshift_r(w, w, h) & __funnelshift_r(w, w, h >> 5) & 1u;
  }
  // (one rotate with the other bits at fixed distances from h mod 32 tests in fewer
  // instructions, but the bits are then one 5-bit choice: ~1% false positives, 1024 x
  // m = 4 2.40 -> 3.76 ms)
}

// 8 bytes of the text at a-space position p (the bytes of a candidate window): from the
// TMA stage in shared memory when staged (cur = shared address of a-space position c0),
// else from global memory with bounds checks (edge tiles, the end of a stage).
__device__ __forceinline__ uint2 short_window_bytes(const TextGeom& g, uint32_t cur, int64_t c0,
                                                    int64_t p, uint32_t stage_bytes) {
  if (cur && p >= c0 && p - c0 + 12 <= (int64_t)stage_bytes) {
    const uint32_t addr = cur + (uint32_t)(p - c0);
    const uint32_t al = addr & ~3u, r = 8u * (addr & 3u);
    const uint32_t x0 = lds_u32(al), x1 = lds_u32(al + 4), x2 = lds_u32(al + 8);
    return make_uint2(__funnelshift_r(x0, x1, r), __funnelshift_r(x1, x2, r));
  }
  const int64_t lo = (int64_t)g.amis, hi = (int64_t)(g.amis + g.n);
  return make_uint2(edge_word(g.abase, lo, hi, p), edge_word(g.abase, lo, hi, p + 4));
}

// Caller's index of the pattern (lo, hb, L) -- a window's bytes, masked to its length --
// in the sweep's cuckoo table, or -1.
__device__ __forceinline__ int short_probe(const MultiArgs& a, uint32_t slots, uint32_t lo,
                                           uint32_t hb, uint32_t L) {
  const uint32_t tag = short_tag(hb, L);  // = the key's high word
  const uint32_t f = tiny_key_hash(lo, tag, a.th);
  uint32_t s1, s2;
  tiny_slots(f, a.th, s1, s2);
  const unsigned long long key = ((unsigned long long)tag << 32) | lo;
  const unsigned long long e1 = ld_shared_u64(slots + 8 * s1);
  const unsigned long long e2 = ld_shared_u64(slots + 8 * s2);
  // a hit leaves only the index bits; empty slots (~0) have the top bit set
  if (((e1 ^ key) & kShortKeyMask) == 0 && !(e1 >> 63)) return (int)((e1 >> 51) & 0xfffu);
  if (((e2 ^ key) & kShortKeyMask) == 0 && !(e2 >> 63)) return (int)((e2 >> 51) & 0xfffu);
  return -1;
}

// Caller's index of the pattern of length L equal to the window at a-space ya, or -1.
__device__ __forceinline__ int short_lookup(const MultiArgs& a, uint32_t slots, uint32_t cur,
                                            int64_t c0, uint32_t stage_bytes, int64_t ya,
                                            uint32_t L, uint64_t ys_hi) {
  if (ya < (int64_t)a.ys_lo || ya >= (int64_t)ys_hi) return -1;
  const uint2 w = short_window_bytes(a.g, cur, c0, ya, stage_bytes);
  const uint32_t lo = L >= 4 ? w.x : (w.x & ((1u << (8 * L)) - 1u));
  const uint32_t hb = L > 4 ? (w.y & ((1u << (8 * (L - 4))) - 1u)) : 0u;
  return short_probe(a, slots, lo, hb, L);
}

// One chunk: the lane's 32 positions end at J (a-space); v = its 32 bytes, lb the 32
// before; cur = shared address of the chunk's 32-byte lookback (0: edge tile, global).
// The sweep's lengths (<= 3 of them: 4..6 or 1..3) and their byte masks, kept in registers.
struct ShortLens {
  uint32_t G, L[3], klo[3], khi[3];
  __device__ explicit ShortLens(const MultiArgs& a) : G(a.G) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      L[i] = i < (int)G ? a.grp[i].m : 0u;
      klo[i] = L[i] >= 4 ? 0xffffffffu : ((1u << (8 * L[i])) - 1u);
      khi[i] = L[i] > 4 ? ((1u << (8 * (L[i] - 4))) - 1u) : 0u;
    }
  }
};

// Anchored sweep, fast pass of one chunk: bit t = the q-gram ending at J + 2t + 1 passed.
template <int Q>
__device__ __forceinline__ uint32_t short_anchor_pass(uint32_t filt, const Vec32& v,
                                                      const uint32_t (&lb)[8]) {
  constexpr uint32_t QK = Q >= 4 ? 0xffffffffu : ((1u << (8 * Q)) - 1u);
  uint32_t pass = 0;
#pragma unroll
  for (int t = 15; t >= 0; --t) {  // pass = 2 pass + bit: one IMAD, bit t = anchor t
    const int k = 2 * t + 1;
    pass = pass * 2u + short_filter_test<Q>(filt, w64(lb, v, 33 + k - Q) & QK);
  }
  if constexpr (short_refined(Q)) {
    // 3-gram sweeps: the text's 3-grams equal the patterns' for real at ~1/400 anchors, so
    // a passing anchor's two windows are first tested on their 4-byte prefixes (the same
    // filter also holds every pattern's first 4 bytes, salted): ~1/1000 of them go on to
    // the warp-round settle.  For q = 3 the prefix of window y0 of the last anchor ends
    // one byte past this lane's 32: the next lane's first byte (lane 31: kept untested).
    if (__any_sync(kFull, pass != 0)) {
      const uint32_t nxt = __shfl_down_sync(kFull, v.w[0], 1);
      const int lane = threadIdx.x & 31;
      uint32_t keep = 0;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        if (!((pass >> t) & 1u)) continue;
        const int k = 2 * t + 1;
        // window y0 - 1 starts at byte 32 + k - Q of (lb, v), window y0 one byte later
        uint32_t ok = short_filter_test<Q>(filt, w64(lb, v, 32 + k - Q) ^ kShortKeySalt);
        if (36 + k - Q <= 63) {
          ok |= short_filter_test<Q>(filt, w64(lb, v, 33 + k - Q) ^ kShortKeySalt);
        } else {  // Q = 3, the last anchor: bytes 61..63 and the next lane's first
          ok |= lane == 31 ? 1u
                           : short_filter_test<Q>(filt, __funnelshift_r(v.w[7], nxt, 8) ^ kShortKeySalt);
        }
        keep |= ok << t;
      }
      pass = keep;
    }
  }
  return pass;
}

// Anchored sweep: the candidates of one chunk (each lane's passing anchors), settled in warp
// rounds (warp-uniform call).
template <int Q>
__device__ __forceinline__ void short_anchor_candidates(const MultiArgs& a, const ShortLens& SL,
                                                        uint32_t pass, int64_t J, uint32_t cur,
                                                        int lane, uint32_t slots,
                                                        uint32_t stage_bytes) {
  const int64_t c0 = J - kR * lane - 32;  // a-space position of the chunk's lookback start
  unsigned act = __ballot_sync(kFull, pass != 0);
  if (!act) return;
  // every candidate window of the chunk lies in the text and in the stage (most chunks):
  // lookups straight from shared memory without per-window checks
  const int64_t ys_hi_min = (int64_t)a.grp[a.G - 1].ys_hi;  // the longest length's
  const bool easy = __all_sync(kFull, cur != 0) && c0 >= (int64_t)a.ys_lo &&
                    c0 + 32 + kChunk <= ys_hi_min && 32u + kChunk + 16u <= stage_bytes;
  while (act) {
    int t = -1;
    if (pass) {
      t = __ffs(pass) - 1;
      pass &= pass - 1;
    }
    const int64_t y0 = J + 2 * t + 2 - Q;  // the anchor's window starts: y0 and y0 - 1
    if (easy) {
      // bytes [y0 - 1, y0 + 7) in shared memory, as the words of each start
      uint32_t lo1 = 0, hi1 = 0, lo0 = 0, hi0 = 0;
      if (t >= 0) {
        const uint32_t addr = cur + (uint32_t)(y0 - 1 - c0);
        const uint32_t al = addr & ~3u, r = 8u * (addr & 3u);
        const uint32_t x0 = lds_u32(al), x1 = lds_u32(al + 4), x2 = lds_u32(al + 8);
        lo1 = __funnelshift_r(x0, x1, r);
        hi1 = __funnelshift_r(x1, x2, r);
        lo0 = __funnelshift_r(lo1, hi1, 8);
        hi0 = __funnelshift_r(hi1, x2 >> r, 8);
      }
#pragma unroll
      for (int gi = 0; gi < 3; ++gi) {
        if (gi >= (int)SL.G) break;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          int idx = -1;
          if (t >= 0) {
            const uint32_t lo = j ? lo1 : lo0, hw = j ? hi1 : hi0;
            idx = short_probe(a, slots, lo & SL.klo[gi], hw & SL.khi[gi], SL.L[gi]);
          }
          multi_append<true>(a, idx, y0 - j - (int64_t)a.g.amis, lane);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t ya = y0 - j;  // candidate window start, a-space
        for (uint32_t gi = 0; gi < a.G; ++gi) {
          const int idx = t >= 0 ? short_lookup(a, slots, cur, c0, stage_bytes, ya,
                                                a.grp[gi].m, a.grp[gi].ys_hi)
                                 : -1;
          multi_append<true>(a, idx, ya - (int64_t)a.g.amis, lane);
        }
      }
    }
    act = __ballot_sync(kFull, pass != 0);
  }
}

template <int Q>
__device__ __forceinline__ void short_chunk_multi(const MultiArgs& a, const ShortLens& SL,
                                                  const Vec32& v, const uint32_t (&lb)[8],
                                                  int64_t J, uint32_t cur, int lane,
                                                  uint32_t slots, uint32_t filt,
                                                  uint32_t stage_bytes) {
  if constexpr (Q > 0) {
    short_anchor_candidates<Q>(a, SL, short_anchor_pass<Q>(filt, v, lb), J, cur, lane, slots,
                               stage_bytes);
  } else {
    const int64_t c0 = J - kR * lane - 32;  // a-space position of the chunk's lookback start
    // per window end J + k and length L (<= 3): the key's filter test
    for (uint32_t gi = 0; gi < a.G; ++gi) {
      const uint32_t L = a.grp[gi].m;
      const uint32_t K = (1u << (8 * L)) - 1u;
      uint32_t pass = 0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        // the L bytes ending at J + k are the top L bytes of the word ending there
        const uint32_t kb = (w64(lb, v, 29 + k) >> (8 * (4 - L))) & K;
        pass = pass * 2u + short_filter_test<0>(filt, tiny_key_hash(kb, short_tag(0u, L), a.th));
      }
      unsigned act = __ballot_sync(kFull, pass != 0);
      while (act) {
        int k = -1;
        if (pass) {
          k = __ffs(pass) - 1;
          pass &= pass - 1;
        }
        const int64_t ya = J + k - (int64_t)L + 1;
        const int idx =
            k >= 0 ? short_lookup(a, slots, cur, c0, stage_bytes, ya, L, a.grp[gi].ys_hi) : -1;
        multi_append<true>(a, idx, ya - (int64_t)a.g.amis, lane);
        act = __ballot_sync(kFull, pass != 0);
      }
    }
  }
}

// Q = anchored q-gram length (3 or 4), 0 = per-window keys.
template <int Q>
__global__ void __launch_bounds__(kMultiBlock) rk_multi_short_kernel(const __grid_constant__ MultiArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  MultiRing* rings = reinterpret_cast<MultiRing*>(smem);
  uint8_t* tab = smem + sizeof(MultiRing) * kMultiWarps + kMultiWarps * multi_append_stride(a.append_cap);
  const uint32_t n16 = (a.th.size * 8u + kShortFilterWords * 4u) / 16u;  // slots, then filter
  const uint4* src = reinterpret_cast<const uint4*>(a.stab);
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<uint4*>(tab)[i] = src[i];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  multi_append_init(a, lane);
  __syncthreads();
  const uint32_t slots = smem_u32(tab);
  const uint32_t filt = slots + a.th.size * 8u;

  MultiRing* R = rings + warp;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * kMultiWarps;
  const uint64_t w = (uint64_t)blockIdx.x * kMultiWarps + warp;
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  const ShortLens SL(a);
  // (the staged structure that speeds up the q-gram kernel -- all of a stage's filter tests
  // first, then the candidates -- measured slower here: 1024 x m = 5 2079 -> 1968 GB/s,
  // m = 4 1510 -> 1333; this kernel's candidates are ~1 per KiB, not ~0.03)
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    stream_tile<8, false>(a.g, R, S, t, lane,
                          [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t&, int64_t J, int c) {
                            // the stage holds the chunk's lookback, itself and the rest of
                            // the stage's chunks
                            const uint32_t sb =
                                32u + (uint32_t)(kMultiStageChunks - c % kMultiStageChunks) * kChunk;
                            short_chunk_multi<Q>(a, SL, v, lb, J, S.cur, lane, slots, filt, sb);
                          });
  }
  multi_flush(a, lane);
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
