// rk_scan_impl.cuh -- single-pattern exact scan for sm_100a (the reference's _scan_range,
// /root/reference/pkg/src/rkmatch/_scan.py:28-50, and the range partition + ordered merge
// of search_parallel, parallel.py:155-172):
//
//   TMA bulk copies (4 KiB stages, 2 per warp) -> shared memory
//     -> per window, the low 32 bits of its hash, by the cheapest exact form for m:
//        m <= 8 dot products (hits settled inline), 9..14 the exact roll, 15..31 the
//        32-byte fold as a filter mod 2^m, m >= 32 the fold itself
//     -> candidate chunks: exact 32/64-bit hash + byte verify -> match / collision counts
//     -> per-tile match count + hit masks (global), consumed by rk_emit.cu, which
//        writes the ordered int64 window starts.
//
// The scan kernel never waits on another warp, and reads the text from HBM once.
#pragma once
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

// Warp-cooperative exact checks of one candidate window (all 32 lanes call them with the
// same arguments): the bytes are read in parallel, lane l taking bytes l, l+32, ...,
// instead of one lane walking up to m bytes with a dependent load per byte.

// 64-bit hash of the window whose last byte is at text index je: sum over its last
// min(m, 64) bytes of b * 2^(je - pos), mod 2^64.
__device__ __forceinline__ uint64_t warp_hash64(const uint8_t* text, uint32_t m, int64_t je,
                                                int lane) {
  const int span = m < 64 ? (int)m : 64;
  uint64_t h = 0;
  for (int d = lane; d < span; d += 32) h += (uint64_t)text[je - d] << d;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(kFull, h, o);
  return h;
}

__device__ __forceinline__ bool warp_equal(const uint8_t* text, const uint8_t* pattern,
                                           uint32_t m, int lane) {
  bool eq = true;
  for (uint32_t i = lane; i < m; i += 32) eq &= (text[i] == pattern[i]);
  return __all_sync(kFull, eq);
}


struct SlowOut {
  uint32_t hm;    // hit bits (window end = J + k)
  uint32_t hits;  // hash hits (matches + collisions)
};

// Slow pass over one chunk that had a candidate: exact per-window decisions.  The lane's
// 32 bytes and the 32 before them come from the TMA stage in shared memory when the chunk
// is still staged (sp = its address, lookback first), else from global memory
// (L2-resident: the chunk was just streamed).
template <int M>
__device__ __forceinline__ SlowOut slow_chunk(const ScanArgs& a, int64_t J,
                                              const uint8_t* sp = nullptr) {
  const TextGeom& g = a.g;
  SlowOut r{0u, 0u};
  const Vec32 v = sp ? lds32(sp + 32) : load_edge(g, J);
  const Vec32 lbv = sp ? lds32(sp) : load_edge(g, J - 32);
  const uint32_t T = (uint32_t)a.hx;
  if constexpr (M >= 32) {
    // the lane's 32 low-32 hashes first (one dependent IMAD each, no vote inside the
    // chain), then the candidates one at a time, each checked by the whole warp
    const uint8_t* text = g.abase + g.amis;
    const int lane = threadIdx.x & 31;
    uint32_t S = fold32(lbv.w);
    uint32_t cm = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      S = 2u * S + bsel(v.w[k >> 2], k & 3);
      if (S == T) cm |= 1u << k;
    }
    cm &= valid_mask(g, J);
    unsigned lanes = __ballot_sync(kFull, cm != 0);
    while (lanes) {
      const int src = __ffs(lanes) - 1;
      lanes &= lanes - 1;
      uint32_t bits = __shfl_sync(kFull, cm, src);
      const int64_t Js = __shfl_sync(kFull, J, src) - (int64_t)g.amis;
      while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        const int64_t je = Js + k;  // text index of the window's last byte
        if (warp_hash64(text, g.m, je, lane) == a.hx) {
          const bool eq = warp_equal(text + je - (int64_t)g.m + 1, a.pattern, g.m, lane);
          if (lane == src) {
            ++r.hits;
            if (eq) r.hm |= 1u << k;
          }
        }
      }
    }
  } else {
    uint32_t L = fold_tail<M>(lbv.w);
    uint32_t cm = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int io = 32 + k - M;
      const uint32_t in = bsel(v.w[k >> 2], k & 3);
      const uint32_t out =
          io < 32 ? bsel(lbv.w[io >> 2], io & 3) : bsel(v.w[(io - 32) >> 2], io & 3);
      L = 2u * L + in - (out << M);
      if (L == T) cm |= 1u << k;
    }
    cm &= valid_mask(g, J);
    // the lane's candidates, one at a time from L1/L2 (rare: kept out of the unrolled code)
    const uint8_t* text = g.abase + g.amis;
    while (cm) {
      const int k = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint8_t* w = text + (J + k - (int64_t)g.amis) - M + 1;  // window start
      bool hit = true;
      if constexpr (M > 24) {  // low 32 bits agree; confirm the whole hash
        uint64_t h = 0;
        for (int i = 0; i < M; ++i) h = (h << 1) + w[i];
        hit = (h == a.hx);
      }
      if (hit) {
        ++r.hits;
        bool eq = true;
        for (int i = 0; i < M; ++i) eq &= (w[i] == a.pattern[i]);
        if (eq) r.hm |= 1u << k;
      }
    }
  }
  return r;
}

// ---------------------------------------------------------------------------------
// Short patterns (M <= 8) have frequent exact-hash hits on small alphabets (m = 4 over
// printable ASCII: ~1.2e-3 per window, most 1 KiB chunks), so their candidates are
// settled inside the fast pass while the bytes are still in registers (short_chunk).
// No chunk is re-read.

// Patterns shorter than this settle candidates inline (see short_chunk).
constexpr int kShortInline = 9;
#ifndef RK_ROLL_UNROLL
#define RK_ROLL_UNROLL false  // 9 <= m <= 14: the exact-roll chunk loop unrolled per stage
#endif
// From this length on, M < 32 filters with the 32-byte fold (see rk_scan_kernel): one
// false positive per 2^M windows sends ~1 KiB/2^(M-10) of chunks to the exact pass, which
// beats the exact roll from M = 15 (measured: m = 20 4.74 vs 4.27 TB/s, m = 15 4.54 vs 4.3,
// m = 14 4.27 vs 4.3).
constexpr int kFoldFilter = 15;
#ifndef RK_FOLD_FMA_BYTES
#define RK_FOLD_FMA_BYTES 0
#endif
constexpr bool kFoldFmaBytes = RK_FOLD_FMA_BYTES;

// M <= 8: the whole hash of a window is a dot product of its (at most two) words with
// the weights 2^(M-1-i), so there is no serial roll chain: per window one funnel shift
// (shared between neighbours) and one or two dp4a that also subtract hx, giving
// d = hash - hx directly.  The 32 positions go in four groups of 8 with one predicate
// each: M <= 4 tests half the group as a product of the d's (zero iff some factor is
// zero, or -- harmlessly -- when 2-adic factors pile up to 2^32: the group is then just
// settled needlessly) so the FMA pipe carries what the ALU pipe would otherwise queue.
// A group that fired (m = 4 over printable ASCII: ~26% of warp-groups) settles from the
// d's and words still in registers: hash hits are counted, and only when some window's
// bytes equal the pattern (or the tile is at the edge of the range) are the hit and
// byte masks built.
template <int M, bool Dense = false>
__device__ __forceinline__ void short_chunk(const ScanArgs& a, const Vec32& v,
                                            const uint32_t (&lb)[8], bool full, uint32_t vmask,
                                            uint32_t& hm, uint32_t& hits) {
  static_assert(M <= 8, "dot-product hashes need M <= 8");
  if constexpr (M == 1) {
    // the hash of a 1-byte window is the byte: four windows per SIMD byte compare, and
    // a hash hit is a match iff hx is the pattern's own hash (hx is a parameter)
    if (a.hx > 255u) return;  // no byte hashes to hx
    const uint32_t splat = (uint32_t)a.hx * 0x01010101u;
    uint32_t hmask = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t eq = __vcmpeq4(v.w[i], splat) & 0x80808080u;
      hmask |= ((eq * 0x00204081u) >> 28) << (4 * i);  // byte MSBs -> 4 window bits
    }
    hmask &= vmask;
    hits += __popc(hmask);
    if (a.hx == (a.pw.w[0] & 0xffu)) hm |= hmask;
    (void)full;
    (void)lb;
    return;
  }
  const uint32_t negT = 0u - (uint32_t)a.hx;
  constexpr uint32_t W0 = win_weights<M>(0), W1 = win_weights<M>(1);
  constexpr uint32_t K0 = M >= 4 ? 0xffffffffu : ((1u << (8 * M)) - 1u);
  constexpr uint32_t K1 = M >= 8 ? 0xffffffffu : M > 4 ? ((1u << (8 * (M - 4))) - 1u) : 0u;
#pragma unroll
  for (int grp = 0; grp < 4; ++grp) {
    uint32_t wA[8], wB[8], d[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int s0 = 33 + grp * 8 + kk - M;
      wA[kk] = w64(lb, v, s0);
      if constexpr (M > 4) {
        wB[kk] = w64(lb, v, s0 + 4);
        d[kk] = __dp4a(wA[kk], W0, __dp4a(wB[kk], W1, negT));
      } else {
        d[kk] = __dp4a(wA[kk], W0, negT);
      }
    }
    bool anyg;
    if constexpr (M <= 4) {
      const uint32_t p = d[0] * d[1] * d[2] * d[3];
      anyg = (p == 0u) | (d[4] == 0u) | (d[5] == 0u) | (d[6] == 0u) | (d[7] == 0u);
    } else {
      anyg = false;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) anyg |= (d[kk] == 0u);
    }
    if (anyg) {
      // Dense (the warp's previous tile was mostly matches, e.g. all 'a'): when the whole
      // group hits and matches -- the OR of its 8 d's and byte differences is 0 -- take
      // it at once
      if (Dense && full) {
        uint32_t dor = 0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          dor |= d[kk] | ((wA[kk] ^ a.pw.w[0]) & K0);
          if constexpr (M > 4) dor |= (wB[kk] ^ a.pw.w[1]) & K1;
        }
        if (dor == 0u) {
          hits += 8;
          hm |= 0xffu << (grp * 8);
          continue;
        }
      }
      bool anyeq = false;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t x = (wA[kk] ^ a.pw.w[0]) & K0;
        if constexpr (M > 4) x |= (wB[kk] ^ a.pw.w[1]) & K1;
        anyeq |= (x == 0u);
      }
      if (full && !anyeq) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) hits += (d[kk] == 0u);
      } else {
        uint32_t hmask = 0, emask = 0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t x = (wA[kk] ^ a.pw.w[0]) & K0;
          if constexpr (M > 4) x |= (wB[kk] ^ a.pw.w[1]) & K1;
          if (d[kk] == 0u) hmask |= 1u << (grp * 8 + kk);
          if (x == 0u) emask |= 1u << (grp * 8 + kk);
        }
        hmask &= vmask;  // (hx is a parameter: equal bytes need not mean a hash hit)
        hits += __popc(hmask);
        hm |= emask & hmask;
      }
    }
  }
}

// M in [2, 8]: lane-flag fast pass + warp-cooperative settle.
// The fast pass only answers "does some window of the lane's chunk have hash == hx": the
// d = hash - hx of two neighbouring windows are multiplied (|d| < 2^16, so the product is
// exact and zero iff one of them is) and the products tested with one accumulated ISETP,
// i.e. per window one dp4a (two for M > 4), half an IMAD and half an ISETP, plus the
// funnel shift that forms the window word.  Lanes whose chunk has a hash hit (m = 4 over
// printable ASCII: ~2.6% of lane-chunks; m = 8: ~0.2%) are settled one at a time by the
// whole warp: the flagged lane publishes its 64 bytes in a per-warp scratch, each lane
// takes one of its 32 windows (exact hash, validity, bytes) and two ballots give the hit
// count and the match mask.  A chunk with many flagged lanes (dense matches, e.g. all 'a')
// goes to the per-lane inline settle instead (short_chunk), where the warp stays while
// the density lasts.
#ifndef RK_COOP_FROM
#define RK_COOP_FROM 5
#endif
constexpr int kCoopFrom = RK_COOP_FROM;
#ifndef RK_UNROLL_FROM
#define RK_UNROLL_FROM 5  // chunk loop unrolled per stage (M >= this)
#endif
// M <= this: test the windows in pairs by the product of their d's (moves half the
// compares to the FMA pipe); longer patterns already load the FMA pipe with two dp4a per
// window and test each d directly
constexpr int kPairProductsTo = 4;
constexpr int kCoopMaxLanes = 6;
constexpr int kScratchWords = 20;  // 64 bytes + padding for the last window (16-B aligned)

template <int M>
__device__ __forceinline__ bool short_any(const ScanArgs& a, const Vec32& v,
                                          const uint32_t (&lb)[8]) {
  static_assert(M >= 2 && M <= 8, "two-word dot products");
  const uint32_t negT = 0u - (uint32_t)a.hx;
  constexpr uint32_t W0 = win_weights<M>(0), W1 = win_weights<M>(1);
  uint32_t d[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int s0 = 33 + k - M;
    if constexpr (M > 4) {
      d[k] = __dp4a(w64(lb, v, s0), W0, __dp4a(w64(lb, v, s0 + 4), W1, negT));
    } else {
      d[k] = __dp4a(w64(lb, v, s0), W0, negT);
    }
  }
  bool any = false;
  if constexpr (M > kPairProductsTo) {
#pragma unroll
    for (int k = 0; k < 32; ++k) any |= (d[k] == 0u);
  } else {
#pragma unroll
    for (int k = 0; k < 32; k += 2) any |= (d[k] * d[k + 1] == 0u);
  }
  return any;
}

// Settles the flagged lanes of one chunk (see above).  sp = the chunk's bytes in shared
// memory from its 32-byte lookback on (the TMA stage), or null for edge tiles, whose
// flagged lanes publish their 64 bytes in the warp's scratch first.  Adds to the caller's
// per-lane hit and match counts; returns the lane's match mask for the chunk.
template <int M>
__device__ __forceinline__ uint32_t coop_settle(const ScanArgs& a, uint32_t sp, const Vec32& v,
                                                const uint32_t (&lb)[8], int64_t J,
                                                unsigned flags, int lane, uint32_t* scratch,
                                                uint32_t& my_hits, uint32_t& my_matches) {
  const uint32_t negT = 0u - (uint32_t)a.hx;
  constexpr uint32_t W0 = win_weights<M>(0), W1 = win_weights<M>(1);
  constexpr uint32_t K0 = M >= 4 ? 0xffffffffu : ((1u << (8 * M)) - 1u);
  constexpr uint32_t K1 = M >= 8 ? 0xffffffffu : M > 4 ? ((1u << (8 * (M - 4))) - 1u) : 0u;
  // valid window ends of the chunk, relative to its first end position (lane 0's J):
  // window 32 L + lane is valid iff it lies in [vlo, vhi)
  const int64_t J0 = J - kR * lane;
  const uint32_t vlo = (uint32_t)min(max((int64_t)a.g.ja_lo - J0, (int64_t)0), (int64_t)kChunk);
  const uint32_t vspan =
      (uint32_t)min(max((int64_t)a.g.ja_hi - J0, (int64_t)0), (int64_t)kChunk) - vlo;
  // this lane takes the window ending at byte 32 + lane of lane L's 64 bytes (lb ++ v),
  // i.e. starting at byte 33 + lane - M; a staged chunk holds lane L's bytes at 32 L
  const uint32_t off = 33u + lane - M, r = 8u * (off & 3u);
  uint32_t hm = 0;
  const auto item = [&](uint32_t p, int L) {
    const uint32_t x1 = lds_u32(p + 4);
    const uint32_t A = __funnelshift_r(lds_u32(p), x1, r);
    uint32_t d, B = 0;
    if constexpr (M > 4) {
      B = __funnelshift_r(x1, lds_u32(p + 8), r);
      d = __dp4a(A, W0, __dp4a(B, W1, negT));
    } else {
      d = __dp4a(A, W0, negT);
    }
    const bool hit = (d == 0u) & ((uint32_t)(kR * L + lane) - vlo < vspan);
    const bool eq = hit & (((A ^ a.pw.w[0]) & K0) == 0u) & (((B ^ a.pw.w[1]) & K1) == 0u);
    my_hits += hit;
    my_matches += eq;
    const unsigned em = __ballot_sync(kFull, eq);
    hm = lane == L ? em : hm;
  };
  if (sp) {
    const uint32_t base = sp + (off & ~3u);
    while (flags) {
      const int L = __ffs(flags) - 1;
      flags &= flags - 1;
      item(base + 32u * L, L);
    }
  } else {
    // edge tile (not staged): the flagged lane publishes its 64 bytes first
    const uint32_t base = smem_u32(scratch) + (off & ~3u);
    while (flags) {
      const int L = __ffs(flags) - 1;
      flags &= flags - 1;
      if (lane == L) {
        uint4* dst = reinterpret_cast<uint4*>(scratch);
        dst[0] = make_uint4(lb[0], lb[1], lb[2], lb[3]);
        dst[1] = make_uint4(lb[4], lb[5], lb[6], lb[7]);
        dst[2] = make_uint4(v.w[0], v.w[1], v.w[2], v.w[3]);
        dst[3] = make_uint4(v.w[4], v.w[5], v.w[6], v.w[7]);
      }
      __syncwarp();
      item(base, L);
      __syncwarp();  // the scratch is rewritten for the next flagged lane
    }
  }
  return hm;
}

// Per-warp totals of hash hits and matches, flushed to the global counters once per
// warp at the end of the kernel (m = 4 hits most tiles: a per-tile atomic on one address
// from every warp would serialise in its L2 slice).
struct WarpTotals {
  uint32_t hits = 0;     // this lane's hash hits (< 2^32: a lane sees 1/32 of a warp's windows)
  uint64_t matches = 0;  // the warp's matches (warp-uniform)
};

// Records a tile's results for the ordered emission and adds to the warp's totals.
__device__ __forceinline__ void record_tile(const ScanArgs& a, uint64_t seq, uint32_t my_matches,
                                            uint32_t my_hits, uint32_t hitflags, int lane,
                                            WarpTotals& tot) {
  const uint32_t agg = __reduce_add_sync(kFull, my_matches);
  tot.hits += my_hits;
  tot.matches += agg;
  if (lane == 0) {
    a.tile_info[seq] = agg | (hitflags << 16);
    if (agg) atomicAdd(&a.block_sums[seq / kEmitTiles], (unsigned long long)agg);
  }
}

__device__ __forceinline__ void flush_totals(const ScanArgs& a, const WarpTotals& tot, int lane) {
  uint64_t hits = tot.hits;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(kFull, hits, o);
  if (lane == 0 && hits) {
    atomicAdd(&a.counters[1], (unsigned long long)hits);
    atomicAdd(&a.counters[2], (unsigned long long)(hits - tot.matches));
    // counters[3]: some warp matched a dense tile's worth (the emit's balanced phase)
    if (kDeferMin && tot.matches >= kDeferMin) a.counters[3] = 1ull;
  }
}

// A tile's exact-pass results, recorded once per tile by record_tile.
struct TileAcc {
  uint32_t hitflags = 0, my_matches = 0, my_hits = 0;
};

// Exact pass over the candidate chunks cand of tile t (staged: the chunks of bits
// [c_lo, c_lo + SC) are at st + (c - c_lo) kChunk in shared memory, lookback first).
template <int M>
__device__ __forceinline__ void exact_chunks(const ScanArgs& a, uint64_t t, uint32_t cand,
                                             int lane, TileAcc& acc, const uint8_t* st = nullptr,
                                             int c_lo = 0) {
  const TextGeom& g = a.g;
  const int64_t ta = g.tile_a(t);
  uint32_t* tmask = a.masks + (g.seq_base + t) * (kTileChunks * 32);
  while (cand) {
    const int c = __ffs(cand) - 1;
    cand &= cand - 1;
    const SlowOut r = slow_chunk<M>(a, ta + c * kChunk + lane * kR,
                                    st ? st + (c - c_lo) * kChunk + lane * kR : nullptr);
    acc.my_hits += r.hits;
    acc.my_matches += __popc(r.hm);
    if (__ballot_sync(kFull, r.hm != 0)) {
      tmask[c * 32 + lane] = r.hm;
      acc.hitflags |= 1u << c;
    }
  }
}

// Exact pass over the candidate chunks of tile t; records the tile's match count,
// chunk bitmap and hit masks for the ordered emission and adds to the warp's totals.
template <int M>
__device__ __forceinline__ void finish_tile(const ScanArgs& a, uint64_t t, uint32_t cand,
                                            int lane, WarpTotals& tot) {
  TileAcc acc;
  exact_chunks<M>(a, t, cand, lane, acc);
  record_tile(a, a.g.seq_base + t, acc.my_matches, acc.my_hits, acc.hitflags, lane, tot);
}

template <int M>
__global__ void __launch_bounds__(32 * scan_warps(M), scan_min_blocks(M))
    rk_scan_kernel(const ScanArgs a) {
  constexpr int kWarps = scan_warps(M);
  using Ring = WarpRingT<scan_stage_chunks(M)>;
  // PDL both ways: wait for the previous grid in the stream (its writes -- the text, the
  // previous emit's reads of our scratch -- must be complete), and let the emit grid be
  // scheduled as our CTAs retire (it waits for our results the same way)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  Ring* R = reinterpret_cast<Ring*>(smem) + warp;
  uint32_t* scratch =
      reinterpret_cast<uint32_t*>(smem + kWarps * sizeof(Ring)) + warp * kScratchWords;
  (void)scratch;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * a.warps;
  const uint64_t w = (uint64_t)blockIdx.x * a.warps + warp;
  const uint32_t T = (uint32_t)a.hx;
  const auto pred = [T](uint32_t L) { return L == T; };
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  WarpTotals tot;
  bool dense = false;  // warp-uniform: M <= 8 and the warp's last tile was mostly matches
  (void)dense;
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    if constexpr (M >= 32) {
      // candidates are ~2^-32 per window: one vote per tile, and a tile with any
      // candidate gets the exact pass over all of its chunks
      bool any = false;
      stream_tile<M>(a.g, R, S, t, lane,
                     [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t& carryS, int64_t, int) {
                       any |= fast_chunk<M>(v, lb, lane, carryS, a.g.K, pred);
                     });
      finish_tile<M>(a, t, __any_sync(kFull, any) ? (1u << kTileChunks) - 1 : 0u, lane, tot);
    } else if constexpr (M >= kFoldFilter) {
      // the 32-byte fold S(j) agrees with the window hash mod 2^M (the out-term is a
      // multiple of 2^M), so the m >= 32 chain with a masked compare is an exact-hit
      // filter (false positives ~2^-M per window); flagged chunks get the exact pass.
      // The masked compares accumulate through lop3's predicate output (one LOP3 per
      // window, as the ISETP.EQ.OR of m >= 32).
      const MaskedEq fpred{T, (uint32_t)((1ull << M) - 1u)};
      uint32_t cand = 0;
      TileAcc acc;
      // flagged chunks (~1.6% at m = 16) are settled while their stage is still in shared
      // memory, not re-read from L2 after the stage is handed back (m = 16: +5%)
      stream_tile<32>(
          a.g, R, S, t, lane,
          [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t& carryS, int64_t, int c) {
            const bool any = fast_chunk<32, kFoldFmaBytes>(v, lb, lane, carryS, a.g.K, fpred);
            if (__any_sync(kFull, any)) cand |= 1u << c;
          },
          [&](const uint8_t* st, int c_lo, int c_n) {
            const uint32_t mine = cand & (((1u << c_n) - 1u) << c_lo);
            if (mine) exact_chunks<M>(a, t, mine, lane, acc, st, c_lo);
            cand &= ~mine;
          });
      exact_chunks<M>(a, t, cand, lane, acc);  // edge tiles (not staged)
      record_tile(a, a.g.seq_base + t, acc.my_matches, acc.my_hits, acc.hitflags, lane, tot);
    } else if constexpr (M >= kShortInline) {
      // exact hits are rare (m = 8 printable ASCII: ~2% of chunks): flag chunks, settle
      // them in the exact pass
      const uint32_t cand = fast_tile<M, RK_ROLL_UNROLL>(a.g, R, S, t, lane, pred);
      finish_tile<M>(a, t, cand, lane, tot);
    } else {
      const uint64_t seq = a.g.seq_base + t;
      uint32_t* tmask = a.masks + seq * (kTileChunks * 32);
      uint32_t hitflags = 0, my_matches = 0, my_hits = 0;
      const int64_t ta = a.g.tile_a(t);
      // computed once per tile (pinned where the per-chunk inline settle reads it: ptxas
      // would otherwise rematerialise the 64-bit compares in every chunk)
      uint32_t full_u = ta >= (int64_t)a.g.ja_lo && ta + kTile <= (int64_t)a.g.ja_hi;
      if constexpr (M < kCoopFrom) asm volatile("" : "+r"(full_u));
      const bool full = full_u != 0u;
      // kDense (M < kCoopFrom): the warp's previous tile was mostly matches (e.g. all
      // 'a'), so this one settles whole all-hit groups at once
      const auto tile_body = [&](auto dense_tag) {
        constexpr bool kDense = decltype(dense_tag)::value;
        stream_tile<M, (M >= RK_UNROLL_FROM)>(
            a.g, R, S, t, lane,
            [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t&, int64_t J, int c) {
              uint32_t hm = 0;
              if constexpr (M >= kCoopFrom) {
                if (!dense) {
                  const unsigned flags = __ballot_sync(kFull, short_any<M>(a, v, lb));
                  if (!flags) return;
                  if (__popc(flags) <= kCoopMaxLanes) {
                    hm = coop_settle<M>(a, S.cur, v, lb, J, flags, lane, scratch, my_hits,
                                        my_matches);
                    if (__ballot_sync(kFull, hm != 0)) {
                      tmask[c * 32 + lane] = hm;
                      hitflags |= 1u << c;
                    }
                    return;
                  }
                }
              }
              uint32_t hits = 0;
              short_chunk<M, kDense>(a, v, lb, full, full ? 0xffffffffu : valid_mask(a.g, J),
                                     hm, hits);
              // M >= kCoopFrom: stay on the inline settle, skipping the flag pass, while
              // most lanes keep hitting
              if constexpr (M >= kCoopFrom)
                dense = __popc(__ballot_sync(kFull, hits != 0)) > kCoopMaxLanes;
              my_hits += hits;
              my_matches += __popc(hm);
              if (__ballot_sync(kFull, hm != 0)) {
                tmask[c * 32 + lane] = hm;
                hitflags |= 1u << c;
              }
            });
      };
      if constexpr (M < kCoopFrom) {
        if (dense) {
          tile_body(std::true_type{});
        } else {
          tile_body(std::false_type{});
        }
      } else {
        tile_body(std::false_type{});
      }
      record_tile(a, seq, my_matches, my_hits, hitflags, lane, tot);
      if constexpr (M < kCoopFrom) {
        // the next tile takes the dense settle when this one was mostly matches
        dense = __reduce_add_sync(kFull, my_matches) > (uint32_t)(kTile / 2);
      }
    }
  }
  flush_totals(a, tot, lane);
}

}  // namespace rkb
