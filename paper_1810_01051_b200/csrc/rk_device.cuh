// rk_device.cuh -- device-side building blocks of the B200 Rabin-Karp scan.
//
// Hash (reference /root/reference/pkg/src/rkmatch/rkhash.py:21-28):
//     h(x) = sum_{i<m} t[x+i] * 2^(m-1-i)   mod 2^64      (base 2, raw bytes, no prime)
// Facts the kernels are built on:
//   * low32(h) depends only on the last min(m,32) bytes of the window;
//   * for m >= 32, low32(h(window ending at j)) = S(j) where S(j) = 2 S(j-1) + t[j] mod 2^32
//     is a single running fold (the out-term 2^m * t[x] vanishes mod 2^32);
//   * for m < 32 the exact 32-bit roll is L' = 2L + in - 2^m out (rkhash.py:48-60 `roll`),
//     and L(j) = S(j) mod 2^m (the out-term is a multiple of 2^m);
//   * for m <= 24, h < 2^32, so low32 equality IS 64-bit hash equality.
// A window is a hash hit iff all 64 bits agree; a hit is a match iff its bytes equal the
// pattern, otherwise it is a collision (_scan.py:38-49).  The kernels filter on the exact
// low-32 value and confirm the high half and the bytes only for the rare survivors.
//
// Work decomposition.  Positions are window END positions in "a-space" (offsets from
// the 32-byte-aligned address at or below the text).  A chunk is 1 KiB of end positions
// (32 per lane); a tile is kTileChunks chunks and is the unit of ordered emission.  Warp
// w of W owns tiles w, w+W, w+2W, ... and streams them through a per-warp ring of
// shared-memory stages filled by TMA bulk copies (cp.async.bulk + mbarrier), so the bytes
// in flight live in shared memory, not registers.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace rkb {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kR = 32;                       // end positions per lane per chunk
constexpr int kChunk = 32 * kR;              // 1 KiB of end positions per warp step
constexpr int kTileChunks = 8;               // chunks per tile
constexpr int kTile = kChunk * kTileChunks;  // 8 KiB per tile (unit of ordered emission)
constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr uint32_t kFoldW = 0x01020408u;     // dp4a weights: 8*b0 + 4*b1 + 2*b2 + b3
constexpr int kEmitTiles = 256;              // tiles per block of the ordered emission
constexpr int kMaxDevices = 64;

// TMA ring: kStages stages of kStageChunks chunks, each stage preceded by the 32 bytes
// before its first chunk (the lookback the first lane needs).
constexpr int kStageChunks = 4;
constexpr int kStages = 2;
static_assert(kTileChunks % kStageChunks == 0, "stage/tile");

struct Vec32 {
  uint32_t w[8];
};

struct PatWords {
  uint32_t w[8];  // pattern bytes (m < 32), little-endian packed
};

// Runtime copies of small constants.  The roll is written as x * k + y with k in a
// register so ptxas emits IMAD (FMA pipe) instead of LEA/IADD3 (ALU pipe): the per-byte
// work is then split between the two integer pipes ("instruction budget").
struct RollConsts {
  uint32_t k2, k8, k16;  // 2, 8, 16
  uint32_t negpow;       // -(2^m) mod 2^32 (m < 32)
};

// Text geometry shared by every streaming kernel.
struct TextGeom {
  const uint8_t* abase;  // 32-byte-aligned address at or below the text
  uint64_t amis;         // text - abase, in [0, 32)
  uint64_t n;            // text length in bytes
  uint64_t ja_lo, ja_hi; // valid window END positions, a-space, [lo, hi)
  uint64_t tile0;        // a-space tile index of the launch's first tile
  uint64_t num_tiles;    // tiles in this launch
  uint64_t seq_base;     // sequence number of this launch's first tile (staged scans)
  uint32_t m;
  RollConsts K;

  __device__ __forceinline__ int64_t tile_a(uint64_t t) const {
    return (int64_t)((tile0 + t) * (uint64_t)kTile);
  }
  // every byte a tile's fast pass touches, [ta - 32, ta + kTile), lies in the text
  __device__ __forceinline__ bool interior(int64_t ta) const {
    return ta - 32 >= (int64_t)amis && ta + kTile <= (int64_t)(amis + n);
  }
  __device__ __forceinline__ bool valid_end(int64_t ja) const {
    return ja >= (int64_t)ja_lo && ja < (int64_t)ja_hi;
  }
};

// ------------------------------------------------------------------------- loads
__device__ __forceinline__ Vec32 ldg256(const uint8_t* p) {
  Vec32 v;
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
        "=r"(v.w[6]), "=r"(v.w[7])
      : "l"(p));
  return v;
}

// 4 text bytes at a-position p, zero outside the text (cold path, kept out of line).
static __device__ __noinline__ uint32_t edge_word(const uint8_t* abase, int64_t lo, int64_t hi,
                                                  int64_t p) {
  uint32_t w = 0;
  for (int b = 0; b < 4; ++b) {
    const int64_t q = p + b;
    const uint32_t byte = (q >= lo && q < hi) ? (uint32_t)abase[q] : 0u;
    w |= byte << (8 * b);
  }
  return w;
}

// 32 bytes at a-position p (32-aligned, may be negative).  Bytes outside the text read
// as 0; positions whose windows would touch them are masked by the validity check.
__device__ __forceinline__ Vec32 load_edge(const TextGeom& g, int64_t p) {
  const int64_t lo = (int64_t)g.amis, hi = (int64_t)(g.amis + g.n);
  if (p >= lo && p + 32 <= hi) return ldg256(g.abase + p);
  Vec32 v;
#pragma unroll 1
  for (int i = 0; i < 8; ++i) v.w[i] = edge_word(g.abase, lo, hi, p + 4 * i);
  return v;
}

// 32 bytes of shared memory at p (16-byte aligned).
__device__ __forceinline__ Vec32 lds32(const uint8_t* p) {
  const uint4 x = *reinterpret_cast<const uint4*>(p);
  const uint4 y = *reinterpret_cast<const uint4*>(p + 16);
  Vec32 v;
  v.w[0] = x.x;
  v.w[1] = x.y;
  v.w[2] = x.z;
  v.w[3] = x.w;
  v.w[4] = y.x;
  v.w[5] = y.y;
  v.w[6] = y.z;
  v.w[7] = y.w;
  return v;
}

// ------------------------------------------------------------------------- bytes
__device__ __forceinline__ uint32_t bsel(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)k);
}

// word (4 bytes) of lb ++ v starting at byte p (static after unrolling; p + 4 <= 64)
__device__ __forceinline__ uint32_t w64(const uint32_t (&lb)[8], const Vec32& v, int p) {
  const int q = p >> 2, r = p & 3;
  const uint32_t lo = q < 8 ? lb[q] : v.w[q - 8];
  if (r == 0) return lo;
  const uint32_t hi = (q + 1) < 8 ? lb[q + 1] : ((q + 1) < 16 ? v.w[q + 1 - 8] : 0u);
  return __funnelshift_r(lo, hi, 8 * r);
}

// dp4a weights of window bytes [4q, 4q+4) in the hash of an M-byte window (M <= 8):
// byte i carries 2^(M-1-i).
template <int M>
__host__ __device__ constexpr uint32_t win_weights(int q) {
  uint32_t w = 0;
  for (int b = 0; b < 4; ++b) {
    const int i = 4 * q + b;
    if (i < M) w |= (uint32_t)(1u << (M - 1 - i)) << (8 * b);
  }
  return w;
}

// Bit k set when window end J + k is in the launch's range [ja_lo, ja_hi).
__device__ __forceinline__ uint32_t valid_mask(const TextGeom& g, int64_t J) {
  const int64_t lo = min(max((int64_t)g.ja_lo - J, (int64_t)0), (int64_t)32);
  const int64_t hi = min(max((int64_t)g.ja_hi - J, (int64_t)0), (int64_t)32);
  const uint32_t above = lo >= 32 ? 0u : (0xffffffffu << lo);
  const uint32_t below = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return above & below;
}

// fold of 32 bytes, mod 2^32 (= S at the last byte): 8 dp4a + 7 shifts.
__device__ __forceinline__ uint32_t fold32(const uint32_t (&w)[8]) {
  uint32_t s = __dp4a(w[0], kFoldW, 0u);
#pragma unroll
  for (int i = 1; i < 8; ++i) s = __dp4a(w[i], kFoldW, s << 4);
  return s;
}

// fold of bytes [32-M, 32) of lb (the M bytes preceding J), exact mod 2^32.
template <int M>
__device__ __forceinline__ uint32_t fold_tail(const uint32_t (&lb)[8]) {
  static_assert(M >= 1 && M < 32, "tail");
  constexpr int first = 32 - M;
  uint32_t s = 0;
#pragma unroll
  for (int i = first; i < ((first + 3) & ~3); ++i) s = 2u * s + bsel(lb[i >> 2], i & 3);
#pragma unroll
  for (int wi = (first + 3) >> 2; wi < 8; ++wi) s = __dp4a(lb[wi], kFoldW, s << 4);
  return s;
}

// dp4a with unsigned text bytes and signed weights (PTX dp4a.u32.s32).
__device__ __forceinline__ uint32_t dp4a_us(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Masked-equality filter test: L is a candidate iff ((L ^ T) & mask) == 0.  Its windows
// are accumulated with lop3's predicate output (PTX lop3.and: p = (result != 0) AND q), so
// each window costs one LOP3.PAND and no separate predicate-combining PLOP3.
struct MaskedEq {
  uint32_t T, mask;
};

// q && ((a ^ b) & c) != 0, in one LOP3.LUT.PAND (ptxas folds the selp/setp wrapper)
__device__ __forceinline__ bool lop3_nz_and(uint32_t a, uint32_t b, uint32_t c, bool q) {
  uint32_t r;
  asm("{.reg .pred p, qq;\n"
      "setp.ne.u32 qq, %4, 0;\n"
      "lop3.and.b32 _|p, %1, %2, %3, 0x28, qq;\n"
      "selp.u32 %0, 1, 0, p;}\n"
      : "=r"(r)
      : "r"(a), "r"(b), "r"(c), "r"((uint32_t)q));
  return r != 0;
}

// ---------------------------------------------------------------------------------
// The fast roll over one chunk: the lane owns window END positions [J, J+32), its 32
// bytes in v; for M < 32, lb holds the 32 bytes before J.  Returns whether
// pred(low32 hash) held at any of its positions.
//
//  M >= 32: S(j) = fold of t[j-31..j] (mod 2^32) = low32 of every window hash.  Per
//    4-byte word w starting from S:  S1 = 2S + b0, S2 = 2S1 + b1 (PRMT + IMAD),
//    S3 = 8S + dp4a(w,{4,2,1,0}), S4 = 16S + dp4a(w,{8,4,2,1}) (IDP + IMAD): 6 ALU +
//    6 FMA-pipe instructions per 4 bytes including the 4 compares.  The lane's seed
//    S(J-1) is the previous lane's 32-byte fold F (one shfl), because 2^32 = 0; lane 0
//    takes carryS (the previous chunk's lane 31, or the tile's lookback fold).
//  M < 32: exact roll L' = 2L + in - 2^M out seeded with the fold of the M bytes before
//    J, alternating two instruction mixes so the ALU and FMA pipes carry ~2.5
//    instructions per byte each.
// (FmaBytes: take b0/b1 with a one-hot dp4a on the FMA pipe instead of a PRMT -- for
// callers whose compares load the ALU pipe.)  pred is either a callable (candidate iff
// pred(L)) or a MaskedEq (M >= 32 chain only), accumulated as "all windows miss".
template <int M, bool FmaBytes = false, class Pred>
__device__ __forceinline__ bool fast_chunk(const Vec32& v, const uint32_t (&lb)[8], int lane,
                                           uint32_t& carryS, const RollConsts& K, Pred pred) {
  bool any = false;
  if constexpr (M >= 32) {
    constexpr bool kMasked = std::is_same<Pred, MaskedEq>::value;
    bool allnz = true;
    const auto test = [&](uint32_t s) {
      if constexpr (kMasked) {
        allnz = lop3_nz_and(s, pred.T, pred.mask, allnz);
      } else {
        any |= pred(s);
      }
    };
    uint32_t c4[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c4[i] = __dp4a(v.w[i], kFoldW, 0u);
    uint32_t F = c4[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) F = F * K.k16 + c4[i];
    const uint32_t up = __shfl_up_sync(kFull, F, 1);
    const uint32_t top = __shfl_sync(kFull, F, 31);
    uint32_t S = lane == 0 ? carryS : up;
    carryS = top;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t w = v.w[i];
      const uint32_t s1 =
          FmaBytes ? __dp4a(w, 0x00000001u, S * K.k2) : S * K.k2 + bsel(w, 0);
      const uint32_t s2 =
          FmaBytes ? __dp4a(w, 0x00000100u, s1 * K.k2) : s1 * K.k2 + bsel(w, 1);
      const uint32_t s3 = S * K.k8 + __dp4a(w, 0x00010204u, 0u);
      const uint32_t s4 = S * K.k16 + c4[i];
      test(s1);
      test(s2);
      test(s3);
      test(s4);
      S = s4;
    }
    if constexpr (kMasked) any = !allnz;
  } else {
    uint32_t L = fold_tail<M>(lb);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int io = 32 + k - M;
      const uint32_t wout = io < 32 ? lb[io >> 2] : v.w[(io - 32) >> 2];
      if (k & 1) {
        // ALU-heavy mix: both bytes by PRMT, two IMADs
        L = L * K.k2 + bsel(v.w[k >> 2], k & 3);
        L = bsel(wout, io & 3) * K.negpow + L;
      } else if constexpr (M <= 7) {
        // out weight -2^M fits a signed byte: both bytes extracted by dp4a (FMA pipe)
        const uint32_t t = __dp4a(v.w[k >> 2], 1u << (8 * (k & 3)), L * K.k2);
        L = dp4a_us(wout, (uint32_t)(uint8_t)(-(1 << M)) << (8 * (io & 3)), t);
      } else {
        // FMA-heavy mix: in by dp4a extract-and-add, out by PRMT + IMAD
        const uint32_t t = __dp4a(v.w[k >> 2], 1u << (8 * (k & 3)), L * K.k2);
        L = bsel(wout, io & 3) * K.negpow + t;
      }
      any |= pred(L);
    }
  }
  return any;
}

// ------------------------------------------------------------------------- TMA ring
// SC = chunks per stage (the scan kernels use kStageChunks; the multi-pattern kernel,
// which runs twice the warps per SM, half that).
template <int SC>
struct __align__(16) WarpRingT {
  static constexpr int kChunks = SC;
  static constexpr int kBytes = SC * kChunk + 32;  // stage + its 32-byte lookback
  uint8_t buf[kStages][kBytes];
  unsigned long long bar[kStages];
};
using WarpRing = WarpRingT<kStageChunks>;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int SC>
__device__ __forceinline__ void ring_init(WarpRingT<SC>* R, int lane) {
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&R->bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// A warp's stream: the stages of its interior tiles in order, kStages in flight.
// Warp-uniform bookkeeping kept in 32-bit registers with incremental addressing; lane 0
// issues the TMA copies.  Tiles outside [int_lo, int_hi) (at most the first and last of a
// launch) are not staged -- the consumer reads them directly.
struct Stream {
  const uint8_t* psrc;  // global address of the next stage to issue (its lookback start)
  uint32_t pt;          // tile of the next stage to issue
  uint32_t ps;          // stage index within that tile
  uint32_t pending;     // stages issued and not yet consumed
  uint32_t cslot;       // ring slot the consumer reads next
  uint32_t cphase;      // its mbarrier parity
  uint32_t pslot;       // ring slot the producer fills next
  uint32_t W, int_lo, int_hi, ntiles;
  int64_t tile_jump;    // bytes from the end of one of the warp's tiles to its next one
  uint32_t ring_s;      // shared-space address of the ring's first stage
  uint32_t cur;         // during op(): shared-space address of the current chunk's bytes
                        // from its 32-byte lookback on, or 0 (edge tiles: read from global)
};

// 4 bytes of shared memory at shared-space address a (4-byte aligned)
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t x;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
  return x;
}

__device__ __forceinline__ void stream_seek(const TextGeom& g, Stream& S) {
  while (S.pt < S.ntiles && (S.pt < S.int_lo || S.pt >= S.int_hi)) S.pt += S.W;
  S.psrc = g.abase + g.tile_a(S.pt) - 32;
}

template <int SC>
__device__ __forceinline__ void stream_issue(WarpRingT<SC>* R, Stream& S, int lane) {
  if (S.pt >= S.ntiles || S.pt >= S.int_hi) return;
  if (lane == 0) bulk_g2s(R->buf[S.pslot], S.psrc, WarpRingT<SC>::kBytes, &R->bar[S.pslot]);
  S.pslot = (S.pslot + 1) & (kStages - 1);
  ++S.pending;
  S.psrc += SC * kChunk;
  if (++S.ps == kTileChunks / SC) {
    S.ps = 0;
    S.pt += S.W;
    S.psrc += S.tile_jump;
  }
}

template <int SC>
__device__ __forceinline__ void stream_init(const TextGeom& g, WarpRingT<SC>* R, Stream& S,
                                            uint32_t w, uint32_t W, int lane) {
  static_assert(kTileChunks % SC == 0, "stage/tile");
  static_assert((kStages & (kStages - 1)) == 0, "ring size must be a power of two");
  // interior tiles are exactly [int_lo, int_hi): tile_a - 32 >= amis and
  // tile_a + kTile <= amis + n, with tile_a = (tile0 + t) * kTile
  const int64_t lo_a = (int64_t)g.amis + 32, hi_a = (int64_t)(g.amis + g.n) - kTile;
  int64_t lo = (lo_a + kTile - 1) / kTile - (int64_t)g.tile0;
  int64_t hi = (hi_a >= 0 ? hi_a / kTile + 1 : 0) - (int64_t)g.tile0;
  S.int_lo = (uint32_t)(lo < 0 ? 0 : lo);
  S.int_hi = (uint32_t)(hi < (int64_t)S.int_lo ? S.int_lo : (hi > (int64_t)g.num_tiles ? g.num_tiles : hi));
  S.ntiles = (uint32_t)g.num_tiles;
  S.W = W;
  S.pt = w;
  S.ps = 0;
  S.pending = 0;
  S.cslot = S.pslot = 0;
  S.cphase = 0;
  S.tile_jump = (int64_t)(W - 1) * kTile;
  S.ring_s = smem_u32(R->buf[0]);
  stream_seek(g, S);
  for (int i = 0; i < kStages; ++i) stream_issue(R, S, lane);
}

// Streams tile t chunk by chunk into op(v, lb, carryS, J, c): v = the lane's 32 bytes
// (window ends [J, J+32)), lb = the 32 bytes before J (0 < M < 32 only; M = 0: neither
// lb nor the fold), carryS = the fold seed for M >= 32 (see fast_chunk), c = chunk index
// in the tile.  Interior tiles come from the TMA ring; edge tiles go through the
// bounds-checked loader.
struct NoStageHook {
  __device__ __forceinline__ void operator()(const uint8_t*, int, int) const {}
};

// stage_done(st, c_lo, c_n), called after the chunks [c_lo, c_lo + c_n) of a staged stage
// have been through op and before the stage is handed back (st = the stage in shared
// memory, its 32-byte lookback first), lets a caller revisit those bytes cheaply.
template <int M, bool UNROLL = true, int SC, class Op, class Hook = NoStageHook>
__device__ __forceinline__ void stream_tile(const TextGeom& g, WarpRingT<SC>* R, Stream& S,
                                            uint32_t t, int lane, Op&& op,
                                            Hook&& stage_done = Hook{}) {
  const int64_t ta = g.tile_a(t);
  uint32_t carryS = 0;
  uint32_t lb[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) lb[i] = 0;
  if (t >= S.int_lo && t < S.int_hi) {
#pragma unroll 1
    for (int s = 0; s < kTileChunks / SC; ++s) {
      mbar_wait(&R->bar[S.cslot], S.cphase);
      const uint8_t* st = R->buf[S.cslot];
      if constexpr (M >= 32) {
        if (s == 0) carryS = fold32(lds32(st).w);  // tile lookback, broadcast read
      }
#pragma unroll(UNROLL ? SC : 1)
      for (int j = 0; j < SC; ++j) {
        const Vec32 v = lds32(st + 32 + j * kChunk + lane * kR);
        if constexpr (M > 0 && M < 32) {
          const Vec32 l = lds32(st + j * kChunk + lane * kR);
#pragma unroll
          for (int i = 0; i < 8; ++i) lb[i] = l.w[i];
        }
        const int c = s * SC + j;
        S.cur = S.ring_s + S.cslot * (uint32_t)WarpRingT<SC>::kBytes + j * kChunk;
        op(v, lb, carryS, ta + c * kChunk + lane * kR, c);
      }
      stage_done(st, s * SC, SC);
      // the slot's bytes are consumed: hand it back to the producer
      S.cslot = (S.cslot + 1) & (kStages - 1);
      S.cphase ^= (S.cslot == 0);
      --S.pending;
      __syncwarp();
      stream_issue(R, S, lane);
    }
  } else {
    if constexpr (M >= 32) carryS = fold32(load_edge(g, ta - 32).w);
    S.cur = 0;
#pragma unroll 1
    for (int c = 0; c < kTileChunks; ++c) {
      const int64_t J = ta + c * kChunk + lane * kR;
      const Vec32 v = load_edge(g, J);
      if constexpr (M > 0 && M < 32) {
        const Vec32 l = load_edge(g, J - 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) lb[i] = l.w[i];
      }
      op(v, lb, carryS, J, c);
    }
  }
}

// Fast pass over tile t: bitmask of its chunks in which some lane saw pred() hold.
template <int M, bool UNROLL = true, int SC, class Pred>
__device__ __forceinline__ uint32_t fast_tile(const TextGeom& g, WarpRingT<SC>* R, Stream& S,
                                              uint32_t t, int lane, Pred pred) {
  uint32_t cand = 0;
  stream_tile<M, UNROLL>(g, R, S, t, lane,
                 [&](const Vec32& v, const uint32_t (&lb)[8], uint32_t& carryS, int64_t, int c) {
                   const bool any = fast_chunk<M>(v, lb, lane, carryS, g.K, pred);
                   if (__any_sync(kFull, any)) cand |= 1u << c;
                 });
  return cand;
}

// ------------------------------------------------------------------------- warp utils
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

}  // namespace rkb
