// rk_device.cuh -- device-side building blocks of the B200 Rabin-Karp scan.
//
// Hash (reference /root/reference/pkg/src/rkmatch/rkhash.py:21-28):
//     h(x) = sum_{i<m} t[x+i] * 2^(m-1-i)   mod 2^64      (base 2, raw bytes, no prime)
// Facts the kernels are built on:
//   * low32(h) depends only on the last min(m,32) bytes of the window;
//   * for m >= 32, low32(h(window ending at j)) = S(j) where S(j) = 2 S(j-1) + t[j] mod 2^32
//     is a single running fold (the out-term 2^m * t[x] vanishes mod 2^32);
//   * for m < 32 the exact 32-bit roll is L' = 2L + in - 2^m out (rkhash.py:48-60 `roll`);
//   * for m <= 24, h < 2^32, so low32 equality IS 64-bit hash equality.
// A window is a hash hit iff all 64 bits agree; a hit is a match iff its bytes equal the
// pattern, otherwise it is a collision (_scan.py:38-49).  The kernels filter on the exact
// low-32 value and confirm the high half and the bytes only for the rare survivors.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rkb {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kR = 32;                       // end positions per lane per chunk
constexpr int kChunk = 32 * kR;              // 1 KiB of end positions per warp step
constexpr int kTileChunks = 16;              // chunks per ordered tile
constexpr int kTile = kChunk * kTileChunks;  // 16 KiB per tile (unit of ordered compaction)
constexpr int kPrefetch = 4;                 // chunks in flight per warp (4 x 1 KiB)
constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr uint32_t kFoldW = 0x01020408u;     // dp4a weights: 8*b0 + 4*b1 + 2*b2 + b3

// Look-back tile status word: [epoch:16 | flag:2 | value:46].
constexpr uint64_t kFlagAgg = 1, kFlagIncl = 2;
__host__ __device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag,
                                                         uint64_t v) {
  return (uint64_t(epoch & 0xffff) << 48) | (flag << 46) | (v & ((1ull << 46) - 1));
}

struct Vec32 {
  uint32_t w[8];
};

struct PatWords {
  uint32_t w[8];  // pattern bytes (m < 32), little-endian packed
};

// Arguments of one single-pattern scan launch.  Positions are in "a-space": offsets
// from `abase`, the 32-byte-aligned address at or below the text pointer; text byte i
// sits at a-position i + amis.
struct ScanArgs {
  const uint8_t* abase;
  uint64_t amis;        // text - abase, in [0, 32)
  uint64_t n;           // text length in bytes
  const uint8_t* pattern;  // device copy of the pattern (m bytes)
  uint64_t hx;          // 64-bit pattern hash
  uint64_t ja_lo, ja_hi;   // valid window END positions, a-space, [lo, hi)
  uint64_t tile0;       // a-space tile index of the first tile of this launch
  uint64_t num_tiles;   // tiles in this launch
  uint64_t seq_base;    // look-back sequence number of this launch's first tile
  uint64_t ticket_base; // value of *ticket before this launch
  int64_t out_bias;     // added to every reported window start (shards / staging)
  int64_t* out;         // ordered window starts, first `cap` written
  uint64_t cap;
  unsigned long long* ticket;
  unsigned long long* counters;  // [0]=matches total, [1]=hash_hits, [2]=collisions
  uint64_t* status;     // look-back status per sequence number
  uint32_t m;
  uint32_t epoch;
  uint32_t last_launch; // 1 if this launch's last tile ends the logical scan
  PatWords pw;
};

__device__ __forceinline__ Vec32 ldg256(const uint8_t* p) {
  Vec32 v;
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
        "=r"(v.w[6]), "=r"(v.w[7])
      : "l"(p));
  return v;
}

// 32 bytes at a-position p (32-aligned, may be negative).  Bytes outside the text read
// as 0; positions whose windows would touch them are masked by the validity check.
__device__ __forceinline__ Vec32 load_edge(const ScanArgs& a, int64_t p) {
  const int64_t lo = (int64_t)a.amis, hi = (int64_t)(a.amis + a.n);
  if (p >= lo && p + 32 <= hi) return ldg256(a.abase + p);
  Vec32 v;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t q = p + 4 * i + b;
      const uint32_t byte = (q >= lo && q < hi) ? (uint32_t)a.abase[q] : 0u;
      w |= byte << (8 * b);
    }
    v.w[i] = w;
  }
  return v;
}

__device__ __forceinline__ uint32_t bsel(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)k);
}

// Byte i of the 64-byte window [J-32, J+32) held as lb[0..7] ++ w[0..7].
template <int I>
__device__ __forceinline__ uint32_t byte64(const uint32_t (&lb)[8], const uint32_t (&w)[8]) {
  static_assert(I >= 0 && I < 64, "byte index");
  if constexpr (I < 32) return bsel(lb[I >> 2], I & 3);
  else return bsel(w[(I - 32) >> 2], I & 3);
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
  // leading partial word byte by byte, then whole words by dp4a
#pragma unroll
  for (int i = first; i < ((first + 3) & ~3); ++i) s = 2u * s + bsel(lb[i >> 2], i & 3);
#pragma unroll
  for (int wi = (first + 3) >> 2; wi < 8; ++wi) s = __dp4a(lb[wi], kFoldW, s << 4);
  return s;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back (single-pass ordered prefix over tiles).  Every tile publishes its
// aggregate before waiting, and only waits on tiles with a smaller sequence number that
// a running warp already owns, so progress is guaranteed.  Returns the exclusive prefix.
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint64_t seq, uint32_t epoch,
                                             uint64_t agg, int lane) {
  if (seq == 0) {
    if (lane == 0) st_relaxed_u64(&status[0], pack_status(epoch, kFlagIncl, agg));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&status[seq], pack_status(epoch, kFlagAgg, agg));
  uint64_t excl = 0;
  int64_t pred = (int64_t)seq - 1;
  for (;;) {
    const int64_t idx = pred - lane;
    uint64_t s = 0, flag = 0;
    for (;;) {
      if (idx >= 0) {
        s = ld_relaxed_u64(&status[idx]);
        flag = ((s >> 48) == (epoch & 0xffff)) ? ((s >> 46) & 3) : 0;
      } else {
        s = 0;
        flag = kFlagIncl;  // before the first tile: prefix 0
      }
      if (!__any_sync(kFull, flag == 0)) break;
      __nanosleep(32);
    }
    const unsigned incl = __ballot_sync(kFull, flag == kFlagIncl);
    const int first = incl ? __ffs(incl) - 1 : 31;
    const uint64_t v = (lane <= first) ? (s & ((1ull << 46) - 1)) : 0;
    excl += warp_sum_u64(v);
    if (incl) break;
    pred -= 32;
  }
  if (lane == 0) st_relaxed_u64(&status[seq], pack_status(epoch, kFlagIncl, excl + agg));
  return excl;
}

}  // namespace rkb
