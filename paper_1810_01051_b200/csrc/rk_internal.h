// rk_internal.h -- host-side declarations shared by the CUDA translation units.
//
// Build-time knobs (RK_*; defaults are the measured best on B200, and tools/ab.sh /
// RK_DEFINES in paper_1810_01051_b200/_build.py build variants to A/B them):
//   RK_PDL               programmatic dependent launch of scan and emit (1)
//   RK_WIDE_FROM         first m with the wide 12-warp x 8 KiB-stage shape (15)
//   RK_WIDE_W/S/B, RK_BASE_W/S/B   warps / stage chunks / CTAs per SM of the shapes
//   RK_FOLD_FMA_BYTES    fold filter takes b0/b1 by dp4a instead of PRMT (0)
//   RK_COOP_FROM         first m with the lane-flag + cooperative settle (5)
//   RK_UNROLL_FROM       first m whose chunk loop is unrolled per stage (5)
//   RK_EMIT_MIN_SMEM_KB  emit CTA shared-memory floor, RK_EMIT_CTAS per SM (115)
//   RK_EMIT_CTAS         emit CTAs per SM (1)
//   RK_EMIT_MAX_GROUPS   groups of 256 tiles one emit block expands, static schedule (4)
//   RK_EMIT_DEFER_MIN    matches from which a tile goes to the balanced phase (1024; 0 off)
//   RK_MULTI_WARPS/STAGE, RK_MULTI_UNROLL   q-gram / tiny multi-pattern kernel shape
//   RK_MULTI_APPEND_MAX  pairs a short-sweep warp buffers before one atomic (256; 0 off)
//   RK_SHORT_KEY_REFINE  3-gram anchors refined on 4-byte prefixes (1)
//   RK_HOST_PROFILE      per-call host time of the enqueue steps, printed at exit (off)
//   RK_DEBUG_CHECKS      device-side bounds checks (trap) in the emit queue (off)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rk_device.cuh"

namespace rkb {

// single pattern (rk_scan.cu, kernels in rk_scan_impl.cuh)
struct ScanArgs {
  TextGeom g;
  const uint8_t* pattern;         // device copy of the pattern (m bytes)
  uint64_t hx;                    // 64-bit pattern hash
  unsigned long long* counters;   // [1]=hash_hits, [2]=collisions ([0] set by emit)
  unsigned long long* block_sums; // matches per kEmitTiles consecutive tiles
  uint32_t* tile_info;            // per sequence number: matches | chunk bitmap << 16
  uint32_t* masks;                // per sequence number: kTileChunks x 32 lane hit masks
  PatWords pw;
  uint32_t warps;                 // warps per CTA launched (<= scan_warps(m): small scans
                                  // spread one or a few warps over every SM)
  uint32_t hx_is_pattern;         // hx == hash_full(pattern): equal bytes imply a hash hit
};
// Shape of the scan kernel per pattern length: m >= 15 (the running fold, the least work
// per byte) streams 8 KiB stages -- one TMA copy and one ring hand-off per tile -- with 12
// warps per SM; the shorter paths keep 4 KiB stages and more warps per SM, the latency
// cover their longer per-byte work needs.
#ifndef RK_PDL
#define RK_PDL 1  // programmatic dependent launch of the scan and emit grids
#endif
#ifndef RK_WIDE_FROM
#define RK_WIDE_FROM 15
#endif
#ifndef RK_WIDE_W
#define RK_WIDE_W 12
#define RK_WIDE_S 8
#define RK_WIDE_B 1
#endif
#ifndef RK_BASE_W
#define RK_BASE_W 12
#define RK_BASE_S 4
#define RK_BASE_B 2
#endif
struct ScanShape {
  int warps, stage_chunks, min_blocks;
};
constexpr uint32_t kWideFrom = RK_WIDE_FROM;  // first m with the wide shape
// measured per length (tools/ab.sh): m = 8 likes 20 warps in one CTA, m = 5..7 two CTAs
// of 8 warps (the two dependent dp4a per window want warps; the cooperative settle's
// chunk-end ballots want smaller CTAs)
// short-pattern shapes (warps, stage chunks, CTAs per SM); separate macros because nvcc
// splits -D values at commas
#ifndef RK_S8_W
#define RK_S8_W 20
#define RK_S8_S 4
#define RK_S8_B 1
#endif
#ifndef RK_S57_W
#define RK_S57_W 20  // (measured: 8 x 2 CTAs 5121 / 4921 / 5280 GB/s at m = 5 / 6 / 7,
#define RK_S57_S 4   //  12 x 2 5312 / 5081 / 5609, 20 x 1 5361 / 5169 / 5556)
#define RK_S57_B 1
#endif
#ifndef RK_S34_W
#define RK_S34_W RK_BASE_W
#define RK_S34_S RK_BASE_S
#define RK_S34_B RK_BASE_B
#endif
__host__ __device__ constexpr ScanShape scan_shape(uint32_t m) {
  return m >= kWideFrom ? ScanShape{RK_WIDE_W, RK_WIDE_S, RK_WIDE_B}
         : m == 8       ? ScanShape{RK_S8_W, RK_S8_S, RK_S8_B}
         : (m >= 5 && m <= 7) ? ScanShape{RK_S57_W, RK_S57_S, RK_S57_B}
         : (m >= 3 && m <= 4) ? ScanShape{RK_S34_W, RK_S34_S, RK_S34_B}
                              : ScanShape{RK_BASE_W, RK_BASE_S, RK_BASE_B};
}
__host__ __device__ constexpr int scan_warps(uint32_t m) { return scan_shape(m).warps; }
__host__ __device__ constexpr int scan_stage_chunks(uint32_t m) { return scan_shape(m).stage_chunks; }
__host__ __device__ constexpr int scan_min_blocks(uint32_t m) { return scan_shape(m).min_blocks; }
size_t scan_smem_bytes(uint32_t m);
int scan_blocks_per_sm(uint32_t m);
cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t s);

// ordered emission (rk_emit.cu)
// A tile with at least this many matches is "dense": the emit queues such tiles for a
// dynamically balanced phase when the scan flagged counters[3] (some warp matched this
// many in all; rk_emit.cu; 0: off).
#ifndef RK_EMIT_DEFER_MIN
#define RK_EMIT_DEFER_MIN 1024
#endif
constexpr uint32_t kDeferMin = RK_EMIT_DEFER_MIN;

struct EmitArgs {
  const uint32_t* tile_info;
  const uint32_t* masks;
  const unsigned long long* block_sums;
  uint64_t num_tiles;   // sequence numbers of the logical scan
  uint64_t tile0;       // a-space tile index of sequence number 0
  int64_t start_bias;   // written value = a-space end position + start_bias
  int64_t* out;
  uint64_t cap;
  unsigned long long* counters;    // [0] <- total matches ([1], [2] from the scan)
  unsigned long long* counts_out;  // optional: {matches, hash_hits, collisions}
  unsigned long long* clear;       // the other counter set, zeroed for the next scan
  uint64_t clear_words;
  uint32_t* bitmap;                // bitmap mode: bit (end position + bit_bias) per match
  int64_t bit_bias;
  uint64_t tiles_per_block;        // set by launch_emit
  // queue of dense tiles for the balanced second phase (all zero between emits):
  // work = {ticket, queued, blocks done, blocks out}; queue[i] = (excl + 1) << 22 | tile
  // (one word: read with a relaxed load, no acquire -- whose L1 invalidation per entry
  // stalled the stores); capacity >= num_tiles (< 2^22 whenever the queue is used)
  unsigned long long* work;
  unsigned long long* queue;
  uint32_t defer_min;              // set by launch_emit (0: no queue)
};
cudaError_t launch_emit(EmitArgs e, int num_sms, cudaStream_t s);

// multi pattern (rk_multi.cu, kernels in rk_multi_impl.cuh)
constexpr int kMultiFilterWords = (1 << 16) / 32;
#ifndef RK_QFILTER_LOG2_BITS
#define RK_QFILTER_LOG2_BITS 19  // q-gram Bloom filter of 2^19 bits = 64 KiB
#endif
constexpr int kQFilterWords = (1 << RK_QFILTER_LOG2_BITS) / 32;
constexpr int kQBlockShift = 32 - (RK_QFILTER_LOG2_BITS - 6);  // h >> this = 64-bit block
constexpr int kQWordShift = 32 - (RK_QFILTER_LOG2_BITS - 5);   // h >> this = 32-bit word
constexpr uint32_t kMultiEmpty = 0xffffffffu;

// Blocked Bloom filter of q-grams of QW = 1..4 little-endian words: 8192 blocks of 64
// bits (64 KiB), one block per q-gram, 2 bits in each 32-bit half -- one 8-byte
// shared-memory load per test.  (Simulated on C3's q-grams: 0.024% false positives
// against 0.095% for a 2-probe filter of the same size.)  The same hash runs on the host
// (filter build) and the device (text q-grams): block = h >> 19, bit positions
// h, h >> 5 (low half) and h >> 10, h >> 15 (high half), each mod 32.
template <int QW>
__host__ __device__ __forceinline__ uint32_t qgram_hash(const uint32_t* w) {
  const uint32_t C[4] = {0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du, 0x165667B1u};
  uint32_t h = w[0] * C[0];
  for (int i = 1; i < QW; ++i) h += w[i] * C[i];
  return h ^ (h >> 15);
}

// Lengths < 7 (rk_multi_short_kernel): a window of length L <= 6 is its own exact key.
// One sweep takes every such length of a set (lengths 4..6 in one "anchored" sweep,
// lengths 1..3 in one per-window sweep); its patterns sit in ONE cuckoo table keyed by
// (bytes, length): slot = bytes (48 bits) | L << 48 (3 bits) | caller index << 51
// (12 bits), empty = ~0.  The two slots of a key come from tiny_key_hash of the low word
// and the tagged high word (bytes 4..5 | L << 16), for the same function on the host
// (build) and the device (lookup).
struct TinyHash {
  uint32_t c1, c2, c3;  // seeds (the host retries others if an insertion cycles)
  uint32_t shift;       // 32 - log2(size)
  uint32_t size;        // slots, a power of two
};
constexpr uint32_t kTinySlotsMax = 8192;  // 64 KiB of shared memory (2 slots per pattern)
constexpr uint64_t kShortKeyMask = (1ull << 51) - 1;  // bytes + length
__host__ __device__ __forceinline__ uint32_t short_tag(uint32_t hi_bytes, uint32_t len) {
  return hi_bytes | (len << 16);
}
__host__ __device__ __forceinline__ uint64_t short_key(uint32_t lo, uint32_t hi_bytes,
                                                       uint32_t len) {
  return (uint64_t)lo | ((uint64_t)hi_bytes << 32) | ((uint64_t)len << 48);
}
__host__ __device__ __forceinline__ uint32_t tiny_key_hash(uint32_t lo, uint32_t tag,
                                                           const TinyHash& t) {
  return lo * t.c1 + tag * t.c2;
}
__host__ __device__ __forceinline__ void tiny_slots(uint32_t f, const TinyHash& t, uint32_t& s1,
                                                    uint32_t& s2) {
  s1 = f >> t.shift;
  s2 = ((f ^ (f >> 15)) * t.c3) >> t.shift;
}
// The sweep's Bloom filter: 8192 32-bit words (32 KiB).  An entry x (an anchored q-gram's
// bytes as a little-endian word, or a per-window sweep's tiny_key_hash) is mixed as
// h = umulhi(x * kGramMul, kFiltMix) and sets bits h, h >> 5 and h >> 10 (mod 32) of word
// h >> 19: one 32-bit shared-memory load per test, two or three bits (short_filter_bits).  The mixing multiplies run on the FMA pipe and leave the bit positions in
// the low bits, where the test's rotates take them without masking.
#ifndef RK_SHORT_FILTER_LOG2_WORDS
#define RK_SHORT_FILTER_LOG2_WORDS 13  // 8192 words = 32 KiB (16 KiB: 1024 x m = 5 -13%)
#endif
constexpr uint32_t kShortFilterWords = 1u << RK_SHORT_FILTER_LOG2_WORDS;
constexpr uint32_t kGramMul = 0x9E3779B1u;
// bits per entry: 2 for 3-gram sweeps (q = 3, i.e. a set with length 4: its text 3-grams
// match the patterns' for real ~1/400 anchors, so more bits only cost instructions; 1024 x
// m = 4: 2.72 -> 2.62 ms), 3 otherwise (1024 x m = 5: 1.92 -> 1.79 ms)
// 3-gram sweeps also hold every pattern's first 4 bytes ^ this salt in their filter: a
// passing anchor's windows are tested on their prefixes before the settle
#ifndef RK_SHORT_KEY_REFINE
#define RK_SHORT_KEY_REFINE 1
#endif
constexpr uint32_t kShortKeySalt = 0x5BD1E995u;
#ifndef RK_SHORT_Q4_BITS
#define RK_SHORT_Q4_BITS 3
#endif
__host__ __device__ constexpr uint32_t short_filter_bits(uint32_t q) {
  return q == 3 ? 2u : (q == 4 ? (uint32_t)RK_SHORT_Q4_BITS : 3u);
}
// anchored sweeps whose passing anchors are refined on the windows' 4-byte prefixes
__host__ __device__ constexpr bool short_refined(uint32_t q) {
  return RK_SHORT_KEY_REFINE && (q == 3 || (q == 4 && RK_SHORT_Q4_BITS == 2));
}

__host__ __device__ __forceinline__ uint32_t short_filter_hash(uint32_t x) {
  // both halves of the 64-bit product: every bit depends on every input bit
  const uint64_t p = (uint64_t)x * kGramMul;
  return (uint32_t)p + (uint32_t)(p >> 32);
}
__host__ __device__ __forceinline__ uint32_t short_filter_word(uint32_t h) {
  return h >> (32 - RK_SHORT_FILTER_LOG2_WORDS);
}
// The bits an entry with hash h sets in its filter word: h, h >> 5 (and h >> 10), mod 32.
inline uint32_t short_filter_bit_set(uint32_t h, uint32_t bits) {
  const auto rot = [](uint32_t b) { return 1u << (b & 31); };
  return rot(h) | rot(h >> 5) | (bits == 3 ? rot(h >> 10) : 0u);
}
// anchored sweeps: anchors every 2 bytes, q-gram length q = 3 when the sweep has length 4
// (q + 2 - 1 <= m), else 4; an occurrence at y holds the q-gram ending at the first anchor
// e >= y + q - 1, i.e. p[j:j+q] with j in {0, 1}
__host__ __device__ constexpr int short_gram_q(int m_min) { return m_min == 4 ? 3 : 4; }

// One length group of a multi-pattern launch (all arrays device-resident).
struct MultiGroup {
  const uint8_t* pats;     // P_g * m bytes, the group's patterns back to back
  const uint64_t* phash;   // 64-bit hash per pattern
  const uint32_t* order;   // group-local pattern indices, grouped by low-32 key
  const uint32_t* gidx;    // group-local index -> the caller's pattern index
  const uint2* table;      // tsize entries: {key, (first << 13) | count}, y = empty marker
  const uint32_t* filter;  // kMultiFilterWords words over the low-32 keys
  uint64_t ys_hi;          // one past the last window start with room for m bytes (a-space)
  uint32_t m, tsize, P;
};
constexpr int kMultiMaxGroups = 64;  // length groups per sweep (kernel parameter space)
#ifndef RK_MULTI_WARPS
#define RK_MULTI_WARPS 16
#define RK_MULTI_STAGE 4
#endif
// one 16-warp CTA per SM shares the 64 KiB q-gram filter, 4 KiB TMA stages (measured
// against 20/24/32 warps with 2 KiB stages: C3 5.23 against 3.64/5.20/4.52 TB/s)
constexpr int kMultiWarps = RK_MULTI_WARPS;
constexpr int kMultiStageChunks = RK_MULTI_STAGE;

struct MultiArgs {
  TextGeom g;                 // q-gram mode: tiles cover the anchors (q-gram ends)
  const uint32_t* qfilter;    // kQFilterWords words (q-gram mode)
  uint32_t qmode;             // sampling step s (8 or 4), 0 = per-window filter (m < 7)
  uint32_t qwords;            // q-gram length in words (q = 4 * qwords)
  uint32_t qf32;              // filter layout: 32-bit words (1) or 64-bit blocks (0)
  uint64_t ys_lo;             // first window start the sweep reports, a-space
  int64_t out_bias;           // added to every reported offset (shards)
  int64_t* out_off;
  uint32_t* out_idx;
  uint64_t cap;
  unsigned long long* counters;  // [0] = pairs found
  const uint4* qmap;             // q-gram hash -> length-group mask (qmode > 0)
  uint32_t qmap_size;            // entries, a power of two
  uint32_t G;                    // length groups in grp
  // short sweeps (qmode == 0): the sweep's cuckoo table (tsize slots) followed by its
  // filter (kShortFilterWords words), and the anchored q-gram length (0: per window)
  const uint8_t* stab;
  TinyHash th;
  uint32_t sq;
  // pairs each warp buffers in shared memory before one atomic reserves their slots (the
  // shared memory the kernel leaves over; 0: one atomic per warp per round)
  uint32_t append_cap;
  MultiGroup grp[kMultiMaxGroups];
};
constexpr size_t kMultiSmemMax = 227 * 1024;  // the sm_100 opt-in per block
__host__ __device__ constexpr uint32_t multi_append_stride(uint32_t cap) {
  return cap ? 16u + 12u * cap : 0u;  // per warp: count (16 B), offsets, indices
}
size_t multi_smem_bytes(uint32_t append_cap);
size_t multi_short_smem_bytes(uint32_t slots, uint32_t append_cap);
void multi_set_append(MultiArgs& a);  // a.append_cap from the kernel's other shared memory
int multi_blocks_per_sm(const MultiArgs& a);
cudaError_t launch_multi(const MultiArgs& a, int grid, cudaStream_t s);

// device ordering of (pattern index, offset) pairs (rk_pairs.cu)
size_t sort_pairs_scratch(uint64_t k);
constexpr uint64_t kSmallSort = 4096;  // pairs ordered by one block (rk_pairs.cu)
cudaError_t small_sort_pairs(int64_t* d_off, uint32_t* d_idx, const unsigned long long* d_count,
                             uint64_t k_host, uint64_t cap, uint64_t n,
                             unsigned long long* count_out, cudaStream_t s);
cudaError_t sort_pairs(int64_t* d_off, uint32_t* d_idx, uint64_t k, uint64_t n, uint32_t P,
                       void* scratch, size_t scratch_bytes, cudaStream_t s);

// auxiliaries (rk_aux.cu)
cudaError_t launch_window_hashes(const uint8_t* text, uint64_t n, uint32_t m, uint64_t start,
                                 uint64_t stop, uint64_t* out, cudaStream_t s);
cudaError_t launch_generate(uint8_t* out, uint64_t count, uint64_t seed, uint64_t skip,
                            const uint8_t* alphabet, uint32_t k, cudaStream_t s);

}  // namespace rkb
