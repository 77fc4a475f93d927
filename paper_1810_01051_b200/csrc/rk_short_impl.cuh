// rk_short_impl.cuh -- the single-pattern scan for 2 <= m <= 8 (the reference's
// _scan_range, /root/reference/pkg/src/rkmatch/_scan.py:28-50, for short patterns).
//
// For m <= 8 the 64-bit hash of a window is < 2^16 and is a dot product of the window's
// (at most two) 4-byte words with the weights 2^(m-1-i) (rkhash.py:21-28), so there is no
// roll chain: per window one funnel shift (the window's word, shared with its neighbours)
// and one or two dp4a that also subtract hx give d = hash - hx.  What makes short patterns
// expensive is not that core (~2.8 instructions per window at m = 4) but the hash HITS:
// at m = 4 over printable ASCII ~0.8 windows per KiB hash to hx, and they must all be
// counted (ScanStats.hash_hits / collisions) and byte-verified exactly.
//
// Structure, per 1 KiB chunk of the TMA stage (rk_device.cuh's per-warp ring):
//   fast pass   every lane tests its 32 windows for d == 0 -- only "any", one accumulated
//               predicate (m <= 4: the d's multiplied in pairs, exact since |d| < 2^12)
//   vote        one ballot; a chunk with no flagged lane costs nothing more
//   settle      each flagged lane is settled by the whole warp straight from shared
//               memory: lane i takes window i of the flagged lane's 32, recomputes d, checks
//               validity and bytes; two ballots give the hits and the match mask
//   dense       a chunk with more than kShortCoopLanes flagged lanes (dense matches, C5's
//               all-'a') is settled per lane from registers instead, and the warp stays in
//               that mode while the density lasts
// Everything the loop needs per chunk (the lane's shared-memory address, -hx, the dp4a
// weights) is computed once per kernel, so the fast pass is the core plus ~8 instructions.
#pragma once
#include "rk_scan_impl.cuh"

namespace rkb {

#ifndef RK_SHORT_PAIRS_TO
#define RK_SHORT_PAIRS_TO 4  // m <= this: windows' d's tested in products of two
#endif
#ifndef RK_SHORT_COOP_LANES
#define RK_SHORT_COOP_LANES 6  // a chunk with more flagged lanes is settled per lane
#endif
constexpr int kShortCoopLanes = RK_SHORT_COOP_LANES;

// d = hash - hx of the 32 windows ending in the lane's bytes; true if some d is 0
template <int M>
__device__ __forceinline__ bool short_flag(uint32_t negT, uint32_t lb6, uint32_t lb7,
                                           const Vec32& v) {
  constexpr uint32_t W0 = win_weights<M>(0), W1 = win_weights<M>(1);
  uint32_t lb[8];
#pragma unroll
  for (int i = 0; i < 6; ++i) lb[i] = 0;
  lb[6] = lb6;
  lb[7] = lb7;
  uint32_t d[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int s0 = 33 + k - M;  // window start within lb ++ v (>= 25: lb[6..7] only)
    if constexpr (M > 4) {
      d[k] = __dp4a(w64(lb, v, s0), W0, __dp4a(w64(lb, v, s0 + 4), W1, negT));
    } else {
      d[k] = __dp4a(w64(lb, v, s0), W0, negT);
    }
  }
  bool any = false;
  if constexpr (M <= RK_SHORT_PAIRS_TO) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) any |= (d[k] * d[k + 1] == 0u);
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) any |= (d[k] == 0u);
  }
  return any;
}

// the lane's 8 bytes before its first window end (lb[6..7]) and its 32 bytes (v), from
// the stage in shared memory at p (the lane's 32-byte lookback)
__device__ __forceinline__ void lds_chunk(uint32_t p, uint32_t& lb6, uint32_t& lb7, Vec32& v) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lb6), "=r"(lb7) : "r"(p + 24));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]) : "r"(p + 32));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]), "=r"(v.w[7]) : "r"(p + 48));
}

// acc += p, as one predicated add
__device__ __forceinline__ void add_if(uint32_t& acc, bool p) {
  asm("{.reg .pred q;\n setp.ne.b32 q, %1, 0;\n @q add.u32 %0, %0, 1;}"
      : "+r"(acc) : "r"((uint32_t)p));
}

template <int M>
__global__ void __launch_bounds__(32 * scan_warps(M), scan_min_blocks(M))
    rk_short_kernel(const ScanArgs a) {
  static_assert(M >= 2 && M <= 8, "short kernel");
  constexpr int kWarps = scan_warps(M);
  constexpr int SC = scan_stage_chunks(M);
  using Ring = WarpRingT<SC>;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  Ring* R = reinterpret_cast<Ring*>(smem) + warp;
  uint32_t* scratch =
      reinterpret_cast<uint32_t*>(smem + kWarps * sizeof(Ring)) + warp * kScratchWords;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * a.warps;
  const uint64_t w = (uint64_t)blockIdx.x * a.warps + warp;
  const TextGeom& g = a.g;
  Stream S;
  stream_init(g, R, S, (uint32_t)w, (uint32_t)W, lane);
  WarpTotals tot;

  // loop invariants
  const uint32_t negT = 0u - (uint32_t)a.hx;
  constexpr uint32_t W0 = win_weights<M>(0), W1 = win_weights<M>(1);
  constexpr uint32_t K0 = M >= 4 ? 0xffffffffu : ((1u << (8 * M)) - 1u);
  constexpr uint32_t K1 = M >= 8 ? 0xffffffffu : M > 4 ? ((1u << (8 * (M - 4))) - 1u) : 0u;
  const uint32_t P0 = a.pw.w[0], P1 = a.pw.w[1];
  const uint32_t lane_s = smem_u32(R->buf[0]) + (uint32_t)lane * kR;  // lane's bytes, slot 0
  // settle: lane i takes the window ending at byte 32 + i of the flagged lane's 64 bytes
  // (its 32-byte lookback ++ its 32 bytes), i.e. starting at byte 33 + i - M
  const uint32_t soff = 33u + (uint32_t)lane - M, sr = 8u * (soff & 3u);
  const uint32_t settle_s = smem_u32(R->buf[0]) + (soff & ~3u);
  bool dense = false;  // warp-uniform

  for (uint32_t t = (uint32_t)w; t < (uint32_t)g.num_tiles; t += (uint32_t)W) {
    const uint64_t seq = g.seq_base + t;
    uint32_t* tmask = a.masks + seq * (kTileChunks * 32);
    const int64_t ta = g.tile_a(t);
    uint32_t hitflags = 0, my_matches = 0, my_hits = 0;
    // every window of the tile is in the launch's range (most tiles)
    uint32_t full_u = ta >= (int64_t)g.ja_lo && ta + kTile <= (int64_t)g.ja_hi;
    asm volatile("" : "+r"(full_u));
    const bool full = full_u != 0u;
    // per-lane inline settle of one chunk (dense chunks, edge tiles)
    const auto inline_settle = [&](const Vec32& v, const uint32_t (&lb)[8], int64_t J, int c) {
      uint32_t hm = 0, hits = 0;
      if (dense && full && a.hx_is_pattern) {
        // a dense run (C5's all-'a'): when every window of the chunk equals the pattern --
        // bytes alone, since hx is the pattern's hash -- the chunk is 1024 matches
        bool all = true;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int s0 = 33 + k - M;
          all &= (w64(lb, v, s0) & K0) == P0;
          if constexpr (M > 4) all &= (w64(lb, v, s0 + 4) & K1) == P1;
        }
        if (__all_sync(kFull, all)) {
          my_hits += 32;
          my_matches += 32;
          tmask[c * 32 + lane] = 0xffffffffu;
          hitflags |= 1u << c;
          return;
        }
      }
      if (dense) {
        short_chunk<M, true>(a, v, lb, full, full ? 0xffffffffu : valid_mask(g, J), hm, hits);
      } else {
        short_chunk<M, false>(a, v, lb, full, full ? 0xffffffffu : valid_mask(g, J), hm, hits);
      }
      dense = __popc(__ballot_sync(kFull, hits != 0)) > kShortCoopLanes;
      my_hits += hits;
      my_matches += __popc(hm);
      if (__ballot_sync(kFull, hm != 0)) {
        tmask[c * 32 + lane] = hm;
        hitflags |= 1u << c;
      }
    };
    if (t >= S.int_lo && t < S.int_hi) {
#pragma unroll 1
      for (int s = 0; s < kTileChunks / SC; ++s) {
        mbar_wait(&R->bar[S.cslot], S.cphase);
        const uint32_t slot_off = S.cslot * (uint32_t)Ring::kBytes;
        const uint32_t stage_p = lane_s + slot_off;  // the lane's lookback in chunk 0
        // fast pass over the stage's SC chunks, unrolled, with nothing but the flag
        // votes in it; the (rare) settle work follows in one rolled loop
        const bool sd = dense;
        uint32_t f[SC];
        uint32_t anyf = 0;
        if (!sd) {
#pragma unroll
          for (int j = 0; j < SC; ++j) {
            uint32_t lb6, lb7;
            Vec32 v;
            lds_chunk(stage_p + (uint32_t)j * kChunk, lb6, lb7, v);
            f[j] = __ballot_sync(kFull, short_flag<M>(negT, lb6, lb7, v));
            anyf |= f[j];
          }
        }
        // settle: flagged chunks of a full tile with few flagged lanes cooperatively, in
        // the unrolled order (no dynamic selection of f[j]); dense chunks, dense mode and
        // partial tiles per lane, in one rolled loop (one copy of that code)
        uint32_t im = sd ? (1u << SC) - 1u : 0u;
        if (!sd && anyf) {
#pragma unroll
          for (int j = 0; j < SC; ++j) {
            uint32_t flags = f[j];
            if (!flags) continue;
            if (!full || __popc(flags) > kShortCoopLanes) {
              im |= 1u << j;
              continue;
            }
            const int c = s * SC + j;
            const uint32_t base = settle_s + slot_off + (uint32_t)j * kChunk;
            uint32_t hm = 0;
            do {
              const int L = __ffs(flags) - 1;
              flags &= flags - 1;
              const uint32_t q = base + 32u * L;
              const uint32_t x1 = lds_u32(q + 4);
              const uint32_t A = __funnelshift_r(lds_u32(q), x1, sr);
              uint32_t d, B = 0;
              if constexpr (M > 4) {
                B = __funnelshift_r(x1, lds_u32(q + 8), sr);
                d = __dp4a(A, W0, __dp4a(B, W1, negT));
              } else {
                d = __dp4a(A, W0, negT);
              }
              const bool hit = d == 0u;
              const bool eq = hit & (((A ^ P0) & K0) == 0u) & (((B ^ P1) & K1) == 0u);
              add_if(my_hits, hit);
              add_if(my_matches, eq);
              const unsigned em = __ballot_sync(kFull, eq);
              hm = lane == L ? em : hm;
            } while (flags);
            if (__ballot_sync(kFull, hm != 0)) {
              tmask[c * 32 + lane] = hm;
              hitflags |= 1u << c;
            }
          }
        }
#pragma unroll 1
        while (im) {
          const int j = __ffs(im) - 1;
          im &= im - 1;
          const int c = s * SC + j;
          uint32_t lb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          Vec32 v;
          lds_chunk(stage_p + (uint32_t)j * kChunk, lb[6], lb[7], v);
          inline_settle(v, lb, ta + c * kChunk + lane * kR, c);
        }
        // the slot's bytes are consumed: hand it back to the producer
        S.cslot = (S.cslot + 1) & (kStages - 1);
        S.cphase ^= (S.cslot == 0);
        --S.pending;
        __syncwarp();
        stream_issue(R, S, lane);
      }
    } else {
      // edge tile (not staged): bounds-checked loads, per-lane settle
#pragma unroll 1
      for (int c = 0; c < kTileChunks; ++c) {
        const int64_t J = ta + c * kChunk + lane * kR;
        const Vec32 v = load_edge(g, J);
        const Vec32 l = load_edge(g, J - 32);
        uint32_t lb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) lb[i] = l.w[i];
        uint32_t hm = 0, hits = 0;
        short_chunk<M, false>(a, v, lb, false, valid_mask(g, J), hm, hits);
        my_hits += hits;
        my_matches += __popc(hm);
        if (__ballot_sync(kFull, hm != 0)) {
          tmask[c * 32 + lane] = hm;
          hitflags |= 1u << c;
        }
      }
    }
    record_tile(a, seq, my_matches, my_hits, hitflags, lane, tot);
    (void)scratch;
  }
  flush_totals(a, tot, lane);
}

// ---------------------------------------------------------------------------------
// Launch of the scan variant of pattern length M (3 <= M <= 8: rk_short_kernel above,
// else rk_scan_kernel of rk_scan_impl.cuh).  Measured against rk_scan_kernel's inline
// settle (tools/ab.sh, C2 corpus, GB/s): m = 3 3789 / 3534, 4 5431 / 4906, 5 5120 / 4833,
// 6 4940 / 4655, 7 5236 / 5056, 8 5748 / 5430; m = 2 2189 / 2471 stays on the inline
// settle.
#ifndef RK_SHORT_KERNEL
#define RK_SHORT_KERNEL 1
#endif
#ifndef RK_SHORT_FROM
#define RK_SHORT_FROM 3  // m = 2: hits are so frequent (~1/256) that the inline settle wins
#endif
template <int M>
constexpr auto scan_kernel() {
  if constexpr (RK_SHORT_KERNEL && M >= RK_SHORT_FROM && M <= 8) {
    return &rk_short_kernel<M>;
  } else {
    return &rk_scan_kernel<M>;
  }
}

template <int M>
cudaError_t launch_m(const ScanArgs& a, int grid, cudaStream_t s) {
  const size_t smem = scan_smem_bytes(M);
  static bool attr[kMaxDevices] = {};  // per-variant, per-device opt-in to > 48 KiB smem
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(scan_kernel<M>(),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDevices) attr[dev] = true;
  }
  // programmatic dependent launch: scheduled as the previous kernel's CTAs retire; the
  // kernel waits for that grid's completion before touching memory (griddepcontrol.wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(32 * a.warps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = RK_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, scan_kernel<M>(), a);
}

template <int M>
int occupancy_m() {
  cudaFuncSetAttribute(scan_kernel<M>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)scan_smem_bytes(M));
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, scan_kernel<M>(), 32 * scan_warps(M),
                                                scan_smem_bytes(M));
  return b > 0 ? b : 1;
}

}  // namespace rkb
