// rk_emit.cu -- ordered emission of match offsets (the ordered concatenation of
// /root/reference/pkg/src/rkmatch/parallel.py:168-172, done on the device).
//
// The scan kernel never waits on other tiles: it leaves, per 16 KiB tile, its match
// count and chunk bitmap (tile_info), the per-lane hit masks of the chunks that matched
// (masks), and per-256-tile sums (block_sums).  This kernel turns that into the ordered
// int64 offsets: block b adds up block_sums[0..b), scans its 256 tile counts, and each
// warp expands the masks of its tiles that have matches into window starts written at
// their final positions -- ascending, deterministic, no sort.  Text bytes are not
// touched again, so for sparse matches this is a few microseconds.
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

__global__ void __launch_bounds__(kEmitTiles) rk_emit_kernel(const EmitArgs e) {
  __shared__ unsigned long long red[kEmitTiles / 32];
  __shared__ uint32_t wsum[kEmitTiles / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t b = blockIdx.x;

  unsigned long long pre = 0;
  for (uint64_t i = tid; i < b; i += kEmitTiles) pre += e.block_sums[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(kFull, pre, o);
  if (lane == 0) red[warp] = pre;

  const uint64_t seq = b * kEmitTiles + tid;
  const uint32_t info = seq < e.num_tiles ? e.tile_info[seq] : 0u;
  const uint32_t cnt = info & 0xffffu;
  const uint32_t inc = warp_incl_scan(cnt, lane);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  unsigned long long base = 0;
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kEmitTiles / 32; ++w) {
    base += red[w];
    if (w < warp) wpre += wsum[w];
  }
  const uint64_t excl = base + wpre + inc - cnt;
  if (seq == e.num_tiles - 1) e.counters[0] = excl + cnt;

  unsigned todo = __ballot_sync(kFull, cnt != 0);
  while (todo) {
    const int j = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint64_t tseq = b * kEmitTiles + warp * 32 + j;
    uint32_t flags = __shfl_sync(kFull, info, j) >> 16;
    uint64_t run = __shfl_sync(kFull, excl, j);
    const int64_t tile_a = (int64_t)((e.tile0 + tseq) * (uint64_t)kTile);
    const uint32_t* tm = e.masks + tseq * (kTileChunks * 32);
    while (flags) {
      const int c = __ffs(flags) - 1;
      flags &= flags - 1;
      uint32_t hm = tm[c * 32 + lane];
      const uint32_t n = __popc(hm);
      const uint32_t i2 = warp_incl_scan(n, lane);
      const uint32_t tot = __shfl_sync(kFull, i2, 31);
      uint64_t pos = run + i2 - n;
      const int64_t v0 = tile_a + c * kChunk + lane * kR + e.start_bias;
      while (hm) {
        const int k = __ffs(hm) - 1;
        hm &= hm - 1;
        if (pos < e.cap) e.out[pos] = v0 + k;
        ++pos;
      }
      run += tot;
    }
  }
}

cudaError_t launch_emit(const EmitArgs& e, cudaStream_t s) {
  const uint64_t blocks = (e.num_tiles + kEmitTiles - 1) / kEmitTiles;
  rk_emit_kernel<<<(unsigned)blocks, kEmitTiles, 0, s>>>(e);
  return cudaGetLastError();
}

}  // namespace rkb
