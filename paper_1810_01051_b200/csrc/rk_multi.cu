// rk_multi.cu -- dispatch of the multi-pattern scan kernels (the short-length variants
// instantiated in rk_multi_g0.cu; kernels in rk_multi_impl.cuh).
#include <algorithm>

#include "rk_multi_impl.cuh"

namespace rkb {

// Every length >= 7 of the set in one sweep: anchored q-grams against the shared filter.
__global__ void __launch_bounds__(kMultiBlock) rk_multi_qgram_kernel(const __grid_constant__ MultiArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  MultiRing* rings = reinterpret_cast<MultiRing*>(smem);
  uint32_t* sfilter = reinterpret_cast<uint32_t*>(smem + sizeof(MultiRing) * kMultiWarps +
                                                  kMultiWarps * multi_append_stride(a.append_cap));
  for (int i = threadIdx.x; i < kQFilterWords; i += blockDim.x) sfilter[i] = a.qfilter[i];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  multi_append_init(a, lane);
  __syncthreads();

  MultiRing* R = rings + warp;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * kMultiWarps;
  const uint64_t w = (uint64_t)blockIdx.x * kMultiWarps + warp;
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  const int s = (int)a.qmode;
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    switch (s * 16 + (int)a.qwords * 2 + (int)a.qf32) {
      case 8 * 16 + 4 * 2: qgram_tile<8, 4, false>(a, R, S, t, lane, sfilter); break;
      case 8 * 16 + 2 * 2: qgram_tile<8, 2, false>(a, R, S, t, lane, sfilter); break;
      case 4 * 16 + 3 * 2: qgram_tile<4, 3, false>(a, R, S, t, lane, sfilter); break;
      case 4 * 16 + 2 * 2: qgram_tile<4, 2, false>(a, R, S, t, lane, sfilter); break;
      case 4 * 16 + 1 * 2: qgram_tile<4, 1, false>(a, R, S, t, lane, sfilter); break;
      case 8 * 16 + 4 * 2 + 1: qgram_tile<8, 4, true>(a, R, S, t, lane, sfilter); break;
      case 8 * 16 + 2 * 2 + 1: qgram_tile<8, 2, true>(a, R, S, t, lane, sfilter); break;
      case 4 * 16 + 3 * 2 + 1: qgram_tile<4, 3, true>(a, R, S, t, lane, sfilter); break;
      case 4 * 16 + 2 * 2 + 1: qgram_tile<4, 2, true>(a, R, S, t, lane, sfilter); break;
      default: qgram_tile<4, 1, true>(a, R, S, t, lane, sfilter); break;
    }
  }
  multi_flush(a, lane);
}

template <int Q>
cudaError_t launch_multi_short(const MultiArgs& a, int grid, cudaStream_t s);
template <int Q>
int multi_short_occupancy(size_t smem);

// rings, the append buffers, the shared filter
size_t multi_smem_bytes(uint32_t append_cap) {
  return sizeof(MultiRing) * kMultiWarps + kMultiWarps * multi_append_stride(append_cap) +
         kQFilterWords * sizeof(uint32_t);
}

// rings, the append buffers, the sweep's cuckoo table + filter
size_t multi_short_smem_bytes(uint32_t slots, uint32_t append_cap) {
  return sizeof(MultiRing) * kMultiWarps + kMultiWarps * multi_append_stride(append_cap) +
         slots * 8u + kShortFilterWords * 4u;
}

#ifndef RK_MULTI_APPEND_MAX
#define RK_MULTI_APPEND_MAX 256  // pairs per warp buffer (0: no buffering)
#endif
void multi_set_append(MultiArgs& a) {
  if (a.qmode) {  // the q-gram sweep appends directly (lengths >= 7 are rarely dense)
    a.append_cap = 0;
    return;
  }
  const size_t base = a.qmode ? multi_smem_bytes(0) : multi_short_smem_bytes(a.th.size, 0);
  const size_t room = base < kMultiSmemMax ? (kMultiSmemMax - base) / kMultiWarps : 0;
  uint32_t cap = room > 16 ? (uint32_t)((room - 16) / 12) & ~3u : 0u;
  cap = std::min<uint32_t>(cap, RK_MULTI_APPEND_MAX);
  a.append_cap = cap >= 32 ? cap : 0u;  // a buffer under one warp's worth is not worth it
}

int multi_blocks_per_sm(const MultiArgs& a) {
  if (a.qmode == 0) {
    static int occ[kTinySlotsMax * 2] = {};  // per table size (a power of two)
    const uint32_t k = a.th.size;
    if (!occ[k]) {
      MultiArgs t = a;
      multi_set_append(t);
      const size_t smem = multi_short_smem_bytes(k, t.append_cap);
      occ[k] = a.sq == 3 ? multi_short_occupancy<3>(smem)
               : a.sq == 4 ? multi_short_occupancy<4>(smem) : multi_short_occupancy<0>(smem);
    }
    return occ[k];
  }
  static int occ = 0;  // same on every B200
  if (!occ) occ = multi_occupancy(rk_multi_qgram_kernel, multi_smem_bytes(a.append_cap));
  return occ;
}

cudaError_t launch_multi(const MultiArgs& a, int grid, cudaStream_t s) {
  if (a.qmode == 0) {
    return a.sq == 3 ? launch_multi_short<3>(a, grid, s)
           : a.sq == 4 ? launch_multi_short<4>(a, grid, s) : launch_multi_short<0>(a, grid, s);
  }
  return multi_launch_kernel<struct QgramAttr>(rk_multi_qgram_kernel, a, grid,
                                               multi_smem_bytes(a.append_cap), s);
}

}  // namespace rkb
