// rk_multi.cu -- dispatch of the multi-pattern scan kernels (m < 7 variants instantiated
// in rk_multi_g0.cu; kernels in rk_multi_impl.cuh).
#include "rk_multi_impl.cuh"

namespace rkb {

// Every length >= 7 of the set in one sweep: anchored q-grams against the shared filter.
__global__ void __launch_bounds__(kMultiBlock) rk_multi_qgram_kernel(const __grid_constant__ MultiArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  MultiRing* rings = reinterpret_cast<MultiRing*>(smem);
  uint32_t* sfilter = reinterpret_cast<uint32_t*>(smem + sizeof(MultiRing) * kMultiWarps);
  for (int i = threadIdx.x; i < kQFilterWords; i += blockDim.x) sfilter[i] = a.qfilter[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  MultiRing* R = rings + warp;
  ring_init(R, lane);
  const uint64_t W = (uint64_t)gridDim.x * kMultiWarps;
  const uint64_t w = (uint64_t)blockIdx.x * kMultiWarps + warp;
  Stream S;
  stream_init(a.g, R, S, (uint32_t)w, (uint32_t)W, lane);
  const int s = (int)a.qmode;
  for (uint32_t t = (uint32_t)w; t < (uint32_t)a.g.num_tiles; t += (uint32_t)W) {
    switch (s * 8 + (int)a.qwords) {
      case 8 * 8 + 4: qgram_tile<8, 4>(a, R, S, t, lane, sfilter); break;
      case 8 * 8 + 2: qgram_tile<8, 2>(a, R, S, t, lane, sfilter); break;
      case 4 * 8 + 3: qgram_tile<4, 3>(a, R, S, t, lane, sfilter); break;
      case 4 * 8 + 2: qgram_tile<4, 2>(a, R, S, t, lane, sfilter); break;
      default: qgram_tile<4, 1>(a, R, S, t, lane, sfilter); break;
    }
  }
}

template <int M>
cudaError_t launch_multi_tiny(const MultiArgs& a, int grid, cudaStream_t s);
template <int M>
int multi_tiny_occupancy();

using MultiLaunchFn = cudaError_t (*)(const MultiArgs&, int, cudaStream_t);
using MultiOccFn = int (*)();
static constexpr MultiLaunchFn kTinyLaunch[6] = {
    &launch_multi_tiny<1>, &launch_multi_tiny<2>, &launch_multi_tiny<3>,
    &launch_multi_tiny<4>, &launch_multi_tiny<5>, &launch_multi_tiny<6>};
static constexpr MultiOccFn kTinyOcc[6] = {
    &multi_tiny_occupancy<1>, &multi_tiny_occupancy<2>, &multi_tiny_occupancy<3>,
    &multi_tiny_occupancy<4>, &multi_tiny_occupancy<5>, &multi_tiny_occupancy<6>};

size_t multi_smem_bytes() {
  return sizeof(MultiRing) * kMultiWarps + kQFilterWords * sizeof(uint32_t);
}

size_t multi_tiny_smem_bytes() {  // rings + the largest cuckoo table
  return sizeof(MultiRing) * kMultiWarps + kTinySlotsMax * 8u + kTinyFilterBytes;
}

int multi_blocks_per_sm(uint32_t qmode, uint32_t m) {
  if (qmode == 0) return kTinyOcc[m - 1]();
  static int occ = 0;  // same on every B200
  if (!occ) occ = multi_occupancy(rk_multi_qgram_kernel, multi_smem_bytes());
  return occ;
}

cudaError_t launch_multi(const MultiArgs& a, int grid, cudaStream_t s) {
  if (a.qmode == 0) return kTinyLaunch[a.g.m - 1](a, grid, s);
  return multi_launch_kernel<struct QgramAttr>(rk_multi_qgram_kernel, a, grid,
                                               multi_smem_bytes(), s);
}

}  // namespace rkb
