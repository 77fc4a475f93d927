// rk_multi_g0.cu -- explicit instantiations of the short-length (m < 7) multi-pattern
// kernel: anchored q-grams of 3 or 4 bytes, or per-window keys (Q = 0).
#include "rk_multi_impl.cuh"

namespace rkb {

template <int Q>
struct rk_multi_short_tag {};

template <int Q>
cudaError_t launch_multi_short(const MultiArgs& a, int grid, cudaStream_t s) {
  // the dynamic shared memory follows the sweep's table size; the opt-in covers the largest
  static bool attr[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(rk_multi_short_kernel<Q>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMultiSmemMax);
    if (e != cudaSuccess) return e;
    if (dev < kMaxDevices) attr[dev] = true;
  }
  rk_multi_short_kernel<Q><<<grid, kMultiBlock, multi_short_smem_bytes(a.th.size, a.append_cap),
                             s>>>(a);
  return cudaGetLastError();
}

template <int Q>
int multi_short_occupancy(size_t smem) {
  // (the opt-in stays at the largest table's size; only the query uses this one's)
  cudaFuncSetAttribute(rk_multi_short_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kMultiSmemMax);
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rk_multi_short_kernel<Q>, kMultiBlock, smem);
  return b > 0 ? b : 1;
}

template cudaError_t launch_multi_short<0>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<3>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<4>(const MultiArgs&, int, cudaStream_t);
template int multi_short_occupancy<0>(size_t);
template int multi_short_occupancy<3>(size_t);
template int multi_short_occupancy<4>(size_t);

}  // namespace rkb
