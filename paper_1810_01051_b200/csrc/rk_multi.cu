// rk_multi.cu -- dispatch of the multi-pattern scan variants (instantiated in
// rk_multi_g0..3.cu, kernels in rk_multi_impl.cuh).
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

template <int M>
cudaError_t launch_multi_m(const MultiArgs& a, int grid, cudaStream_t s);
template <int M>
int multi_occupancy_m(uint32_t tsize);

using MultiLaunchFn = cudaError_t (*)(const MultiArgs&, int, cudaStream_t);
using MultiOccFn = int (*)(uint32_t);
template <int... Ms>
struct MultiTable {
  static constexpr MultiLaunchFn launch[sizeof...(Ms)] = {&launch_multi_m<Ms>...};
  static constexpr MultiOccFn occ[sizeof...(Ms)] = {&multi_occupancy_m<Ms>...};
};
using MTable = MultiTable<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                          21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32>;

static int mvariant(uint32_t m) { return m >= 32 ? 31 : (int)m - 1; }

size_t multi_smem_bytes(uint32_t) {
  return sizeof(WarpRing) * 16 + kQFilterWords * sizeof(uint32_t);
}

int multi_blocks_per_sm(uint32_t m, uint32_t tsize) { return MTable::occ[mvariant(m)](tsize); }

cudaError_t launch_multi(const MultiArgs& a, int grid, cudaStream_t s) {
  return MTable::launch[mvariant(a.g.m)](a, grid, s);
}

}  // namespace rkb
