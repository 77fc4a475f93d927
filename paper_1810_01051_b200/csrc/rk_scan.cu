// rk_scan.cu -- dispatch of the single-pattern scan variants (instantiated in
// rk_scan_g0..3.cu, kernels in rk_scan_impl.cuh).
#include "rk_device.cuh"
#include "rk_internal.h"

namespace rkb {

template <int M>
cudaError_t launch_m(const ScanArgs& a, int grid, cudaStream_t s);
template <int M>
int occupancy_m();

using LaunchFn = cudaError_t (*)(const ScanArgs&, int, cudaStream_t);
using OccFn = int (*)();

template <int... Ms>
struct Table {
  static constexpr LaunchFn launch[sizeof...(Ms)] = {&launch_m<Ms>...};
  static constexpr OccFn occ[sizeof...(Ms)] = {&occupancy_m<Ms>...};
};
using ScanTable = Table<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                        21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32>;
static int variant_of(uint32_t m) { return m >= 32 ? 31 : (int)m - 1; }

size_t scan_smem_bytes(uint32_t m) {
  // per warp: its TMA ring + the short-pattern settle scratch (rk_scan_impl.cuh)
  const size_t scratch = 20 * sizeof(uint32_t);
  size_t b;
  switch (scan_stage_chunks(m)) {
    case 8: b = (sizeof(WarpRingT<8>) + scratch) * scan_warps(m); break;
    case 4: b = (sizeof(WarpRingT<4>) + scratch) * scan_warps(m); break;
    case 2: b = (sizeof(WarpRingT<2>) + scratch) * scan_warps(m); break;
    default: b = (sizeof(WarpRingT<1>) + scratch) * scan_warps(m); break;
  }
  return b;
}

int scan_blocks_per_sm(uint32_t m) {
  static int cache[32] = {0};  // same on every B200
  const int v = variant_of(m);
  if (!cache[v]) cache[v] = ScanTable::occ[v]();
  return cache[v];
}

cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t s) {
  return ScanTable::launch[variant_of(a.g.m)](a, grid, s);
}

}  // namespace rkb
