// rk_scan_g0.cu -- explicit instantiations of the single-pattern scan for m in
// {1, 2, 3, 4, 5, 6, 7, 8} (m = 32 stands for every m >= 32).  The 32 variants are split
// over four translation units to keep each ptxas run small and the build parallel.
#include "rk_short_impl.cuh"

namespace rkb {
template cudaError_t launch_m<1>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<1>();
template cudaError_t launch_m<2>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<2>();
template cudaError_t launch_m<3>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<3>();
template cudaError_t launch_m<4>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<4>();
template cudaError_t launch_m<5>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<5>();
template cudaError_t launch_m<6>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<6>();
template cudaError_t launch_m<7>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<7>();
template cudaError_t launch_m<8>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<8>();
}  // namespace rkb
