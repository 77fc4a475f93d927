// rk_scan_g1.cu -- explicit instantiations of the single-pattern scan for m in
// {9, 10, 11, 12, 13, 14, 15, 16} (m = 32 stands for every m >= 32).  The 32 variants are split
// over four translation units to keep each ptxas run small and the build parallel.
#include "rk_short_impl.cuh"

namespace rkb {
template cudaError_t launch_m<9>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<9>();
template cudaError_t launch_m<10>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<10>();
template cudaError_t launch_m<11>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<11>();
template cudaError_t launch_m<12>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<12>();
template cudaError_t launch_m<13>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<13>();
template cudaError_t launch_m<14>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<14>();
template cudaError_t launch_m<15>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<15>();
template cudaError_t launch_m<16>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<16>();
}  // namespace rkb
