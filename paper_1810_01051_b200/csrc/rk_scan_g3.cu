// rk_scan_g3.cu -- explicit instantiations of the single-pattern scan for m in
// {25, 26, 27, 28, 29, 30, 31, 32} (m = 32 stands for every m >= 32).  The 32 variants are split
// over four translation units to keep each ptxas run small and the build parallel.
#include "rk_short_impl.cuh"

namespace rkb {
template cudaError_t launch_m<25>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<25>();
template cudaError_t launch_m<26>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<26>();
template cudaError_t launch_m<27>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<27>();
template cudaError_t launch_m<28>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<28>();
template cudaError_t launch_m<29>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<29>();
template cudaError_t launch_m<30>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<30>();
template cudaError_t launch_m<31>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<31>();
template cudaError_t launch_m<32>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<32>();
}  // namespace rkb
