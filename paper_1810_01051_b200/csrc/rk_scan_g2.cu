// rk_scan_g2.cu -- explicit instantiations of the single-pattern scan for m in
// {17, 18, 19, 20, 21, 22, 23, 24} (m = 32 stands for every m >= 32).  The 32 variants are split
// over four translation units to keep each ptxas run small and the build parallel.
#include "rk_short_impl.cuh"

namespace rkb {
template cudaError_t launch_m<17>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<17>();
template cudaError_t launch_m<18>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<18>();
template cudaError_t launch_m<19>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<19>();
template cudaError_t launch_m<20>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<20>();
template cudaError_t launch_m<21>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<21>();
template cudaError_t launch_m<22>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<22>();
template cudaError_t launch_m<23>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<23>();
template cudaError_t launch_m<24>(const ScanArgs&, int, cudaStream_t);
template int occupancy_m<24>();
}  // namespace rkb
