// rk_multi_g1.cu -- explicit instantiations of the multi-pattern scan for m in
// {9, 10, 11, 12, 13, 14, 15, 16} (m = 32 stands for every m >= 32).
#include "rk_multi_impl.cuh"

namespace rkb {
template cudaError_t launch_multi_m<9>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<9>(uint32_t);
template cudaError_t launch_multi_m<10>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<10>(uint32_t);
template cudaError_t launch_multi_m<11>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<11>(uint32_t);
template cudaError_t launch_multi_m<12>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<12>(uint32_t);
template cudaError_t launch_multi_m<13>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<13>(uint32_t);
template cudaError_t launch_multi_m<14>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<14>(uint32_t);
template cudaError_t launch_multi_m<15>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<15>(uint32_t);
template cudaError_t launch_multi_m<16>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<16>(uint32_t);
}  // namespace rkb
