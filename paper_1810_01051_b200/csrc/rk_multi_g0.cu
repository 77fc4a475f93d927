// rk_multi_g0.cu -- explicit instantiations of the multi-pattern scan for m in
// {1, 2, 3, 4, 5, 6, 7, 8} (m = 32 stands for every m >= 32).
#include "rk_multi_impl.cuh"

namespace rkb {
template cudaError_t launch_multi_m<1>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<1>(uint32_t);
template cudaError_t launch_multi_m<2>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<2>(uint32_t);
template cudaError_t launch_multi_m<3>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<3>(uint32_t);
template cudaError_t launch_multi_m<4>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<4>(uint32_t);
template cudaError_t launch_multi_m<5>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<5>(uint32_t);
template cudaError_t launch_multi_m<6>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<6>(uint32_t);
template cudaError_t launch_multi_m<7>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<7>(uint32_t);
template cudaError_t launch_multi_m<8>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<8>(uint32_t);
}  // namespace rkb
