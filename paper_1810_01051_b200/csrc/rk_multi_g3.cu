// rk_multi_g3.cu -- explicit instantiations of the multi-pattern scan for m in
// {25, 26, 27, 28, 29, 30, 31, 32} (m = 32 stands for every m >= 32).
#include "rk_multi_impl.cuh"

namespace rkb {
template cudaError_t launch_multi_m<25>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<25>(uint32_t);
template cudaError_t launch_multi_m<26>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<26>(uint32_t);
template cudaError_t launch_multi_m<27>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<27>(uint32_t);
template cudaError_t launch_multi_m<28>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<28>(uint32_t);
template cudaError_t launch_multi_m<29>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<29>(uint32_t);
template cudaError_t launch_multi_m<30>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<30>(uint32_t);
template cudaError_t launch_multi_m<31>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<31>(uint32_t);
template cudaError_t launch_multi_m<32>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<32>(uint32_t);
}  // namespace rkb
