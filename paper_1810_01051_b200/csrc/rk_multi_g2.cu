// rk_multi_g2.cu -- explicit instantiations of the multi-pattern scan for m in
// {17, 18, 19, 20, 21, 22, 23, 24} (m = 32 stands for every m >= 32).
#include "rk_multi_impl.cuh"

namespace rkb {
template cudaError_t launch_multi_m<17>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<17>(uint32_t);
template cudaError_t launch_multi_m<18>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<18>(uint32_t);
template cudaError_t launch_multi_m<19>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<19>(uint32_t);
template cudaError_t launch_multi_m<20>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<20>(uint32_t);
template cudaError_t launch_multi_m<21>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<21>(uint32_t);
template cudaError_t launch_multi_m<22>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<22>(uint32_t);
template cudaError_t launch_multi_m<23>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<23>(uint32_t);
template cudaError_t launch_multi_m<24>(const MultiArgs&, int, cudaStream_t);
template int multi_occupancy_m<24>(uint32_t);
}  // namespace rkb
