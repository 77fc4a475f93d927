// rk_multi_g0.cu -- explicit instantiations of the m < 7 multi-pattern kernels.
#include "rk_multi_impl.cuh"

namespace rkb {

template <int M>
struct rk_multi_tiny_tag {};

template <int M>
cudaError_t launch_multi_tiny(const MultiArgs& a, int grid, cudaStream_t s) {
  return multi_launch_kernel<rk_multi_tiny_tag<M>>(rk_multi_tiny_kernel<M>, a, grid,
                                                   multi_tiny_smem_bytes(), s);
}

template <int M>
int multi_tiny_occupancy() {
  return multi_occupancy(rk_multi_tiny_kernel<M>, multi_tiny_smem_bytes());
}

template cudaError_t launch_multi_tiny<1>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_tiny<2>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_tiny<3>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_tiny<4>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_tiny<5>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_tiny<6>(const MultiArgs&, int, cudaStream_t);
template int multi_tiny_occupancy<1>();
template int multi_tiny_occupancy<2>();
template int multi_tiny_occupancy<3>();
template int multi_tiny_occupancy<4>();
template int multi_tiny_occupancy<5>();
template int multi_tiny_occupancy<6>();

}  // namespace rkb
