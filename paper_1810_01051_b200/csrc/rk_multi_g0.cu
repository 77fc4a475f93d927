// rk_multi_g0.cu -- explicit instantiations of the m < 7 multi-pattern kernels.
#include "rk_multi_impl.cuh"

namespace rkb {

template <int M>
struct rk_multi_short_tag {};

template <int M>
cudaError_t launch_multi_short(const MultiArgs& a, int grid, cudaStream_t s) {
  return multi_launch_kernel<rk_multi_short_tag<M>>(rk_multi_short_kernel<M>, a, grid, s);
}

template <int M>
int multi_short_occupancy() {
  return multi_occupancy(rk_multi_short_kernel<M>);
}

template cudaError_t launch_multi_short<1>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<2>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<3>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<4>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<5>(const MultiArgs&, int, cudaStream_t);
template cudaError_t launch_multi_short<6>(const MultiArgs&, int, cudaStream_t);
template int multi_short_occupancy<1>();
template int multi_short_occupancy<2>();
template int multi_short_occupancy<3>();
template int multi_short_occupancy<4>();
template int multi_short_occupancy<5>();
template int multi_short_occupancy<6>();

}  // namespace rkb
