// rk_pairs.cu -- ordering of multi-pattern (pattern index, offset) pairs on the device,
// for result sets too large to round-trip through the host: the reference returns each
// pattern's offsets ascending (matcher.py:154-157), i.e. pairs ordered by (index, offset).
// Key = index << 40 | offset (offsets < 2^40: a B200 holds < 180 GB), radix-sorted over
// its 52 significant bits (CUB, CUDA toolkit headers), then split back.
#include <cub/device/device_radix_sort.cuh>

#include "rk_internal.h"

namespace rkb {

static __global__ void pack_pairs_kernel(const int64_t* off, const uint32_t* idx, uint64_t k,
                                         unsigned long long* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((unsigned long long)idx[i] << 40) | (unsigned long long)off[i];
}

static __global__ void unpack_pairs_kernel(const unsigned long long* keys, uint64_t k,
                                           int64_t* off, uint32_t* idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    off[i] = (int64_t)(keys[i] & ((1ull << 40) - 1));
    idx[i] = (uint32_t)(keys[i] >> 40);
  }
}

size_t sort_pairs_scratch(uint64_t k) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int64_t)k, 0, 52);
  return 2 * k * sizeof(unsigned long long) + ((tmp + 255) & ~(size_t)255);
}

cudaError_t sort_pairs(int64_t* d_off, uint32_t* d_idx, uint64_t k, void* scratch,
                       size_t scratch_bytes, cudaStream_t s) {
  unsigned long long* a = static_cast<unsigned long long*>(scratch);
  unsigned long long* b = a + k;
  void* tmp = b + k;
  size_t tmp_bytes = scratch_bytes - 2 * k * sizeof(unsigned long long);
  const unsigned grid = (unsigned)std::min<uint64_t>((k + 255) / 256, 4096);
  pack_pairs_kernel<<<grid, 256, 0, s>>>(d_off, d_idx, k, a);
  cudaError_t e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int64_t)k, 0, 52, s);
  if (e != cudaSuccess) return e;
  unpack_pairs_kernel<<<grid, 256, 0, s>>>(b, k, d_off, d_idx);
  return cudaGetLastError();
}

}  // namespace rkb
