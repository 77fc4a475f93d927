// rk_pairs.cu -- ordering of multi-pattern (pattern index, offset) pairs on the device,
// for result sets too large to round-trip through the host: the reference returns each
// pattern's offsets ascending (matcher.py:154-157), i.e. pairs ordered by (index, offset).
// Key = index << bits(n - 1) | offset, radix-sorted over its significant bits only (CUB,
// CUDA toolkit headers), then split back.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "rk_internal.h"

namespace rkb {

template <class K>
static __global__ void pack_pairs_kernel(const int64_t* off, const uint32_t* idx, uint64_t k,
                                         uint32_t shift, K* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((K)idx[i] << shift) | (K)off[i];
}

template <class K>
static __global__ void unpack_pairs_kernel(const K* keys, uint64_t k, uint32_t shift,
                                           int64_t* off, uint32_t* idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x) {
    off[i] = (int64_t)(keys[i] & (((K)1 << shift) - 1));
    idx[i] = (uint32_t)(keys[i] >> shift);
  }
}

static uint32_t bit_width(uint64_t x) {
  uint32_t b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

size_t sort_pairs_scratch(uint64_t k) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int64_t)k, 0, 64);
  return 2 * k * sizeof(unsigned long long) + ((tmp + 255) & ~(size_t)255);
}

template <class K>
static cudaError_t sort_keys(int64_t* d_off, uint32_t* d_idx, uint64_t k, uint32_t shift,
                             uint32_t bits, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  K* a = static_cast<K*>(scratch);
  K* b = a + k;
  void* tmp = reinterpret_cast<uint8_t*>(scratch) + ((2 * k * sizeof(K) + 255) & ~(size_t)255);
  size_t tmp_bytes = scratch_bytes - ((2 * k * sizeof(K) + 255) & ~(size_t)255);
  const unsigned grid = (unsigned)std::min<uint64_t>((k + 255) / 256, 4096);
  pack_pairs_kernel<K><<<grid, 256, 0, s>>>(d_off, d_idx, k, shift, a);
  cudaError_t e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int64_t)k, 0, (int)bits, s);
  if (e != cudaSuccess) return e;
  unpack_pairs_kernel<K><<<grid, 256, 0, s>>>(b, k, shift, d_off, d_idx);
  return cudaGetLastError();
}

// Orders k pairs whose offsets are < n and indices < P by (index, offset): the key holds
// only the bits those need (index << bits(n - 1) | offset), so the radix sort makes
// ceil(bits / 8) passes, over 4-byte keys when they fit (all 'a' with three patterns over
// 64 MiB: 28 bits, 4 passes of 4-byte keys instead of 7 of 8-byte ones).
cudaError_t sort_pairs(int64_t* d_off, uint32_t* d_idx, uint64_t k, uint64_t n, uint32_t P,
                       void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const uint32_t ob = std::max<uint32_t>(1, bit_width(n > 0 ? n - 1 : 0));
  const uint32_t bits = ob + bit_width(P > 0 ? P - 1 : 0);
  if (bits <= 32 && ob < 32)
    return sort_keys<uint32_t>(d_off, d_idx, k, ob, bits, scratch, scratch_bytes, s);
  return sort_keys<unsigned long long>(d_off, d_idx, k, ob, bits, scratch, scratch_bytes, s);
}

// Small sets (k <= kSmallSort pairs) are ordered by one block in shared memory (bitonic
// sort of the packed keys), so a sparse search_multi needs no host round trip for the
// pairs: the host copies cost ~15 us each way against ~5 us for this kernel (C3).  The
// count is read on the device (d_count, clamped to cap) or given (k_host); count_out, if
// set, receives *d_count (pinned host memory mapped through UVA: no copy either).
constexpr int kSmallSortThreads = 1024;
static __global__ void __launch_bounds__(kSmallSortThreads)
    small_sort_kernel(int64_t* off, uint32_t* idx, const unsigned long long* d_count,
                      uint64_t k_host, uint64_t cap, uint32_t ob,
                      unsigned long long* count_out) {
  __shared__ unsigned long long key[kSmallSort];
  const int tid = threadIdx.x;
  uint64_t k = k_host;
  if (d_count) {
    const unsigned long long c = *d_count;
    if (count_out && tid == 0) *count_out = c;
    k = c < cap ? c : cap;
  }
  if (k <= 1 || k > kSmallSort) return;
  uint32_t N = 2;
  while (N < k) N <<= 1;
  for (uint32_t i = tid; i < N; i += kSmallSortThreads)
    key[i] = i < k ? ((unsigned long long)idx[i] << ob) | (unsigned long long)off[i] : ~0ull;
  __syncthreads();
  for (uint32_t size = 2; size <= N; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < N; i += kSmallSortThreads) {
        const uint32_t j = i ^ stride;
        if (j > i) {
          const unsigned long long a = key[i], b = key[j];
          if ((a > b) == ((i & size) == 0)) {
            key[i] = b;
            key[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  const unsigned long long mask = (1ull << ob) - 1;
  for (uint32_t i = tid; i < k; i += kSmallSortThreads) {
    off[i] = (int64_t)(key[i] & mask);
    idx[i] = (uint32_t)(key[i] >> ob);
  }
}

cudaError_t small_sort_pairs(int64_t* d_off, uint32_t* d_idx, const unsigned long long* d_count,
                             uint64_t k_host, uint64_t cap, uint64_t n,
                             unsigned long long* count_out, cudaStream_t s) {
  const uint32_t ob = std::max<uint32_t>(1, bit_width(n > 0 ? n - 1 : 0));
  small_sort_kernel<<<1, kSmallSortThreads, 0, s>>>(d_off, d_idx, d_count, k_host, cap, ob,
                                                     count_out);
  return cudaGetLastError();
}

}  // namespace rkb
