// rk_aux.cu -- auxiliary device kernels:
//   * window_hashes: the batched 64-bit window hash of
//     /root/reference/pkg/src/rkmatch/_scan.py:71-91 (parity / debugging surface);
//   * generate: the counter-based splitmix64 corpus of
//     /root/reference/pkg/src/rkmatch/datagen.py:28-77, bit-identical, on device
//     (byte i = alphabet[z_{skip+i+1} mod k], z_s = mix(seed + s*GOLDEN)).
#include "rk_internal.h"

namespace rkb {

constexpr int kHashPerThread = 16;

__global__ void window_hashes_kernel(const uint8_t* __restrict__ text, uint32_t m, uint64_t start,
                                     uint64_t stop, uint64_t* __restrict__ out) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t x0 = start + t * kHashPerThread;
  if (x0 >= stop) return;
  const uint64_t x1 = x0 + kHashPerThread < stop ? x0 + kHashPerThread : stop;
  const uint32_t span = m < 64 ? m : 64;
  uint64_t h = 0;
  for (uint64_t i = x0 + m - span; i < x0 + m; ++i) h = (h << 1) + text[i];
  out[x0 - start] = h;
  for (uint64_t x = x0 + 1; x < x1; ++x) {
    const uint64_t outb = text[x - 1];
    const uint64_t inb = text[x + m - 1];
    const uint64_t top = m <= 64 ? (outb << (m - 1)) : 0;  // roll (rkhash.py:48-60)
    h = ((h - top) << 1) + inb;
    out[x - start] = h;
  }
}

cudaError_t launch_window_hashes(const uint8_t* text, uint64_t n, uint32_t m, uint64_t start,
                                 uint64_t stop, uint64_t* out, cudaStream_t s) {
  (void)n;
  if (stop <= start) return cudaSuccess;
  const uint64_t threads = (stop - start + kHashPerThread - 1) / kHashPerThread;
  const int block = 256;
  const uint64_t grid = (threads + block - 1) / block;
  window_hashes_kernel<<<(unsigned)grid, block, 0, s>>>(text, m, start, stop, out);
  return cudaGetLastError();
}

struct Alphabet {
  uint8_t b[256];
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <bool POW2>
__global__ void generate_kernel(uint8_t* __restrict__ out, uint64_t count, uint64_t seed,
                                uint64_t skip, Alphabet alpha, uint32_t k) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t i0 = t * 16;
  if (i0 >= count) return;
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint64_t i = i0 + j;
    const uint64_t z = mix64(seed + 0x9E3779B97F4A7C15ull * (skip + i + 1));
    const uint32_t sym = POW2 ? (uint32_t)(z & (k - 1)) : (uint32_t)(z % (uint64_t)k);
    w[j >> 2] |= (uint32_t)alpha.b[sym] << (8 * (j & 3));
  }
  if (i0 + 16 <= count && ((uintptr_t)(out + i0) & 15) == 0) {
    *reinterpret_cast<uint4*>(out + i0) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    for (int j = 0; j < 16 && i0 + j < count; ++j) out[i0 + j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
  }
}

cudaError_t launch_generate(uint8_t* out, uint64_t count, uint64_t seed, uint64_t skip,
                            const uint8_t* alphabet, uint32_t k, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  Alphabet a{};
  for (uint32_t i = 0; i < k; ++i) a.b[i] = alphabet[i];
  const uint64_t threads = (count + 15) / 16;
  const int block = 256;
  const uint64_t grid = (threads + block - 1) / block;
  if ((k & (k - 1)) == 0)
    generate_kernel<true><<<(unsigned)grid, block, 0, s>>>(out, count, seed, skip, a, k);
  else
    generate_kernel<false><<<(unsigned)grid, block, 0, s>>>(out, count, seed, skip, a, k);
  return cudaGetLastError();
}

}  // namespace rkb
