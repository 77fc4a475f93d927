// rk_internal.h -- host-side declarations shared by the CUDA translation units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rk_device.cuh"

namespace rkb {

// single pattern (rk_scan.cu)
int scan_blocks_per_sm(uint32_t m);
cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t s);

// multi pattern (rk_multi.cu)
struct MultiHostPlan {
  const uint8_t* abase;
  uint64_t amis, n, ja_lo, ja_hi, tile0, num_tiles, ticket_base, cap;
  const uint8_t* pats;
  const uint64_t* phash;
  const uint32_t* filter;
  const uint2* table;
  const uint32_t* order;
  int64_t* out_off;
  uint32_t* out_idx;
  unsigned long long* ticket;
  unsigned long long* counters;
  uint32_t m, P, tsize;
};
constexpr int kMultiFilterWords = (1 << 16) / 32;
constexpr uint32_t kMultiEmpty = 0xffffffffu;
cudaError_t launch_multi_plan(const MultiHostPlan& p, int grid, cudaStream_t s);

// auxiliaries (rk_aux.cu)
cudaError_t launch_window_hashes(const uint8_t* text, uint64_t n, uint32_t m, uint64_t start,
                                 uint64_t stop, uint64_t* out, cudaStream_t s);
cudaError_t launch_generate(uint8_t* out, uint64_t count, uint64_t seed, uint64_t skip,
                            const uint8_t* alphabet, uint32_t k, cudaStream_t s);

}  // namespace rkb
