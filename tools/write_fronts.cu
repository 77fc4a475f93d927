// Write-bandwidth probe: 2 GiB of int64 written (a) as one global front (grid-stride,
// 1 KiB per warp instruction) and (b) as F independent fronts (each warp owns a contiguous
// region and walks it in 8 KiB steps, the ordered emission's dense pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/write_fronts.cu -o tools/write_fronts.bin
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void st4(int64_t* p, int64_t a) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(a + 1),
               "l"(a + 2), "l"(a + 3) : "memory");
}

template <int MODE>
__global__ void probe(int64_t* o, uint64_t n) {
  // MODE 0: STG.256 of i; 1: STG.256 of 0; 2: STG.128 of i; 3: STG.128 of 0; 4: st.cs.v4 of i
  const int W = (MODE == 2 || MODE == 3) ? 2 : 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * W;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += stride) {
    const int64_t v = (MODE == 1 || MODE == 3) ? 0 : (int64_t)i;
    if (MODE == 0 || MODE == 1)
      st4(o + i, v);
    else if (MODE == 4)
      asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(o + i), "l"(v), "l"(v + 1),
                   "l"(v + 2), "l"(v + 3) : "memory");
    else
      asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(o + i), "l"(v), "l"(v + 1) : "memory");
  }
}

// torch's fill pattern: a 128-thread block writes 8 KiB, each thread 4 x 16 B at 2 KiB
// strides, one block per 8 KiB (no grid-stride loop)
__global__ void torch_like(int64_t* o, int64_t v) {
  int64_t* p = o + (uint64_t)blockIdx.x * 1024 + threadIdx.x * 2;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p + k * 256), "l"(v), "l"(v) : "memory");
}
// the same, block -> 8 KiB region through a bijective scramble of the block index
__global__ void torch_like_perm(int64_t* o, uint32_t nb_log2, int64_t v) {
  const uint32_t mask = (1u << nb_log2) - 1;
  const uint32_t b = (blockIdx.x * 2654435761u) & mask;  // odd multiplier: a bijection mod 2^k
  int64_t* p = o + (uint64_t)b * 1024 + threadIdx.x * 2;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p + k * 256), "l"(v), "l"(v) : "memory");
}
// short-lived blocks writing K KiB each (blockDim threads, 16 B per store)
template <int KB>
__global__ void big_blocks(int64_t* o, int64_t v) {
  int64_t* p = o + (uint64_t)blockIdx.x * (KB * 128) + threadIdx.x * 2;
  const int per = KB * 128 / (blockDim.x * 2);
  for (int k = 0; k < per; ++k)
    asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p + k * blockDim.x * 2), "l"(v), "l"(v) : "memory");
}
// persistent blocks taking units of U KiB from an atomic ticket counter (dynamic balance)
__device__ unsigned long long g_ticket;
template <int UKB>
__global__ void tickets(int64_t* o, uint64_t n, int64_t v) {
  __shared__ unsigned long long u;
  const uint64_t nu = n / (UKB * 128);
  for (;;) {
    if (threadIdx.x == 0) u = atomicAdd(&g_ticket, 1ull);
    __syncthreads();
    const uint64_t my = u;
    __syncthreads();
    if (my >= nu) break;
    int64_t* p = o + my * (UKB * 128) + threadIdx.x * 4;
    for (int k = 0; k < UKB * 128 / ((int)blockDim.x * 4); ++k) st4(p + k * blockDim.x * 4, v);
  }
}
// warp-level tickets: a warp claims a U KiB unit and writes it 8 KiB (1024 values) at a
// time, STG.256 (the emit's balanced phase)
__device__ unsigned long long g_wticket;
template <int UKB>
__global__ void warp_tickets(int64_t* o, uint64_t n, int64_t v) {
  const int lane = threadIdx.x & 31;
  const uint64_t nu = n / (UKB * 128);
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(&g_wticket, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nu) break;
    int64_t* p = o + u * (UKB * 128);
    for (int c = 0; c < UKB * 128; c += 1024)
#pragma unroll 2
      for (int i = 4 * lane; i < 1024; i += 128) st4(p + c + i, v + c + i);
  }
}
// the same with every 8 KiB run starting 3 values past a 32-byte boundary: up to 3
// scalar stores, the 32-byte body, then the tail (the emit's store_run on C5's offsets)
template <int UKB>
__global__ void warp_tickets_mis(int64_t* o, uint64_t n, int64_t v) {
  const int lane = threadIdx.x & 31;
  const uint64_t nu = n / (UKB * 128) - 1;
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(&g_wticket, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nu) break;
    int64_t* p = o + 3 + u * (UKB * 128);
    for (int c = 0; c < UKB * 128; c += 1024) {
      int64_t* q = p + c;
      const int head = (int)(((32u - ((uint32_t)(uintptr_t)q & 31u)) & 31u) >> 3);
      if (lane < head) q[lane] = v + lane;
      int64_t* ob = q + head;
      const int body = (1024 - head) & ~3;
#pragma unroll 2
      for (int i = 4 * lane; i < body; i += 128) st4(ob + i, v + i);
      if (lane < 1024 - head - body) ob[body + lane] = v + body + lane;
    }
  }
}
// the same pattern, grid-stride over 8 KiB blocks with a persistent grid
__global__ void torch_like_persist(int64_t* o, uint64_t nb, int64_t v) {
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int64_t* p = o + b * 1024 + threadIdx.x * 2;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p + k * 256), "l"(v), "l"(v) : "memory");
  }
}

__global__ void one_front(int64_t* o, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride)
    st4(o + i, (int64_t)i);
}

// warp w of the grid owns [w * per, (w + 1) * per), writes it 1024 elements at a time
__global__ void fronts(int64_t* o, uint64_t n, uint64_t per) {
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t b = w * per, e = b + per < n ? b + per : n;
  for (uint64_t c = b; c < e; c += 1024)
#pragma unroll
    for (int i = 4 * lane; i < 1024; i += 128) st4(o + c + i, (int64_t)(c + i));
}

// block-cooperative: block's 8 warps write 8 adjacent KiB-chunks per step (one 64 KiB
// front per block, blocks own contiguous regions)
__global__ void block_fronts(int64_t* o, uint64_t n, uint64_t per) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint64_t b = blockIdx.x * per, e = b + per < n ? b + per : n;
  for (uint64_t c = b + warp * 1024; c < e; c += 1024 * nw)
#pragma unroll
    for (int i = 4 * lane; i < 1024; i += 128) st4(o + c + i, (int64_t)(c + i));
}

int main() {
  const uint64_t n = 1ull << 28;  // 2 GiB of int64
  int64_t* o;
  cudaMalloc(&o, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run10 = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %.3f ms  %.2f TB/s (10 back to back)\n", name, ms / 10, n * 8 / (ms / 10) / 1e9);
  };
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-28s %.3f ms  %.2f TB/s\n", name, best, n * 8 / best / 1e9);
  };
  run("one front 148x1024", [&] { one_front<<<148 * 2, 1024>>>(o, n); });
  run10("torch-like 8KiB blocks", [&] { torch_like<<<n / 1024, 128>>>(o, 7); });
  auto zt = [&] { unsigned long long z = 0; cudaMemcpyToSymbolAsync(g_ticket, &z, 8); };
  run10("tickets 8KiB 256thr 148x8", [&] { zt(); tickets<8><<<148 * 8, 256>>>(o, n, 7); });
  run10("tickets 64KiB 256thr 148x8", [&] { zt(); tickets<64><<<148 * 8, 256>>>(o, n, 7); });
  run10("tickets 64KiB 256thr 148x1", [&] { zt(); tickets<64><<<148, 256>>>(o, n, 7); });
  run10("tickets 512KiB 256thr 148x1", [&] { zt(); tickets<512><<<148, 256>>>(o, n, 7); });
  run10("tickets 2MiB 256thr 148x1", [&] { zt(); tickets<2048><<<148, 256>>>(o, n, 7); });
  run10("tickets 64KiB 1024thr 148x2", [&] { zt(); tickets<64><<<148 * 2, 1024>>>(o, n, 7); });
  auto zw = [&] { unsigned long long z = 0; cudaMemcpyToSymbolAsync(g_wticket, &z, 8); };
  run10("warp tickets 64KiB 148x256", [&] { zw(); warp_tickets<64><<<148, 256>>>(o, n, 7); });
  run10("warp tickets mis 64KiB 148x256", [&] { zw(); warp_tickets_mis<64><<<148, 256>>>(o, n, 7); });
  run10("warp tickets 64KiB 148x512", [&] { zw(); warp_tickets<64><<<148, 512>>>(o, n, 7); });
  run10("warp tickets 64KiB 148x1024", [&] { zw(); warp_tickets<64><<<148, 1024>>>(o, n, 7); });
  run10("warp tickets 64KiB 296x1024", [&] { zw(); warp_tickets<64><<<296, 1024>>>(o, n, 7); });
  run10("warp tickets 8KiB 148x256", [&] { zw(); warp_tickets<8><<<148, 256>>>(o, n, 7); });
  run10("warp tickets 512KiB 148x256", [&] { zw(); warp_tickets<512><<<148, 256>>>(o, n, 7); });
  run10("torch-like permuted", [&] { torch_like_perm<<<n / 1024, 128>>>(o, 18, 7); });
  run10("blocks 64KiB x256thr", [&] { big_blocks<64><<<n / (64 * 128), 256>>>(o, 7); });
  run10("blocks 64KiB x1024thr", [&] { big_blocks<64><<<n / (64 * 128), 1024>>>(o, 7); });
  run10("blocks 1MiB x256thr", [&] { big_blocks<1024><<<n / (1024 * 128), 256>>>(o, 7); });
  run10("blocks 1MiB x1024thr", [&] { big_blocks<1024><<<n / (1024 * 128), 1024>>>(o, 7); });
  run10("blocks 14MiB x256thr", [&] { big_blocks<14336><<<n / (14336 * 128), 256>>>(o, 7); });
  run10("torch-like persist 148x16", [&] { torch_like_persist<<<148 * 16, 128>>>(o, n / 1024, 7); });
  run10("torch-like persist 148x4", [&] { torch_like_persist<<<148 * 4, 128>>>(o, n / 1024, 7); });
  run10("torch-like persist 148x2", [&] { torch_like_persist<<<148 * 2, 128>>>(o, n / 1024, 7); });
  run10("STG.256 of i", [&] { probe<0><<<148 * 4, 512>>>(o, n); });
  run10("STG.256 of 0", [&] { probe<1><<<148 * 4, 512>>>(o, n); });
  run10("cudaMemset 0x5a", [&] { cudaMemsetAsync(o, 0x5a, n * 8); });
  run("STG.256 of i", [&] { probe<0><<<148 * 4, 512>>>(o, n); });
  run("STG.256 of 0", [&] { probe<1><<<148 * 4, 512>>>(o, n); });
  run("STG.128 of i", [&] { probe<2><<<148 * 4, 512>>>(o, n); });
  run("STG.128 of 0", [&] { probe<3><<<148 * 4, 512>>>(o, n); });
  run("st.cs.v4 of i", [&] { probe<4><<<148 * 4, 512>>>(o, n); });
  run("cudaMemset 0", [&] { cudaMemsetAsync(o, 0, n * 8); });
  run("cudaMemset 0x5a", [&] { cudaMemsetAsync(o, 0x5a, n * 8); });
  run("one front 148x256", [&] { one_front<<<148, 256>>>(o, n); });
  for (int warps : {1184, 2368, 148 * 4}) {
    const uint64_t per = ((n + warps - 1) / warps + 1023) / 1024 * 1024;
    char nm[64];
    snprintf(nm, sizeof nm, "warp fronts %d", warps);
    run(nm, [&] { fronts<<<(warps + 7) / 8, 256>>>(o, n, per); });
  }
  for (int blocks : {148, 296}) {
    const uint64_t per = ((n + blocks - 1) / blocks + 8191) / 8192 * 8192;
    char nm[64];
    snprintf(nm, sizeof nm, "block fronts %d x 8 warps", blocks);
    run(nm, [&] { block_fronts<<<blocks, 256>>>(o, n, per); });
  }
  return 0;
}
