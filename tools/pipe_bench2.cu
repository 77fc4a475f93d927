// pipe_bench2.cu -- which pipe do the fp16x2 / vector-int instructions run on (sm_100a)?
// Each op is timed alone and interleaved 1:1 with IMAD (FMA pipe) and with LOP3 (ALU pipe):
// a pair rate near the sum of the single rates means separate pipes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench2.bin tools/pipe_bench2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kIndep = 8;

__device__ __forceinline__ uint32_t op_x(int OP, uint32_t x, uint32_t a) {
  uint32_t d;
  switch (OP) {
    case 0:  // HSET2.BF eq  (1.0 per equal half)
      asm volatile("set.eq.f16x2.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(a));
      return d;
    case 1:  // HADD2
      asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(a));
      return d;
    case 2:  // HMNMX2 plain min
      asm volatile("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(a));
      return d;
    case 3:  // min.xorsign.abs
      asm volatile("min.xorsign.abs.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(a));
      return d;
    case 4:  // vector u16 min (VIMNMX?)
      return __vminu2(x, a);
    case 5:  // 3-way u16 min (DPX)
      return __vimin3_u16x2(x, a, x ^ 0x5u);
    case 6:  // HFMA2
      asm volatile("fma.rn.f16x2 %0, %1, %2, %1;" : "=r"(d) : "r"(x), "r"(a));
      return d;
    case 7:  // FSETP (non-ftz) -> selp
      asm volatile("{.reg .pred p; setp.eq.f32 p, %1, %2; selp.u32 %0, %1, %2, p;}"
                   : "=r"(d)
                   : "r"(x), "r"(a));
      return d;
    case 8:  // IMNMX
      return min(x, a);
    case 9:  // FMNMX
      return __float_as_uint(fminf(__uint_as_float(x), __uint_as_float(a)));
  }
  return x;
}

// MIX: 0 alone, 1 with IMAD, 2 with LOP3
template <int OP, int MIX>
__global__ void bench(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[kIndep], y[kIndep];
  for (int i = 0; i < kIndep; ++i) {
    x[i] = threadIdx.x * 7u + i + a;
    y[i] = threadIdx.x * 3u + i + b;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kIndep; ++i) {
      x[i] = op_x(OP, x[i], x[(i + 3) % kIndep]);
      if constexpr (MIX == 1) y[i] = y[i] * a + b;
      if constexpr (MIX == 2) y[i] = (y[i] ^ a) | (b & y[i]);
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < kIndep; ++i) s += x[i] + y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP, int MIX>
double run1(uint32_t* out, long long* cyc, int sms, int warps) {
  for (int r = 0; r < 2; ++r) bench<OP, MIX><<<sms, 32 * warps>>>(out, 0x3c003c01u, 5u, cyc);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  return (double)warps * kIters * kIndep / (double)c;  // ops (of the tested kind) per cycle per SM
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc, int sms) {
  const int w = 32;
  printf("%-22s alone %.2f   +IMAD %.2f   +LOP3 %.2f  (op/cycle/SM; pair rates count the op only)\n",
         name, run1<OP, 0>(out, cyc, sms, w), run1<OP, 1>(out, cyc, sms, w),
         run1<OP, 2>(out, cyc, sms, w));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<0>("HSET2.BF", out, cyc, sms);
  run<1>("HADD2", out, cyc, sms);
  run<2>("HMNMX2", out, cyc, sms);
  run<3>("HMNMX2.xorsign.abs", out, cyc, sms);
  run<4>("vminu2", out, cyc, sms);
  run<5>("vimin3_u16x2", out, cyc, sms);
  run<6>("HFMA2", out, cyc, sms);
  run<7>("FSETP+SEL", out, cyc, sms);
  run<8>("IMNMX", out, cyc, sms);
  run<9>("FMNMX", out, cyc, sms);
  return 0;
}
