// pipe_bench.cu -- issue-rate microbenchmark of the integer instruction mixes the scan
// kernels are built from (sm_100a).  One CTA per SM, W warps, each running a long chain of
// independent instructions of one kind; prints warp-instructions per cycle per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_bench tools/pipe_bench.cu
//   /tmp/pipe_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kIndep = 8;  // independent chains per thread

template <int OP>
__global__ void bench(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[kIndep];
  for (int i = 0; i < kIndep; ++i) x[i] = threadIdx.x * 7u + i + a;
  bool p = false;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kIndep; ++i) {
      if constexpr (OP == 0) {  // IMAD, register multiplier
        x[i] = x[i] * a + b;
      } else if constexpr (OP == 1) {  // IMAD, immediate multiplier
        asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(x[i]) : "r"(b));
      } else if constexpr (OP == 2) {  // dp4a
        x[i] = __dp4a(x[i], a, b);
      } else if constexpr (OP == 3) {  // LOP3
        x[i] = (x[i] ^ a) & (b | x[i]);
      } else if constexpr (OP == 4) {  // PRMT
        x[i] = __byte_perm(x[i], a, 0x5140);
      } else if constexpr (OP == 5) {  // IMAD + ISETP.EQ.OR accumulate
        x[i] = x[i] * a + b;
        p |= (x[i] == b);
      } else if constexpr (OP == 6) {  // IADD3
        x[i] = x[i] + x[(i + 1) % kIndep] + a;
      } else if constexpr (OP == 7) {  // funnel shift
        x[i] = __funnelshift_r(x[i], a, 8);
      } else if constexpr (OP == 8) {  // FFMA reg
        float f = __uint_as_float(x[i]);
        f = fmaf(f, __uint_as_float(a), __uint_as_float(b));
        x[i] = __float_as_uint(f);
      } else if constexpr (OP == 9) {  // IMAD + masked compare (LOP3 pred + PLOP3)
        x[i] = x[i] * a + b;
        p |= ((x[i] ^ b) & 0xfff0u) == 0u;
      } else if constexpr (OP == 10) {  // HSETP2-like: half2 compare
        x[i] = x[i] * a + b;
        uint32_t q;
        asm("{.reg .pred q, r; setp.eq.f16x2 q|r, %1, %2; selp.u32 %0, 1, 0, q;}"
            : "=r"(q)
            : "r"(x[i]), "r"(b));
        acc |= q;
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = acc;
  for (int i = 0; i < kIndep; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + p;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps, uint32_t* out, long long* cyc, int sms) {
  bench<OP><<<sms, 32 * warps>>>(out, 0x01020408u, 5u, cyc);
  cudaDeviceSynchronize();
  bench<OP><<<sms, 32 * warps>>>(out, 0x01020408u, 5u, cyc);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double instr = (double)warps * kIters * kIndep;  // per SM (one CTA per SM)
  printf("%-22s warps=%2d  %.3f warp-instr/cycle/SM\n", name, warps, instr / (double)c);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  for (int w : {16, 32}) {
    run<0>("IMAD reg", w, out, cyc, sms);
    run<1>("IMAD imm", w, out, cyc, sms);
    run<9>("IMAD+LOP3mask cmp", w, out, cyc, sms);
    run<2>("IDP.4A", w, out, cyc, sms);
    run<3>("LOP3", w, out, cyc, sms);
    run<4>("PRMT", w, out, cyc, sms);
    run<5>("IMAD+ISETP.OR", w, out, cyc, sms);
    run<6>("IADD3", w, out, cyc, sms);
    run<7>("SHF funnel", w, out, cyc, sms);
    run<8>("FFMA reg", w, out, cyc, sms);
    run<10>("IMAD+HSETP2+sel", w, out, cyc, sms);
  }
  return 0;
}
