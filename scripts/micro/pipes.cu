// Development microbenchmark: issue rates of the integer ops the FNV kernel
// is built from (LOP3+IMAD chains, IMAD.WIDE chains), per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
  uint32_t x0 = threadIdx.x ^ seed, x1 = x0 * 7, x2 = x0 * 13, x3 = x0 * 17;
  uint32_t y = seed * 0x9e3779b9u + threadIdx.x;
  uint32_t lo = x0, hi = 0, lo2 = x1, hi2 = 0, lo3 = x2, hi3 = 0, lo4 = x3, hi4 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      y = y * 0x01000193u + j;  // vary y (one IMAD, FMA pipe)
      if (MODE == 0) {  // 2 chains: LOP3 + IMAD x3
        x0 = ((x0 ^ y) & 0x0f0f0f0fu) * 3u;
        x1 = ((x1 ^ y) & 0x0f0f0f0fu) * 3u;
      } else if (MODE == 1) {  // 4 chains: LOP3 + IMAD xb3
        x0 = ((x0 ^ y) & 0x00ff00ffu) * 0xb3u;
        x1 = ((x1 ^ y) & 0x00ff00ffu) * 0xb3u;
        x2 = ((x2 ^ y) & 0x00ff00ffu) * 0xb3u;
        x3 = ((x3 ^ y) & 0x00ff00ffu) * 0xb3u;
      } else {  // 4 fnv chains
#define FB(L, H)                                                   \
  {                                                                \
    L ^= (y >> 8) & 0xffu;                                         \
    const uint64_t t = static_cast<uint64_t>(L) * 0x1b3u;          \
    uint32_t f;                                                    \
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(f) : "r"(L), "r"(static_cast<uint32_t>(t >> 32))); \
    asm("mad.lo.u32 %0, %1, 0x1b3, %2;" : "=r"(H) : "r"(H), "r"(f)); \
    L = static_cast<uint32_t>(t);                                  \
  }
        FB(lo, hi) FB(lo2, hi2) FB(lo3, hi3) FB(lo4, hi4)
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ lo ^ hi ^ lo2 ^ hi2 ^ lo3 ^ hi3 ^ lo4 ^ hi4 ^ y;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  cudaMalloc(&out, 148 * 1024 * 4 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      kern<<<sms, 32 * warps>>>(out, 10, 1);
      cudaEventRecord(a);
      kern<<<sms, 32 * warps>>>(out, iters, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // steps per SM per ns
      const double steps = double(iters) * 32 * 32 * warps;  // per SM: thread-steps (inner j)
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      const double cycles = ms * 1e-3 * clk * 1e3;
      printf("mode %d warps/SM %2d: %.3f ms, %.1f thread-steps/cycle/SM\n", mode, warps, ms, steps / cycles);
    }
  return 0;
}
