// Development microbenchmark: the FNV kernel's round and final-pass bodies
// alone (16 compute warps per SM, data in shared memory like the kernel).
#include <cstdio>
#include "../../paper_2412_15411_b200/csrc/fnv.cuh"
using namespace mlck::fnv;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters) {
  extern __shared__ uint4 data[];
  const int t = threadIdx.x;
  for (int q = 0; q < kGranStride; ++q) data[granule(t, q)] = make_uint4(t * 77 + q, t ^ 0x5555 + q, q * 3, t);
  __syncthreads();
  uint32_t acc = 0, st = t & 0xff;
  for (int i = 0; i < iters; ++i) {
    uint32_t m[kSegs];
    const uint4* g = &data[granule(t, 0)];
    if (MODE == 0) {
      round_maps_low(g, st, 0, m);
      round_maps_low(g, st, 1, m);
    } else if (MODE == 1) {
      round_maps_high(g, st, 2, m);
      round_maps_high(g, st, 3, m);
    } else {
      uint32_t lo[kSegs], hi[kSegs];
      for (int s = 0; s < kSegs; ++s) { lo[s] = (st >> (8 * s)) & 0xff; hi[s] = 0; }
      uint4 nx = g[0];
#pragma unroll 2
      for (int q = 0; q < kGranules; ++q) {
        const uint4 v = nx;
        if (q + 1 < kGranules) nx = g[q + 1];
        for (const uint32_t y : {v.x, v.y, v.z, v.w})
#pragma unroll
          for (int s = 0; s < kSegs; ++s) fnv_byte(lo[s], hi[s], (y >> (8 * s)) & 0xffu);
      }
      for (int s = 0; s < kSegs; ++s) m[s] = lo[s] ^ hi[s];
    }
    for (int s = 0; s < kSegs; ++s) acc += m[s];
    st += acc;
  }
  out[blockIdx.x * 512 + t] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 200;
  for (int mode = 0; mode < 3; ++mode) {
    auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    const int smem = 512 * kGranStride * 16;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, 512, smem>>>(out, 2);
    cudaEventRecord(a);
    kern<<<sms, 512, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double cyc = ms * 1e-3 * clk * 1e3 / iters;
    printf("%s: %.0f cycles per %s (64 KB chunk, 16 warps/SM)\n",
           mode == 0 ? "rounds 0+1" : mode == 1 ? "rounds 2+3" : "final pass", cyc,
           mode == 2 ? "pass" : "two rounds");
  }
  return 0;
}
