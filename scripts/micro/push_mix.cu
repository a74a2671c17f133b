// Development microbenchmark: NVLink egress GPU0 -> GPU1 when the copy
// engines and SM stores share the push (CE: the first fraction f of the
// buffer, k SMs of 128-bit stores: the rest, concurrently), and with two
// copy-engine streams on halves.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) push(const uint4* __restrict__ src, uint64_t n, uint4* dst) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) dst[i] = src[i];
}

int main() {
  const uint64_t bytes = 8ull << 30;
  uint4 *src, *dst;
  cudaSetDevice(0);
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaSetDevice(1);
  cudaMalloc(&dst, bytes);
  cudaSetDevice(0);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t a, b0, b1;
  cudaEventCreate(&a);
  cudaEventCreate(&b0);
  cudaEventCreate(&b1);
  auto run = [&](double f, int sms, bool two_ce) {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s0);
      cudaStreamWaitEvent(s1, a, 0);
      const uint64_t ce = static_cast<uint64_t>(bytes * f) / 4096 * 4096;
      if (two_ce) {
        cudaMemcpyPeerAsync(dst, 1, src, 0, ce / 2, s0);
        cudaMemcpyPeerAsync(reinterpret_cast<uint8_t*>(dst) + ce / 2, 1, reinterpret_cast<uint8_t*>(src) + ce / 2, 0,
                            ce - ce / 2, s1);
      } else if (ce) {
        cudaMemcpyPeerAsync(dst, 1, src, 0, ce, s0);
      }
      if (ce < bytes && sms)
        push<<<sms, 1024, 0, s1>>>(reinterpret_cast<const uint4*>(reinterpret_cast<uint8_t*>(src) + ce), (bytes - ce) / 16,
                                   reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(dst) + ce));
      cudaEventRecord(b1, s1);
      cudaStreamWaitEvent(s0, b1, 0);
      cudaEventRecord(b0, s0);
      cudaEventSynchronize(b0);
      float ms;
      cudaEventElapsedTime(&ms, a, b0);
      if (ms < best) best = ms;
    }
    printf("ce_frac %.2f sms %3d two_ce %d: %.3f ms  %.1f GB/s\n", f, sms, two_ce, best, bytes / (best * 1e-3) / 1e9);
  };
  run(1.0, 0, false);
  run(1.0, 0, true);
  run(0.0, 148, false);
  for (double f : {0.95, 0.9, 0.85, 0.8, 0.7})
    for (int sms : {16, 32, 64}) run(f, sms, false);
  return 0;
}
