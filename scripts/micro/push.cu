// Development microbenchmark: peer push bandwidth GPU0 -> GPU1 with k SMs of
// 128-bit NVLink stores (one 1024-thread CTA per SM) vs a copy-engine
// cudaMemcpyPeerAsync, and with 2 destinations (r = 2 ring replicas).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) push(const uint4* __restrict__ src, uint64_t n, uint4* d0, uint4* d1) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) {
    const uint4 v = src[i];
    d0[i] = v;
    if (d1) d1[i] = v;
  }
}

int main() {
  int ndev;
  cudaGetDeviceCount(&ndev);
  const uint64_t bytes = 4ull << 30;
  uint4 *src, *d0, *d1 = nullptr;
  cudaSetDevice(0);
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaDeviceEnablePeerAccess(1, 0);
  if (ndev > 2) cudaDeviceEnablePeerAccess(2, 0);
  cudaSetDevice(1);
  cudaMalloc(&d0, bytes);
  if (ndev > 2) {
    cudaSetDevice(2);
    cudaMalloc(&d1, bytes);
  }
  cudaSetDevice(0);
  cudaFuncSetAttribute(push, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyPeerAsync(d0, 1, src, 0, bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("copy engine 1 dst: %.0f GB/s\n", bytes / ms / 1e6);
  for (int dsts = 1; dsts <= (d1 ? 2 : 1); ++dsts)
    for (int k : {4, 8, 16, 24, 32, 48, 64, 148}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        push<<<k, 1024, 120 * 1024>>>(src, bytes / 16, d0, dsts == 2 ? d1 : nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("SM push %d dst, %3d SMs: %.0f GB/s egress (%s)\n", dsts, k, dsts * bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
