// Development microbenchmark: device-local copy of a record-sized buffer on
// the copy engines, split over 1/2/4/8 streams, vs an SM copy kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/mlck_b200.h"

__global__ void __launch_bounds__(1024) copyk(const uint4* __restrict__ s, uint4* __restrict__ d, uint64_t n) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) d[i] = s[i];
}

int main() {
  const uint64_t bytes = 1713239274ull / 65536 * 65536;
  char *src, *dst;
  cudaMalloc(&src, bytes);
  cudaMalloc(&dst, bytes);
  cudaMemset(src, 1, bytes);
  cudaStream_t st[8];
  cudaEvent_t e[8], a, b;
  for (int i = 0; i < 8; ++i) {
    cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&e[i], cudaEventDisableTiming);
  }
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k : {1, 2, 4, 8}) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a, st[0]);
      for (int i = 1; i < k; ++i) cudaStreamWaitEvent(st[i], a);
      const uint64_t piece = bytes / k / 65536 * 65536;
      for (int i = 0; i < k; ++i) {
        const uint64_t lo = i * piece, len = i == k - 1 ? bytes - lo : piece;
        cudaMemcpyAsync(dst + lo, src + lo, len, cudaMemcpyDeviceToDevice, st[i]);
        cudaEventRecord(e[i], st[i]);
      }
      for (int i = 1; i < k; ++i) cudaStreamWaitEvent(st[0], e[i]);
      cudaEventRecord(b, st[0]);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("CE %d streams: %.3f ms = %.0f GB/s (copy bytes)\n", k, ms, bytes / ms / 1e6);
  }
  {  // beside the real hash kernel (libmlck_b200) on its own stream
    mlck_ctx* ctx;
    mlck_ctx_create(0, &ctx);
    uint64_t h;
    char* other;
    cudaMalloc(&other, bytes);
    cudaMemset(other, 2, bytes);
    mlck_fnv1a64(ctx, other, bytes, 0xcbf29ce484222325ull, &h);
    for (int src_is_hashed = 0; src_is_hashed < 2; ++src_is_hashed)
      for (int k : {1, 4}) {
        float ms = 0, fms = 0;
        cudaEvent_t fa, fb;
        cudaEventCreate(&fa);
        cudaEventCreate(&fb);
        for (int rep = 0; rep < 3; ++rep) {
          cudaDeviceSynchronize();
          cudaEventRecord(a, st[0]);
          for (int i = 1; i < k; ++i) cudaStreamWaitEvent(st[i], a);
          const uint64_t piece = bytes / k / 65536 * 65536;
          for (int i = 0; i < k; ++i) {
            const uint64_t lo = i * piece, len = i == k - 1 ? bytes - lo : piece;
            cudaMemcpyAsync(dst + lo, src + lo, len, cudaMemcpyDeviceToDevice, st[i]);
            cudaEventRecord(e[i], st[i]);
          }
          for (int i = 1; i < k; ++i) cudaStreamWaitEvent(st[0], e[i]);
          cudaEventRecord(b, st[0]);
          cudaEventRecord(fa, 0);
          mlck_fnv1a64(ctx, src_is_hashed ? src : other, bytes, 0xcbf29ce484222325ull, &h);
          cudaEventRecord(fb, 0);
          cudaDeviceSynchronize();
          cudaEventElapsedTime(&ms, a, b);
          cudaEventElapsedTime(&fms, fa, fb);
        }
        printf("CE %d streams beside the hash of %s: copy %.3f ms, hash %.3f ms\n", k,
               src_is_hashed ? "the copied buffer" : "another buffer", ms, fms);
      }
  }
  for (int g : {148, 296, 592}) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a, st[0]);
      copyk<<<g, 1024, 0, st[0]>>>((const uint4*)src, (uint4*)dst, bytes / 16);
      cudaEventRecord(b, st[0]);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("SM copy %d CTAs: %.3f ms = %.0f GB/s (copy bytes)\n", g, ms, bytes / ms / 1e6);
  }
  return 0;
}
