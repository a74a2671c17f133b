// Development microbenchmark: the N > 1 replica push as bench.py runs it --
// one process per GPU, ring successor buffers opened through CUDA IPC --
// copy engines (cudaMemcpyAsync, Default kind) vs SM stores, alone and
// beside a busy all-SM kernel.
#include <cstdio>
#include <cstdint>
#include <atomic>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../include/mlck_b200.h"

struct Shared {
  std::atomic<int> arrive[64];
  cudaIpcMemHandle_t h0[8], h1[8];
};

__global__ void __launch_bounds__(1024, 1) push(const uint4* __restrict__ src, uint64_t n, uint4* d0, uint4* d1) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) {
    const uint4 v = src[i];
    d0[i] = v;
    d1[i] = v;
  }
}
__global__ void __launch_bounds__(1024, 1) busy(const uint4* __restrict__ src, uint64_t n, int iters, uint4* sink) {
  uint4 acc{};
  for (int it = 0; it < iters; ++it)
    for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) {
      const uint4 v = src[i];
      acc.x ^= v.x * 0x9e3779b1u; acc.y += v.y; acc.z ^= v.z; acc.w += v.w * 3u;
    }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

static Shared* sh;
static int N, bar_gen = 0;
static void barrier() {
  const int k = bar_gen++;
  sh->arrive[k].fetch_add(1);
  while (sh->arrive[k].load() < N) usleep(50);
}

static void child(int g) {
  cudaSetDevice(g);
  const uint64_t bytes = (uint64_t)(atof(getenv("GB") ? getenv("GB") : "4") * (1ull << 30)) / 4096 * 4096 + (getenv("ODD") ? atoi(getenv("ODD")) : 0);
  uint4 *src, *mine0, *mine1;
  // ROUND=1: allocations rounded up to 2 MiB, copies keep the odd size
  const uint64_t alloc = getenv("ROUND") ? (bytes + (2u << 20) - 1) / (2u << 20) * (2u << 20) : bytes;
  cudaMalloc(&src, alloc);
  cudaMemset(src, g, bytes);
  cudaMalloc(&mine0, alloc);
  cudaMalloc(&mine1, alloc);
  cudaIpcGetMemHandle(&sh->h0[g], mine0);
  cudaIpcGetMemHandle(&sh->h1[g], mine1);
  barrier();
  void *d0, *d1;
  cudaIpcOpenMemHandle(&d0, sh->h0[(g + 1) % N], cudaIpcMemLazyEnablePeerAccess);
  cudaIpcOpenMemHandle(&d1, sh->h1[(g + 2) % N], cudaIpcMemLazyEnablePeerAccess);
  cudaFuncSetAttribute(push, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  cudaFuncSetAttribute(busy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t a, b, j, ba, bb;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&ba); cudaEventCreate(&bb);
  cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
  auto run = [&](const char* name, int mode) {
    float ms = 0, bms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      barrier();
      cudaEventRecord(a, s0);
      if (mode >= 10) {  // busy kernel on s1 beside the push
        cudaStreamWaitEvent(s1, a);
        cudaEventRecord(ba, s1);
        busy<<<148, 1024, 200 * 1024, s1>>>(src, bytes / 16, 12, mine0);
        cudaEventRecord(bb, s1);
      }
      if (mode % 10 == 0) {
        cudaMemcpyAsync(d0, src, bytes, cudaMemcpyDefault, s0);
        cudaMemcpyAsync(d1, src, bytes, cudaMemcpyDefault, s0);
      } else if (mode % 10 == 1) {
        push<<<148, 1024, 120 * 1024, s0>>>(src, bytes / 16, (uint4*)d0, (uint4*)d1);
      } else if (mode % 10 == 2) {
        cudaMemcpyPeerAsync(d0, (g + 1) % N, src, g, bytes, s0);
        cudaMemcpyPeerAsync(d1, (g + 2) % N, src, g, bytes, s0);
      }
      cudaEventRecord(b, s0);
      cudaDeviceSynchronize();
      cudaEventElapsedTime(&ms, a, b);
      if (mode >= 10) cudaEventElapsedTime(&bms, ba, bb);
    }
    printf("rank %d %-28s push %.2f ms = %.0f GB/s egress%s%.2f ms (%s)\n", g, name, ms, 2 * bytes / ms / 1e6,
           mode >= 10 ? ", busy kernel " : "", mode >= 10 ? bms : 0.f, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  };
  if (getenv("FNV")) {  // the real hash kernel (libmlck_b200) beside the copy-engine push
    mlck_ctx* ctx;
    mlck_ctx_create(g, &ctx);
    uint64_t h;
    mlck_fnv1a64(ctx, src, bytes, 0xcbf29ce484222325ull, &h);
    // bench order: producer kernel on s0 -> event -> copies on s1 wait on it ->
    // hash on s0 (ctx stream = s0), i.e. copies and hash released together
    mlck_ctx_set_stream(ctx, s0);
    for (int rep = 0; rep < 3; ++rep) {
      float ms = 0, fms = 0;
      cudaDeviceSynchronize();
      barrier();
      busy<<<148, 1024, 200 * 1024, s0>>>(src, bytes / 16, 1, mine0);
      cudaEventRecord(j, s0);
      cudaStreamWaitEvent(s1, j);
      cudaEventRecord(a, s1);
      cudaMemcpyAsync(d0, src, bytes, cudaMemcpyDefault, s1);
      cudaMemcpyAsync(d1, src, bytes, cudaMemcpyDefault, s1);
      cudaEventRecord(b, s1);
      cudaEventRecord(ba, s0);
      mlck_fnv1a64(ctx, src, bytes, 0xcbf29ce484222325ull, &h);
      cudaEventRecord(bb, s0);
      cudaDeviceSynchronize();
      cudaEventElapsedTime(&ms, a, b);
      cudaEventElapsedTime(&fms, ba, bb);
      printf("rank %d bench order: push %.2f ms = %.0f GB/s, hash %.2f ms\n", g, ms, 2 * bytes / ms / 1e6, fms);
    }
    mlck_ctx_set_stream(ctx, nullptr);
    for (int mode = 0; mode < 3; ++mode) {
      float ms = 0, fms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        barrier();
        cudaEventRecord(a, s0);
        if (mode < 2) {
          cudaMemcpyAsync(d0, src, bytes, cudaMemcpyDefault, s0);
          cudaMemcpyAsync(d1, src, bytes, cudaMemcpyDefault, s0);
        }
        cudaEventRecord(b, s0);
        cudaEventRecord(ba, 0);
        if (mode > 0) for (int k = 0; k < 3; ++k) mlck_fnv1a64(ctx, src, bytes, 0xcbf29ce484222325ull, &h);
        cudaEventRecord(bb, 0);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, a, b);
        cudaEventElapsedTime(&fms, ba, bb);
      }
      printf("rank %d FNV mode %d (0 push, 1 push||3 hashes, 2 hashes): push %.2f ms = %.0f GB/s, 3 hashes %.2f ms\n",
             g, mode, ms, 2 * bytes / ms / 1e6, fms);
      fflush(stdout);
    }
    return;
  }
  run("CE memcpyAsync Default", 0);
  run("CE memcpyPeerAsync", 2);
  run("SM push 148", 1);
  run("CE Default || busy", 10);
  run("CE Peer || busy", 12);
}

int main(int argc, char** argv) {
  N = argc > 1 ? atoi(argv[1]) : 4;  // no CUDA call before fork
  sh = static_cast<Shared*>(mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0));
  for (int g = 0; g < N; ++g)
    if (fork() == 0) {
      child(g);
      _exit(0);
    }
  for (int g = 0; g < N; ++g) wait(nullptr);
  return 0;
}
