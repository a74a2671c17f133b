// Development microbenchmark: every GPU pushes a buffer to its r = 2 ring
// successors at once (the N > 1 snapshot replica pattern). Copy engines
// (one stream, or one stream per successor, optionally split in pieces) vs
// SM stores from k SMs.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) push(const uint4* __restrict__ src, uint64_t n, uint4* d0, uint4* d1) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) {
    const uint4 v = src[i];
    d0[i] = v;
    d1[i] = v;
  }
}

// stand-in for the hash: every SM busy (one 1024-thread CTA with 200 KB of
// smem each, like the FNV kernel) reading HBM for `iters` passes
__global__ void __launch_bounds__(1024, 1) busy(const uint4* __restrict__ src, uint64_t n, int iters, uint4* sink) {
  uint4 acc{};
  for (int it = 0; it < iters; ++it)
    for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n; i += gridDim.x * 1024ull) {
      const uint4 v = src[i];
      acc.x ^= v.x * 0x9e3779b1u; acc.y += v.y; acc.z ^= v.z; acc.w += v.w * 3u;
    }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

int main() {
  int N;
  cudaGetDeviceCount(&N);
  const uint64_t bytes = 4ull << 30;
  std::vector<uint4*> src(N), dst0(N), dst1(N);
  std::vector<cudaStream_t> s0(N), s1(N);
  std::vector<cudaEvent_t> a(N), b(N);
  for (int g = 0; g < N; ++g) {
    cudaSetDevice(g);
    for (int p = 0; p < N; ++p) if (p != g) cudaDeviceEnablePeerAccess(p, 0);
    cudaMalloc(&src[g], bytes);
    cudaMemset(src[g], g, bytes);
    cudaMalloc(&dst0[g], bytes);  // written by predecessor g-1
    cudaMalloc(&dst1[g], bytes);  // written by g-2
    cudaStreamCreateWithFlags(&s0[g], cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1[g], cudaStreamNonBlocking);
    cudaEventCreate(&a[g]);
    cudaEventCreate(&b[g]);
    cudaFuncSetAttribute(push, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    cudaFuncSetAttribute(busy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  auto run = [&](const char* name, auto launch) {
    float worst = 0;
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < N; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
      for (int g = 0; g < N; ++g) { cudaSetDevice(g); cudaEventRecord(a[g], s0[g]); }
      for (int g = 0; g < N; ++g) { cudaSetDevice(g); launch(g); }
      worst = 0;
      for (int g = 0; g < N; ++g) {
        cudaSetDevice(g);
        cudaEventRecord(b[g], s0[g]);
        cudaEventSynchronize(b[g]);
        float ms;
        cudaEventElapsedTime(&ms, a[g], b[g]);
        if (ms > worst) worst = ms;
      }
    }
    printf("%-34s %.2f ms, egress %.0f GB/s/GPU (%s)\n", name, worst, 2 * bytes / worst / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  cudaEvent_t j[16];
  for (int g = 0; g < N; ++g) { cudaSetDevice(g); cudaEventCreateWithFlags(&j[g], cudaEventDisableTiming); }
  run("CE one stream, serial", [&](int g) {
    cudaMemcpyPeerAsync(dst0[(g + 1) % N], (g + 1) % N, src[g], g, bytes, s0[g]);
    cudaMemcpyPeerAsync(dst1[(g + 2) % N], (g + 2) % N, src[g], g, bytes, s0[g]);
  });
  run("CE two streams", [&](int g) {
    cudaEventRecord(j[g], s0[g]);
    cudaStreamWaitEvent(s1[g], j[g]);
    cudaMemcpyPeerAsync(dst0[(g + 1) % N], (g + 1) % N, src[g], g, bytes, s0[g]);
    cudaMemcpyPeerAsync(dst1[(g + 2) % N], (g + 2) % N, src[g], g, bytes, s1[g]);
    cudaEventRecord(j[g], s1[g]);
    cudaStreamWaitEvent(s0[g], j[g]);
  });
  run("busy kernel alone (s0)", [&](int g) {
    busy<<<148, 1024, 200 * 1024, s0[g]>>>(src[g], bytes / 16, 2, dst1[g]);
  });
  run("CE serial || busy kernel", [&](int g) {
    cudaEventRecord(j[g], s0[g]);
    cudaStreamWaitEvent(s1[g], j[g]);
    busy<<<148, 1024, 200 * 1024, s1[g]>>>(src[g], bytes / 16, 2, dst1[g]);
    cudaMemcpyPeerAsync(dst0[(g + 1) % N], (g + 1) % N, src[g], g, bytes, s0[g]);
    cudaMemcpyPeerAsync(dst1[(g + 2) % N], (g + 2) % N, src[g], g, bytes, s0[g]);
    cudaEventRecord(j[g], s1[g]);
    cudaStreamWaitEvent(s0[g], j[g]);
  });
  run("CE serial (cudaMemcpyAsync Default) || busy", [&](int g) {
    cudaEventRecord(j[g], s0[g]);
    cudaStreamWaitEvent(s1[g], j[g]);
    busy<<<148, 1024, 200 * 1024, s1[g]>>>(src[g], bytes / 16, 2, dst1[g]);
    cudaMemcpyAsync(dst0[(g + 1) % N], src[g], bytes, cudaMemcpyDefault, s0[g]);
    cudaMemcpyAsync(dst1[(g + 2) % N], src[g], bytes, cudaMemcpyDefault, s0[g]);
    cudaEventRecord(j[g], s1[g]);
    cudaStreamWaitEvent(s0[g], j[g]);
  });
  for (int pieces : {4, 16}) {
    char nm[64];
    snprintf(nm, 64, "CE two streams, %d pieces interleaved", pieces);
    run(nm, [&](int g) {
      cudaEventRecord(j[g], s0[g]);
      cudaStreamWaitEvent(s1[g], j[g]);
      const uint64_t piece = bytes / pieces;
      for (int p = 0; p < pieces; ++p) {
        cudaMemcpyPeerAsync((char*)dst0[(g + 1) % N] + p * piece, (g + 1) % N, (char*)src[g] + p * piece, g, piece, s0[g]);
        cudaMemcpyPeerAsync((char*)dst1[(g + 2) % N] + p * piece, (g + 2) % N, (char*)src[g] + p * piece, g, piece, s1[g]);
      }
      cudaEventRecord(j[g], s1[g]);
      cudaStreamWaitEvent(s0[g], j[g]);
    });
  }
  for (int k : {16, 32, 48, 64, 96, 148}) {
    char nm[64];
    snprintf(nm, 64, "SM push, %d SMs", k);
    run(nm, [&](int g) {
      push<<<k, 1024, 120 * 1024, s0[g]>>>(src[g], bytes / 16, dst0[(g + 1) % N], dst1[(g + 2) % N]);
    });
  }
  return 0;
}
