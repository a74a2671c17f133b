// mlck_common.cuh -- shared helpers for the sm_100a checkpoint data path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace mlck {

// Error kinds carried across the C ABI (include/mlck_b200.h): the C++ shim
// rethrows kInvalid as std::invalid_argument and kRuntime / kCuda as
// std::runtime_error with the same text the reference uses.
enum Status : int { kOk = 0, kInvalid = 1, kRuntime = 2, kCuda = 3 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(kInvalid, m); }
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Error(kRuntime, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(kCuda, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define MLCK_CUDA(call) ::mlck::cuda_check((call), #call)

// Device allocation rounded up to whole 2 MiB pages.  Measured on B200
// (scripts/micro/ring_ipc.cu): a buffer whose cudaMalloc size is not a
// 64 KiB multiple is mapped with small pages, and copy-engine NVLink pushes
// into / out of it run at ~540 GB/s instead of 776 GB/s.
inline void dev_malloc(void** p, uint64_t n) {
  constexpr uint64_t kPage = 2ull << 20;
  MLCK_CUDA(cudaMalloc(p, n >= kPage ? (n + kPage - 1) / kPage * kPage : n));
}

// Copy-engine copy split into a 64 KiB-multiple bulk and a short tail.
// Measured on B200 (scripts/micro/ring_ipc.cu): a peer copy whose size is
// not a multiple of 64 KiB runs at 548 GB/s instead of 776 GB/s -- records
// have arbitrary byte sizes.
inline void ce_copy(void* dst, const void* src, uint64_t n, cudaMemcpyKind kind, cudaStream_t s) {
  constexpr uint64_t kGrain = 64 << 10;
  const uint64_t bulk = n >= kGrain ? n / kGrain * kGrain : 0;
  if (bulk) MLCK_CUDA(cudaMemcpyAsync(dst, src, bulk, kind, s));
  if (n > bulk)
    MLCK_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + bulk, static_cast<const uint8_t*>(src) + bulk,
                              n - bulk, kind, s));
}

// Thread-local message of the last failing C-ABI call (defined in capi.cu).
std::string& last_error();

// Runs f, mapping exceptions to the C-ABI status codes.
template <typename F>
int api_call(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return kRuntime;
  }
}

__host__ __device__ constexpr uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ constexpr uint64_t align_up(uint64_t a, uint64_t b) { return div_up(a, b) * b; }

constexpr int kSmCount = 148;  // B200: 2 dies x 74 SMs

// ---- memory-model helpers (inline PTX, sm_100a) -------------------------
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming 128-bit load that does not allocate in L1 (each byte of the
// state arena is read exactly once per pack).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
#ifndef MLCK_ST_HINT
#define MLCK_ST_HINT ".cs"  // streaming (evict-first): the outputs are GB-sized and read once later; pack 0.80 -> 0.78 ms
#endif
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global" MLCK_ST_HINT ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

}  // namespace mlck
