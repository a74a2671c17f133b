// log.cu -- K4: upstream boundary logging (LogKey / UpstreamLog / gc_logs,
// engine.hpp:55-94; producers engine.hpp:381-387 and 404-411).
//
// The reference copies each boundary tensor into a std::map<LogKey,
// std::vector<float>> on the critical path.  Here put() only records an
// event on the producer stream; the copy runs on a low-priority side stream:
//   kind 0 -> pinned host ring, copy engine D2H (PCIe / C2C bound);
//   kind 1 -> device ring (a peer GPU's HBM over NVLink when `device`
//             differs from the context's device), SM copy kernel;
//   kind 2 -> a caller-owned device ring (e.g. a ring successor's buffer
//             opened through CUDA IPC), copy engine over NVLink.
// The key index stays on the host in std::map order, so entry(i) enumerates
// exactly like the reference map; gc_logs drops iteration < window start and
// returns the ring ranges to a first-fit free list.
#include <cstring>
#include <map>
#include <string>
#include <tuple>

#include "../../include/mlck_b200.h"
#include "kernels.cuh"

using namespace mlck;

namespace {

struct Key {
  uint64_t iteration;
  uint32_t micro_batch, boundary;
  uint8_t direction;
  bool operator<(const Key& o) const {
    return std::tie(iteration, micro_batch, boundary, direction) <
           std::tie(o.iteration, o.micro_batch, o.boundary, o.direction);
  }
};
struct Entry {
  uint64_t off, n_floats;
};

std::string missing(const Key& k) {  // engine.hpp:74-77
  return "upstream log missing entry: iteration " + std::to_string(k.iteration) + " micro-batch " +
         std::to_string(k.micro_batch) + " boundary " + std::to_string(k.boundary) +
         (k.direction ? " bwd" : " fwd");
}
}  // namespace

struct mlck_ctx;
extern "C" int mlck_ctx_device_stream_(mlck_ctx* ctx, int* device, void** stream);

struct mlck_log {
  mlck_ctx* ctx = nullptr;
  int kind = 0, device = 0, ctx_device = 0;  // kind 2: caller-owned device ring
  uint8_t* base = nullptr;
  uint64_t cap = 0, used = 0;
  std::map<Key, Entry> entries;
  std::map<uint64_t, uint64_t> free_list;  // off -> size
  cudaStream_t side = nullptr;
  cudaEvent_t ev = nullptr;
  cudaEvent_t copied = nullptr;  // recorded on `side` after every copy
  bool async = false;            // false: the ctx stream waits for each copy (src reusable)

  uint64_t alloc(uint64_t bytes) {
    bytes = align_up(bytes ? bytes : 16, 256);
    for (auto it = free_list.begin(); it != free_list.end(); ++it) {
      if (it->second >= bytes) {
        const uint64_t off = it->first, rest = it->second - bytes;
        free_list.erase(it);
        if (rest) free_list[off + bytes] = rest;
        used += bytes;
        return off;
      }
    }
    throw_runtime("upstream log budget exceeded: need " + std::to_string(bytes) +
                  " bytes, ring capacity " + std::to_string(cap) + " (" + std::to_string(used) +
                  " in use)");
  }
  void release(uint64_t off, uint64_t bytes) {
    bytes = align_up(bytes ? bytes : 16, 256);
    used -= bytes;
    auto it = free_list.emplace(off, bytes).first;
    auto nx = std::next(it);
    if (nx != free_list.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_list.erase(nx);
    }
    if (it != free_list.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_list.erase(it);
      }
    }
  }
};

namespace {
template <typename F>
int log_api(F&& f) {
  return api_call(static_cast<F&&>(f));
}
}  // namespace

extern "C" {

int mlck_log_create(mlck_ctx* ctx, int kind, int device, uint64_t capacity, mlck_log** out) {
  return log_api([&] {
    if (kind != 0 && kind != 1) throw_invalid("log kind must be 0 (pinned host) or 1 (device)");
    auto* l = new mlck_log();
    l->ctx = ctx;
    l->kind = kind;
    void* stream = nullptr;
    mlck_ctx_device_stream_(ctx, &l->ctx_device, &stream);
    l->device = kind == 1 ? device : l->ctx_device;
    l->cap = align_up(capacity ? capacity : 256, 256);
    if (kind == 0) {
      MLCK_CUDA(cudaSetDevice(l->ctx_device));
      MLCK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&l->base), l->cap, cudaHostAllocPortable));
    } else {
      MLCK_CUDA(cudaSetDevice(l->device));
      dev_malloc(reinterpret_cast<void**>(&l->base), l->cap);
      MLCK_CUDA(cudaSetDevice(l->ctx_device));
      if (l->device != l->ctx_device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(l->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MLCK_CUDA(e);
        cudaGetLastError();
      }
    }
    int lo = 0, hi = 0;
    MLCK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MLCK_CUDA(cudaStreamCreateWithPriority(&l->side, cudaStreamNonBlocking, lo));  // lowest
    MLCK_CUDA(cudaEventCreateWithFlags(&l->ev, cudaEventDisableTiming));
    MLCK_CUDA(cudaEventCreateWithFlags(&l->copied, cudaEventDisableTiming));
    l->free_list[0] = l->cap;
    *out = l;
  });
}

int mlck_log_create_external(mlck_ctx* ctx, void* device_base, uint64_t capacity, mlck_log** out) {
  return log_api([&] {
    if (!device_base || capacity < 256) throw_invalid("external log ring: null base or capacity < 256");
    auto* l = new mlck_log();
    l->ctx = ctx;
    l->kind = 2;
    void* stream = nullptr;
    mlck_ctx_device_stream_(ctx, &l->ctx_device, &stream);
    l->device = l->ctx_device;
    l->base = static_cast<uint8_t*>(device_base);
    l->cap = capacity / 256 * 256;
    int lo = 0, hi = 0;
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    MLCK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MLCK_CUDA(cudaStreamCreateWithPriority(&l->side, cudaStreamNonBlocking, lo));  // lowest
    MLCK_CUDA(cudaEventCreateWithFlags(&l->ev, cudaEventDisableTiming));
    MLCK_CUDA(cudaEventCreateWithFlags(&l->copied, cudaEventDisableTiming));
    l->free_list[0] = l->cap;
    *out = l;
  });
}

int mlck_log_destroy(mlck_log* l) {
  return log_api([&] {
    if (!l) return;
    cudaSetDevice(l->ctx_device);
    cudaStreamSynchronize(l->side);
    if (l->kind == 2) {
      // the ring belongs to the caller
    } else if (l->kind == 0) {
      cudaFreeHost(l->base);
    } else {
      cudaSetDevice(l->device);
      cudaFree(l->base);
      cudaSetDevice(l->ctx_device);
    }
    cudaStreamDestroy(l->side);
    cudaEventDestroy(l->ev);
    cudaEventDestroy(l->copied);
    delete l;
  });
}

int mlck_log_put(mlck_log* l, uint64_t it, uint32_t mb, uint32_t boundary, uint8_t dir,
                 const float* src, uint64_t n) {
  return log_api([&] {
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    const Key k{it, mb, boundary, dir};
    auto found = l->entries.find(k);
    if (found != l->entries.end()) {  // map assignment overwrites (engine.hpp:384)
      MLCK_CUDA(cudaStreamSynchronize(l->side));
      l->release(found->second.off, 4 * found->second.n_floats);
      l->entries.erase(found);
    }
    const uint64_t off = l->alloc(4 * n);
    void* stream = nullptr;
    int dev = 0;
    mlck_ctx_device_stream_(l->ctx, &dev, &stream);
    // the copy starts once the producer's work on the ctx stream is done
    MLCK_CUDA(cudaEventRecord(l->ev, static_cast<cudaStream_t>(stream)));
    MLCK_CUDA(cudaStreamWaitEvent(l->side, l->ev, 0));
    if (n) {
      if (l->kind == 0) {
        MLCK_CUDA(cudaMemcpyAsync(l->base + off, src, 4 * n, cudaMemcpyDeviceToHost, l->side));
      } else if (l->kind == 2) {  // copy engine (a peer's HBM over NVLink for an IPC ring)
        ce_copy(l->base + off, src, 4 * n, cudaMemcpyDefault, l->side);
      } else if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        launch_copy16(l->base + off, src, 4 * n, l->side);
      } else {
        ce_copy(l->base + off, src, 4 * n, cudaMemcpyDefault, l->side);
      }
    }
    l->entries[k] = {off, n};
    MLCK_CUDA(cudaEventRecord(l->copied, l->side));
    // ordered mode: later work on the ctx stream may overwrite src
    if (!l->async) MLCK_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), l->copied, 0));
  });
}

int mlck_log_set_async(mlck_log* l, int async) {
  return log_api([&] { l->async = async != 0; });
}

int mlck_log_fence(mlck_log* l, void* stream) {
  return log_api([&] {
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!st) {
      void* cs = nullptr;
      int dev = 0;
      mlck_ctx_device_stream_(l->ctx, &dev, &cs);
      st = static_cast<cudaStream_t>(cs);
    }
    MLCK_CUDA(cudaEventRecord(l->copied, l->side));
    MLCK_CUDA(cudaStreamWaitEvent(st, l->copied, 0));
  });
}

int mlck_log_sync(mlck_log* l) {
  return log_api([&] {
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    MLCK_CUDA(cudaStreamSynchronize(l->side));
  });
}

static int log_get_impl(mlck_log* l, const Key& k, float* out, uint64_t cap, uint64_t* n,
                        bool device_out) {
  return log_api([&] {
    auto it = l->entries.find(k);
    if (it == l->entries.end()) throw_runtime(missing(k));
    if (n) *n = it->second.n_floats;
    if (!out) return;
    if (cap < it->second.n_floats) throw_invalid("log get: buffer too small");
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    const uint64_t bytes = 4 * it->second.n_floats;
    if (device_out) {
      // stream-ordered on the ctx stream (after the entry's copy landed): the
      // destination may still be read by work queued before this call
      void* cs = nullptr;
      int dev = 0;
      mlck_ctx_device_stream_(l->ctx, &dev, &cs);
      MLCK_CUDA(cudaEventRecord(l->copied, l->side));
      MLCK_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(cs), l->copied, 0));
      MLCK_CUDA(cudaMemcpyAsync(out, l->base + it->second.off, bytes, cudaMemcpyDefault,
                                static_cast<cudaStream_t>(cs)));
      return;
    }
    MLCK_CUDA(cudaStreamSynchronize(l->side));
    if (l->kind == 0) {
      std::memcpy(out, l->base + it->second.off, bytes);
    } else {
      MLCK_CUDA(cudaMemcpy(out, l->base + it->second.off, bytes, cudaMemcpyDefault));
    }
  });
}

int mlck_log_get(mlck_log* l, uint64_t it, uint32_t mb, uint32_t boundary, uint8_t dir,
                 float* host_out, uint64_t cap, uint64_t* n) {
  return log_get_impl(l, Key{it, mb, boundary, dir}, host_out, cap, n, false);
}
int mlck_log_get_device(mlck_log* l, uint64_t it, uint32_t mb, uint32_t boundary, uint8_t dir,
                        float* dst, uint64_t cap, uint64_t* n) {
  return log_get_impl(l, Key{it, mb, boundary, dir}, dst, cap, n, true);
}

uint64_t mlck_log_count(mlck_log* l) { return l ? l->entries.size() : 0; }
uint64_t mlck_log_bytes(mlck_log* l) {  // UpstreamLog::bytes (engine.hpp:81-85)
  uint64_t b = 0;
  if (l)
    for (const auto& kv : l->entries) b += 4 * kv.second.n_floats;
  return b;
}

int mlck_log_entry(mlck_log* l, uint64_t index, uint64_t* it, uint32_t* mb, uint32_t* boundary,
                   uint8_t* dir, float* host_out, uint64_t cap, uint64_t* n) {
  if (!l || index >= l->entries.size())
    return log_api([&] { throw_invalid("log entry index out of range"); });
  auto e = l->entries.begin();
  std::advance(e, static_cast<long>(index));
  *it = e->first.iteration;
  *mb = e->first.micro_batch;
  *boundary = e->first.boundary;
  *dir = e->first.direction;
  return log_get_impl(l, e->first, host_out, cap, n, false);
}

int mlck_gc_logs(mlck_log* l, uint64_t persisted_window_start) {
  return log_api([&] {
    MLCK_CUDA(cudaSetDevice(l->ctx_device));
    MLCK_CUDA(cudaStreamSynchronize(l->side));
    for (auto it = l->entries.begin(); it != l->entries.end();) {
      if (it->first.iteration < persisted_window_start) {  // engine.hpp:91-93
        l->release(it->second.off, 4 * it->second.n_floats);
        it = l->entries.erase(it);
      } else {
        ++it;
      }
    }
  });
}

// ---- log storage budget (recovery.hpp:296-317) ---------------------------
int64_t mlck_upstream_log_bytes(int32_t token_dim, int32_t pp_stages, int32_t microbatches,
                                int64_t microbatch_size, int32_t dp_degree, int64_t wsparse) {
  const int64_t boundaries = pp_stages > 1 ? pp_stages - 1 : 0;
  const int64_t per_tensor = microbatch_size * token_dim * static_cast<int64_t>(sizeof(float));
  const int64_t entries_per_iter = 2 * boundaries * microbatches * dp_degree;
  return 2 * wsparse * entries_per_iter * per_tensor;  // live window + the one being persisted
}

int mlck_check_log_budget(int32_t token_dim, int32_t pp_stages, int32_t microbatches, int64_t microbatch_size,
                          int32_t dp_degree, int64_t wsparse, double cpu_mem_per_node, int32_t nodes) {
  return log_api([&] {
    if (cpu_mem_per_node <= 0) return;
    const int64_t need = mlck_upstream_log_bytes(token_dim, pp_stages, microbatches, microbatch_size, dp_degree, wsparse);
    const double have = cpu_mem_per_node * nodes;
    if (static_cast<double>(need) > have)
      throw_invalid("upstream log budget exceeded: need " + std::to_string(need) + " bytes of host memory, budget " +
                    std::to_string(static_cast<int64_t>(have)));
  });
}

}  // extern "C"
