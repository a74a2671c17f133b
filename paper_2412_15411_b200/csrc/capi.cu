// capi.cu -- host runtime behind include/mlck_b200.h.
//
// Owns the device arenas, blobs, gradient log and boundary log, builds the
// per-call segment tables and launches the sm_100a kernels of kernels.cu.
// Error texts follow the reference exceptions they replace (file:line at
// each site) so the C++ shim (include/moelab_b200) can rethrow them verbatim.
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include <cuda.h>

#include "../../include/mlck_b200.h"
#include "engine.cuh"
#include "kernels.cuh"

using namespace mlck;

namespace mlck {
std::string& last_error() {
  thread_local std::string e;
  return e;
}
}  // namespace mlck

namespace {

template <typename F>
int api(F&& f) {
  return api_call(static_cast<F&&>(f));
}

constexpr uint64_t kAlign = 256;
constexpr uint32_t kMagic = 0x4b434c4du;

}  // namespace

// =========================================================================
// context
// =========================================================================
struct mlck_ctx {
  int device = 0;
  // device ranges opened through CUDA IPC (another GPU's memory: pointer
  // attributes report the mapping device, not the owner)
  std::vector<std::pair<uint64_t, uint64_t>> ipc_ranges;
  std::vector<mlck_blob*> blobs;  // live blobs (mlck_ipc_close drops replicas inside a closed mapping)
  bool is_ipc(const void* p) const {
    const uint64_t a = reinterpret_cast<uint64_t>(p);
    for (const auto& r : ipc_ranges)
      if (a >= r.first && a < r.first + r.second) return true;
    return false;
  }
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  struct Stage {
    uint8_t* host = nullptr;
    uint8_t* dev = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
    bool used = false;
  } stage[2];
  int cur = 0;
  uint32_t* fnv_scratch = nullptr;
  size_t fnv_words = 0;
  // record verification (parse_record's checksum) alternates between two
  // side streams, each with its own look-back scratch, so one record's hash
  // fills the SMs the previous one leaves as it drains, and the ctx stream
  // stays free for the walk and the conversion replay
  cudaStream_t vside[2] = {};
  cudaEvent_t ev_vside[2] = {}, ev_vmain = nullptr;
  uint32_t* vscratch[2] = {};
  size_t vwords[2] = {};
  uint32_t* vscratch_for(int i, uint64_t n) {
    const size_t need = fnv_scratch_words(n);
    if (need > vwords[i]) {
      MLCK_CUDA(cudaStreamSynchronize(vside[i]));
      if (vscratch[i]) MLCK_CUDA(cudaFree(vscratch[i]));
      vwords[i] = align_up(std::max<size_t>(need, 4096), 1024);
      MLCK_CUDA(cudaMalloc(&vscratch[i], vwords[i] * 4));
      MLCK_CUDA(cudaMemsetAsync(vscratch[i], 0, vwords[i] * 4, vside[i]));
    }
    return vscratch[i];
  }
  // SMs the hash kernel leaves free (mlck_ctx_set_hash_reserve)
  int hash_reserve = 0;
  // Asynchronous trailer hash (mlck_ctx_set_hash_async, default on): the
  // default transport's FNV kernel runs on hstream after the pack, so the
  // next pack (next slot, another blob) need not wait for it -- the hash is
  // off the snapshot's critical path, as PAPER.md's overlap intends.  Every
  // reader of a record waits for its `written` event; the raw helpers and
  // synchronize join all hashes (join_hash).
  bool hash_async = false;
  // conversion: the records' witnessed verification on `convert_overlap`
  // SMs beside the replay (0 = verification first, then the replay)
  int convert_overlap = 0;
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_packed_h = nullptr, ev_hash_last = nullptr;
  bool hash_pending = false;
  uint32_t* hscratch = nullptr;
  size_t hwords = 0;
  unsigned long long* hresult = nullptr;
  uint32_t* hscratch_for(uint64_t n) {
    const size_t need = fnv_scratch_words(n);
    if (need > hwords) {
      MLCK_CUDA(cudaStreamSynchronize(hstream));
      if (hscratch) MLCK_CUDA(cudaFree(hscratch));
      hwords = align_up(std::max<size_t>(need, 4096), 1024);
      MLCK_CUDA(cudaMalloc(&hscratch, hwords * 4));
      MLCK_CUDA(cudaMemsetAsync(hscratch, 0, hwords * 4, hstream));
    }
    return hscratch;
  }
  void join_hash() {
    if (hash_pending) MLCK_CUDA(cudaStreamWaitEvent(stream, ev_hash_last, 0));
  }
  // records keep the hash kernel's segment starts (a witness) and are
  // re-verified against it (fnv.cuh); counters for tests and the bench
  bool witness = true;
  uint64_t witness_used = 0, witness_fallbacks = 0;
  unsigned long long* results = nullptr;       // device [results_cap]
  unsigned long long* host_results = nullptr;  // pinned [results_cap]
  size_t results_cap = 0;
  // grows both result arrays to >= n words (the stream is idle or synchronized)
  void results_for(size_t n) {
    if (n <= results_cap) return;
    MLCK_CUDA(cudaStreamSynchronize(stream));
    if (results) MLCK_CUDA(cudaFree(results));
    if (host_results) MLCK_CUDA(cudaFreeHost(host_results));
    results_cap = align_up(std::max<size_t>(n, 64), 64);
    MLCK_CUDA(cudaMalloc(&results, results_cap * 8));
    MLCK_CUDA(cudaMallocHost(&host_results, results_cap * 8));
  }
  cudaEvent_t ev[16] = {};
  // Optional per-kernel timing (CUDA events on the launch stream), read back
  // with mlck_ctx_timings() -- the benchmark's roofline denominator.
  bool timing = false;
  struct Timed {
    const char* label;
    cudaEvent_t a, b;
  };
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  void activate() const { MLCK_CUDA(cudaSetDevice(device)); }

  cudaEvent_t next_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      MLCK_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  // Brackets one launch; returns -1 when timing is off.
  int tbegin(const char* label, cudaStream_t on = nullptr) {
    if (!timing) return -1;
    Timed t{label, next_event(), next_event()};
    MLCK_CUDA(cudaEventRecord(t.a, on ? on : stream));
    timed.push_back(t);
    return static_cast<int>(timed.size()) - 1;
  }
  void tend(int idx, cudaStream_t on = nullptr) {
    if (idx >= 0) MLCK_CUDA(cudaEventRecord(timed[idx].b, on ? on : stream));
  }

  // Pinned staging + device mirror for one call's metadata.
  Stage& stage_for(size_t bytes) {
    cur ^= 1;
    Stage& s = stage[cur];
    if (s.used) MLCK_CUDA(cudaEventSynchronize(s.done));
    if (bytes > s.cap) {
      // the device copy may still be read by an in-flight kernel
      MLCK_CUDA(cudaStreamSynchronize(stream));
      if (s.host) MLCK_CUDA(cudaFreeHost(s.host));
      if (s.dev) MLCK_CUDA(cudaFree(s.dev));
      s.cap = align_up(std::max<size_t>(bytes, 1 << 16), 4096);
      MLCK_CUDA(cudaMallocHost(&s.host, s.cap));
      MLCK_CUDA(cudaMalloc(&s.dev, s.cap));
    }
    return s;
  }
  void stage_upload(Stage& s, size_t bytes) {
    MLCK_CUDA(cudaMemcpyAsync(s.dev, s.host, bytes, cudaMemcpyHostToDevice, stream));
    MLCK_CUDA(cudaEventRecord(s.done, stream));
    s.used = true;
  }
  uint32_t fnv_epoch = 0;
  // Snapshot transport (-1 = auto: 0 for replicas in local HBM, 1 for peer
  // replicas -- scripts/micro/push.cu: one copy engine drives 782 GB/s of
  // NVLink egress, SM stores saturate at ~717 GB/s and need >= 48 SMs; a
  // local copy-engine copy beside the hash contends with it (2.3 ms vs 0.6
  // ms alone), while the pack kernel writes the local replica for +0.24 ms):
  // 5 = pack kernel, then the FNV kernel stores the replicas as it hashes;
  // 3 = pack kernel, then kPushSms SMs push the replicas with NVLink
  // stores while the FNV kernel hashes on the other SMs; 1 = pack kernel,
  // then copy engines push the replicas while the FNV kernel hashes; 2 = one fused
  // kernel gathers, stores (local record and replicas, NVLink stores for
  // peers) and hashes; 0 = the pack kernel stores the replicas, then the FNV
  // kernel.
  int replica_mode = -1;
  // one copy stream for the replica push (measured: more streams do not
  // raise NVLink throughput and slow the concurrent hash)
  static constexpr int kPushStreams = 3;  // one per replica (pack::kMaxDst - 1)
  // transport 3: SMs reserved for the replica push (the FNV kernel runs on the rest)
  static constexpr int kPushSms = 16;
  cudaStream_t side[kPushStreams] = {};
  // transport 1: the record is packed in up to kPieces pieces of >= 64 MiB
  // (swept 4-64 at N=2: 16 best, 14.5 -> 14.0 ms),
  // each pushed as soon as it is packed
#ifndef MLCK_PUSH_PIECES
#define MLCK_PUSH_PIECES 16
#endif
  static constexpr int kPieces = MLCK_PUSH_PIECES;
  cudaEvent_t ev_packed = nullptr, ev_hashed = nullptr, ev_pushed[kPushStreams] = {}, ev_piece[kPieces] = {};
  uint8_t* patch = nullptr;
  uint64_t patch_cap = 0;
  uint8_t* patch_for(uint64_t bytes) {
    if (bytes > patch_cap) {
      MLCK_CUDA(cudaStreamSynchronize(stream));
      if (patch) MLCK_CUDA(cudaFree(patch));
      patch_cap = align_up(std::max<uint64_t>(bytes, 1 << 16), 1 << 16);
      MLCK_CUDA(cudaMalloc(&patch, patch_cap));
    }
    return patch;
  }
  // The hash kernel's look-back watchdog (fnv.cuh kSpinLimit) leaves a sticky
  // word in the scratch header; checked after the stream synchronizes.
  bool watchdog_seen = false;
  void read_watchdog() {
    for (uint32_t* sc : {fnv_scratch, vscratch[0], vscratch[1], hscratch}) {
      if (!sc) continue;
      uint32_t w = 0;
      MLCK_CUDA(cudaMemcpy(&w, sc + fnv_sticky_word(), 4, cudaMemcpyDeviceToHost));
      if (w) {
        MLCK_CUDA(cudaMemset(sc + fnv_sticky_word(), 0, 4));
        watchdog_seen = true;
      }
    }
  }
  void check_watchdog() {  // the stream is synchronized
    read_watchdog();
    if (watchdog_seen) {
      watchdog_seen = false;
      throw_runtime("fnv: the look-back watchdog tripped (a CTA of the hash kernel was not resident; "
                    "the hash of this call is invalid)");
    }
  }
  uint32_t* fnv_scratch_for(uint64_t n) {
    const size_t need = fnv_scratch_words(n);
    if (need > fnv_words) {
      MLCK_CUDA(cudaStreamSynchronize(stream));
      read_watchdog();
      if (fnv_scratch) MLCK_CUDA(cudaFree(fnv_scratch));
      fnv_words = align_up(std::max<size_t>(need, 4096), 1024);
      MLCK_CUDA(cudaMalloc(&fnv_scratch, fnv_words * 4));
      // epoch 0 never matches a launch: a zeroed array reads as "unpublished"
      MLCK_CUDA(cudaMemsetAsync(fnv_scratch, 0, fnv_words * 4, stream));
    }
    return fnv_scratch;
  }
  uint32_t next_epoch() {
    if (++fnv_epoch == 0) {  // wrapped: clear stale tags once
      MLCK_CUDA(cudaStreamSynchronize(stream));
      for (int i = 0; i < 2; ++i) MLCK_CUDA(cudaStreamSynchronize(vside[i]));
      MLCK_CUDA(cudaStreamSynchronize(hstream));
      if (hscratch) MLCK_CUDA(cudaMemset(hscratch, 0, hwords * 4));
      if (fnv_scratch) MLCK_CUDA(cudaMemset(fnv_scratch, 0, fnv_words * 4));
      for (int i = 0; i < 2; ++i)
        if (vscratch[i]) MLCK_CUDA(cudaMemset(vscratch[i], 0, vwords[i] * 4));
      fnv_epoch = 1;
    }
    return fnv_epoch;
  }
};

// =========================================================================
// state arena
// =========================================================================
struct mlck_state {
  mlck_ctx* ctx = nullptr;
  uint32_t n_ops = 0;
  int cb = 2;
  std::vector<uint64_t> P, step, full_off, code_off;
  std::vector<uint8_t> has_full, present;
  uint8_t* arena = nullptr;
  uint64_t arena_bytes = 0;
  uint64_t iteration = 0, data_seed = 0;

  float* master(uint32_t i) const { return reinterpret_cast<float*>(arena + full_off[i]); }
  void* codes(uint32_t i) const { return arena + code_off[i]; }
  void check_id(uint32_t id) const {
    if (id >= n_ops) throw_invalid("operator id " + std::to_string(id) + " out of range");
  }
};

// u32 words a record's witness buffer holds: one per 128-byte row of the body,
// plus the verifier's bulk over-read of a chunk's words (fnv_witness_tc_kernel)
inline uint64_t witness_alloc_words(uint64_t body) { return fnv_witness_words(body) + 1 + 520; }

struct mlck_blob {
  mlck_ctx* ctx = nullptr;
  uint8_t* dev = nullptr;
  uint64_t cap = 0, size = 0;
  std::vector<std::pair<uint8_t*, uint64_t>> replicas;
  // recorded on the ctx stream once the last record is complete in the blob
  // and in every replica (mlck_blob_replication polls it)
  cudaEvent_t written = nullptr;
  uint32_t written_replicas = 0;
  // the segment starts of the last record's hash (fnv.cuh, witness): valid
  // for a body of witness_n bytes when witness_n == size - 8
  uint32_t* witness = nullptr;
  uint64_t witness_cap = 0, witness_n = ~0ull;
  // witness buffers next to replicas (mlck_blob_add_replica_witness): each
  // record's witness follows it there, so a blob wrapped over the replica
  // verifies on the witnessed path
  std::vector<std::pair<uint8_t*, uint64_t>> witness_dsts;
  // mlck_blob_wrap: a read-only view of a record (and witness) the caller owns
  bool external = false, external_witness = false;

  void reserve(uint64_t n) {
    if (external) throw_invalid("a wrapped blob (mlck_blob_wrap) is read-only");
    if (n <= cap) return;
    ctx->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (dev) MLCK_CUDA(cudaFree(dev));
    cap = align_up(n, kAlign);
    dev_malloc(reinterpret_cast<void**>(&dev), cap);
    witness_n = ~0ull;
    if (ctx->witness) reserve_witness(cap);  // with the record buffer: never inside a snapshot
  }
  void reserve_witness(uint64_t body) {
    const uint64_t words = witness_alloc_words(body);
    if (words <= witness_cap) return;
    if (external_witness) throw_invalid("a wrapped blob (mlck_blob_wrap) is read-only");
    ctx->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (witness) MLCK_CUDA(cudaFree(witness));
    witness_cap = align_up(words, 1024);
    dev_malloc(reinterpret_cast<void**>(&witness), 4 * witness_cap);
  }
  uint32_t* witness_for(uint64_t body) {
    witness_n = ~0ull;
    if (!ctx->witness) return nullptr;
    reserve_witness(body);
    return witness;
  }
  bool has_witness() const { return witness && size >= 8 && witness_n == size - 8; }
};

struct mlck_gradlog {
  mlck_ctx* ctx = nullptr;
  uint32_t n_ops = 0;
  std::vector<uint64_t> P, off;  // float offsets inside one iteration slot
  uint64_t per_iter = 0;
  uint32_t cap = 0;
  float* pool = nullptr;
  std::vector<int64_t> ring_iter;
  std::vector<std::vector<uint8_t>> present;

  float* slot(uint64_t it, uint32_t op) {
    if (op >= n_ops) throw_invalid("gradient log: operator " + std::to_string(op) + " out of range");
    const uint32_t r = static_cast<uint32_t>(it % cap);
    if (ring_iter[r] != static_cast<int64_t>(it)) {
      ring_iter[r] = static_cast<int64_t>(it);
      std::fill(present[r].begin(), present[r].end(), 0);
    }
    present[r][op] = 1;
    return pool + r * per_iter + off[op];
  }
  const float* lookup(uint64_t it, uint32_t op) const {
    const uint32_t r = static_cast<uint32_t>(it % cap);
    if (op < n_ops && ring_iter[r] == static_cast<int64_t>(it) && present[r][op])
      return pool + r * per_iter + off[op];
    throw_runtime("gradient log missing iteration " + std::to_string(it) + " operator " +
                  std::to_string(op));
  }
};

namespace {

uint64_t state_mlst_size(const mlck_state* st) {
  uint64_t s = 28;
  for (uint32_t i = 0; i < st->n_ops; ++i) s += 16 + (st->present[i] ? 12 * st->P[i] : 0);
  return s;
}

template <typename T>
void put_le(std::vector<uint8_t>& b, T v) {
  const size_t o = b.size();
  b.resize(o + sizeof(T));
  std::memcpy(b.data() + o, &v, sizeof(T));
}

// Assembles a byte image as segments: inline bytes (headers) live in the
// staging buffer's meta region, payload spans point into device memory.
struct SegmentBuilder {
  std::vector<pack::Segment> segs;  // src of inline segments = meta offset (patched)
  std::vector<uint8_t> is_meta;
  std::vector<uint8_t> meta;
  uint64_t pos = 0;

  void begin_meta() {}
  template <typename T>
  void value(T v) {
    const uint64_t moff = meta.size();
    put_le(meta, v);
    if (!segs.empty() && is_meta.back() && segs.back().dst + segs.back().len == pos &&
        reinterpret_cast<uint64_t>(segs.back().src) + segs.back().len == moff) {
      segs.back().len += sizeof(T);
    } else {
      segs.push_back({pos, sizeof(T), reinterpret_cast<const uint8_t*>(moff)});
      is_meta.push_back(1);
    }
    pos += sizeof(T);
  }
  void span(const void* dev, uint64_t len) {
    if (!len) return;
    segs.push_back({pos, len, static_cast<const uint8_t*>(dev)});
    is_meta.push_back(0);
    pos += len;
  }
};

// ---- fused snapshot plan (replica mode 2) --------------------------------
// The allocation holding p (driver: cuMemGetAddressRange); false when the
// pointer is not device memory the driver knows.
bool alloc_range(const void* p, uint64_t* base, uint64_t* bytes) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    if (!fn) return false;
  }
  CUdeviceptr b = 0;
  size_t n = 0;
  if (fn(&b, &n, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
  *base = static_cast<uint64_t>(b);
  *bytes = static_cast<uint64_t>(n);
  return true;
}

struct FusedPlan {
  std::vector<std::pair<uint64_t, uint64_t>> src;  // source allocations (base, bytes); the patch map follows
  std::vector<FnvRun> runs;
  std::vector<int64_t> patch;  // chunks gathered whole into the patch buffer
};

// Record chunks as runs of whole chunks inside one payload span (loaded by
// TMA from the span's allocation, shifted by the span's misalignment
// against the record's rows) and single patch chunks (everything else: the
// headers, entry boundaries, the record's partial last chunk).  False when
// the record does not suit the fused kernel (too many allocations or mostly
// patch chunks): the caller packs instead.
bool plan_fused(const SegmentBuilder& b, uint64_t body, FusedPlan* fp) {
  const uint64_t cb = fnv_chunk_bytes(), n_chunks = fnv_chunks(body);
  const uint64_t win = cb + 128;  // the rows a shifted chunk lands
  size_t k = 0;
  for (uint64_t c = 0; c < n_chunks;) {
    const uint64_t lo = c * cb;
    while (k + 1 < b.segs.size() && b.segs[k].dst + b.segs[k].len <= lo) ++k;
    const pack::Segment& g = b.segs[k];
    // whole chunks of the span from c on (the last chunk of the record is partial: patch)
    uint64_t c_end = std::min((g.dst + g.len) / cb, body / cb);
    int map = -1;
    uint64_t off = 0;
    if (!b.is_meta[k] && g.dst <= lo && c_end > c) {
      const uint64_t src = reinterpret_cast<uint64_t>(g.src) + (lo - g.dst);
      for (size_t m = 0; m < fp->src.size() && map < 0; ++m)
        if (src >= fp->src[m].first && src < fp->src[m].first + fp->src[m].second) map = static_cast<int>(m);
      if (map < 0) {
        uint64_t base = 0, bytes = 0;
        if (alloc_range(g.src, &base, &bytes) && base % 16 == 0 && src >= base && src < base + bytes) {
          if (fp->src.size() + 1 >= static_cast<size_t>(kFnvMaxSrc)) return false;
          fp->src.emplace_back(base, bytes);
          map = static_cast<int>(fp->src.size()) - 1;
        }
      }
      if (map >= 0) {
        off = src - fp->src[map].first;
        // every chunk's window (512 rows + the overhang row) inside the allocation's rows
        const uint64_t rows_end = fp->src[map].second / 128 * 128;
        while (c_end > c && off + (c_end - 1 - c) * cb + win > rows_end) --c_end;
        if (c_end == c) map = -1;
      }
    }
    if (map >= 0) {
      fp->runs.push_back(FnvRun{static_cast<int64_t>(c), static_cast<int64_t>(c_end),
                                static_cast<int64_t>(off / 128), map, static_cast<int32_t>(off % 128)});
      c = c_end;
    } else {
      fp->patch.push_back(static_cast<int64_t>(c));
      ++c;
    }
  }
  const int patch_map = static_cast<int>(fp->src.size());
  // patch chunks as one-chunk runs of the patch map, merged in chunk order
  std::vector<FnvRun> all;
  all.reserve(fp->runs.size() + fp->patch.size());
  size_t r = 0;
  for (size_t j = 0; j < fp->patch.size(); ++j) {
    while (r < fp->runs.size() && fp->runs[r].c0 < fp->patch[j]) all.push_back(fp->runs[r++]);
    all.push_back(FnvRun{fp->patch[j], fp->patch[j] + 1, static_cast<int64_t>(j * (cb / 128)), patch_map, 0});
  }
  while (r < fp->runs.size()) all.push_back(fp->runs[r++]);
  fp->runs.swap(all);
  return fp->patch.size() * 4 <= n_chunks + 4 && fp->patch.size() <= 65535;  // (patch grid: y <= 65535)
}

// The transport of a record (mlck_ctx_set_replica_mode): auto (-1) is the
// fused kernel (2) when every replica is in this GPU's HBM, else the pack
// kernel with copy-engine pushes to the peers (1).
int resolve_mode(const mlck_ctx* ctx, const mlck_blob* out) {
  if (ctx->replica_mode != -1) return ctx->replica_mode;
  for (auto& r : out->replicas) {
    cudaPointerAttributes a{};
    if (ctx->is_ipc(r.first) || cudaPointerGetAttributes(&a, r.first) != cudaSuccess ||
        a.type != cudaMemoryTypeDevice || a.device != ctx->device) {
      cudaGetLastError();
      return 1;
    }
  }
  return 2;
}

// Uploads the segment table + meta, launches pack (and the FNV trailer when
// `trailer`): the blob body is [0, builder.pos), the trailer at pos.
cudaStream_t run_pack_impl(mlck_ctx* ctx, SegmentBuilder& b, mlck_blob* out, bool trailer);
void run_pack(mlck_ctx* ctx, SegmentBuilder& b, mlck_blob* out, bool trailer) {
  if (out->external) throw_invalid("a wrapped blob (mlck_blob_wrap) is read-only");
  const uint64_t wit_bytes = 4 * fnv_witness_words(b.pos);
  for (const auto& d : out->witness_dsts)
    if (trailer && ctx->witness && d.second < 4 * witness_alloc_words(b.pos))
      throw_invalid("replica witness capacity " + std::to_string(d.second) + " < " +
                    std::to_string(4 * witness_alloc_words(b.pos)) + " (mlck_witness_bytes)");
  // the blob's previous record may still be read by its asynchronous hash
  if (out->written) MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, out->written, 0));
  out->witness_n = ~0ull;
  const cudaStream_t last = run_pack_impl(ctx, b, out, trailer);
  if (out->witness_n == b.pos)  // the record's witness to every replica witness buffer (NVLink for peers)
    for (const auto& d : out->witness_dsts)
      MLCK_CUDA(cudaMemcpyAsync(d.first, out->witness, wit_bytes, cudaMemcpyDefault, last));
  if (!out->written) MLCK_CUDA(cudaEventCreateWithFlags(&out->written, cudaEventDisableTiming));
  MLCK_CUDA(cudaEventRecord(out->written, last));  // every path ends with the pushes joined
  out->written_replicas = static_cast<uint32_t>(out->replicas.size());
}
cudaStream_t run_pack_impl(mlck_ctx* ctx, SegmentBuilder& b, mlck_blob* out, bool trailer) {
  const uint64_t body = b.pos;
  const uint64_t total = body + (trailer ? 8 : 0);
  out->reserve(total);
  for (auto& r : out->replicas)
    if (r.second < total)
      throw_invalid("replica capacity " + std::to_string(r.second) + " < record size " +
                    std::to_string(total));
  out->size = total;
  const size_t seg_bytes = b.segs.size() * sizeof(pack::Segment);
  const size_t meta_off = align_up(seg_bytes, 16);
  // fused (mode 2, or auto with local copies): the FNV kernel loads the
  // chunks from their sources by TMA and stores them to the record and its
  // replicas -- no pack pass
  FusedPlan fp;
  // (TMA stores need 16-byte aligned destinations: the record is, a replica may not be)
  bool aligned = (reinterpret_cast<uintptr_t>(out->dev) & 15u) == 0;
  for (auto& r : out->replicas) aligned = aligned && (reinterpret_cast<uintptr_t>(r.first) & 15u) == 0;
  const bool fused = trailer && body >= 128 && aligned && resolve_mode(ctx, out) == 2 && plan_fused(b, body, &fp);
  const size_t runs_off = align_up(meta_off + b.meta.size(), 16);
  const size_t pl_off = runs_off + sizeof(FnvRun) * fp.runs.size();
  const size_t stage_bytes = fused ? pl_off + 8 * fp.patch.size() : meta_off + b.meta.size();
  auto& s = ctx->stage_for(stage_bytes);
  for (size_t i = 0; i < b.segs.size(); ++i)
    if (b.is_meta[i])
      b.segs[i].src = s.dev + meta_off + reinterpret_cast<uint64_t>(b.segs[i].src);
  std::memcpy(s.host, b.segs.data(), seg_bytes);
  std::memcpy(s.host + meta_off, b.meta.data(), b.meta.size());
  if (fused) {
    std::memcpy(s.host + runs_off, fp.runs.data(), sizeof(FnvRun) * fp.runs.size());
    std::memcpy(s.host + pl_off, fp.patch.data(), 8 * fp.patch.size());
  }
  ctx->stage_upload(s, stage_bytes);
  pack::Dsts d{};
  d.p[0] = out->dev;
  d.n = 1;
  for (auto& r : out->replicas) d.p[d.n++] = r.first;
  const auto* segs = reinterpret_cast<const pack::Segment*>(s.dev);
  const int n_segs = static_cast<int>(b.segs.size());
  if (fused) {
    uint8_t* patch = ctx->patch_for(fnv_chunk_bytes() * std::max<size_t>(fp.patch.size(), 1));
    launch_patch_chunks(segs, n_segs, reinterpret_cast<const int64_t*>(s.dev + pl_off), fp.patch.size(), body, patch,
                        ctx->stream);
    ctx->launches += fp.patch.empty() ? 0 : 1;
    FnvFused f{};
    f.runs = reinterpret_cast<const FnvRun*>(s.dev + runs_off);
    f.n_runs = static_cast<int>(fp.runs.size());
    f.n_src = static_cast<int>(fp.src.size()) + 1;
    for (size_t m = 0; m < fp.src.size(); ++m) {
      f.src[m] = reinterpret_cast<const uint8_t*>(fp.src[m].first);
      f.src_bytes[m] = fp.src[m].second;
    }
    f.src[fp.src.size()] = patch;
    f.src_bytes[fp.src.size()] = fnv_chunk_bytes() * std::max<size_t>(fp.patch.size(), 1);
    TrailerDsts t{};
    for (int r = 0; r < d.n; ++r) t.p[r] = d.p[r] + body;
    t.n = d.n;
    uint32_t* scratch = ctx->fnv_scratch_for(body);
    const int tf = ctx->tbegin("pack_fnv");
    uint32_t* wit = out->witness_for(body);
    launch_fnv(out->dev, body, kFnvOffset, scratch, ctx->next_epoch(), ctx->results, t, ctx->stream, nullptr,
               nullptr, &f, ctx->hash_reserve, &d, wit);
    if (wit) out->witness_n = body;
    ctx->tend(tf);
    ctx->launches += 1;
    return ctx->stream;
  }
  const int mode = resolve_mode(ctx, out);  // 2 fell through: the record did not suit the fused kernel
  if (trailer && mode == 5 && !out->replicas.empty() && body >= 128 && aligned) {
    // pack the local record; the FNV kernel stores the replicas from the
    // bytes it stages in shared memory (coalesced warp stores) and appends
    // the trailer to every copy -- no second read of the record
    pack::Dsts local{};
    local.p[0] = out->dev;
    local.n = 1;
    const int tp = ctx->tbegin("pack");
    launch_pack(segs, n_segs, body, local, ctx->stream);
    ctx->tend(tp);
    pack::Dsts reps{};
    for (auto& r : out->replicas) reps.p[reps.n++] = r.first;
    TrailerDsts t{};
    for (int r = 0; r < d.n; ++r) t.p[r] = d.p[r] + body;
    t.n = d.n;
    uint32_t* scratch = ctx->fnv_scratch_for(body);
    const int tf = ctx->tbegin("fnv");
    uint32_t* wit = out->witness_for(body);
    launch_fnv(out->dev, body, kFnvOffset, scratch, ctx->next_epoch(), ctx->results, t, ctx->stream, nullptr,
               nullptr, nullptr, ctx->hash_reserve, &reps, wit);
    if (wit) out->witness_n = body;
    ctx->tend(tf);
    ctx->launches += 2;
    return ctx->stream;
  }
  if (trailer && mode == 3 && !out->replicas.empty() && body) {
    // pack the local record; push it to the replicas with SM stores from
    // kPushSms reserved SMs while the FNV kernel hashes on the others; the
    // FNV kernel appends the trailer to every copy.
    pack::Dsts local{};
    local.p[0] = out->dev;
    local.n = 1;
    const int tp = ctx->tbegin("pack");
    launch_pack(segs, n_segs, body, local, ctx->stream);
    ctx->tend(tp);
    MLCK_CUDA(cudaEventRecord(ctx->ev_packed, ctx->stream));
    MLCK_CUDA(cudaStreamWaitEvent(ctx->side[0], ctx->ev_packed, 0));
    pack::Dsts peers{};
    for (auto& r : out->replicas) peers.p[peers.n++] = r.first;
    const int tq = ctx->tbegin("push", ctx->side[0]);
    launch_push(out->dev, body, peers, mlck_ctx::kPushSms, ctx->side[0]);
    ctx->tend(tq, ctx->side[0]);
    TrailerDsts t{};
    for (int r = 0; r < d.n; ++r) t.p[r] = d.p[r] + body;
    t.n = d.n;
    uint32_t* scratch = ctx->fnv_scratch_for(body);
    const int tf = ctx->tbegin("fnv");
    uint32_t* wit = out->witness_for(body);
    launch_fnv(out->dev, body, kFnvOffset, scratch, ctx->next_epoch(), ctx->results, t, ctx->stream, nullptr,
               nullptr, nullptr, std::max(mlck_ctx::kPushSms, ctx->hash_reserve), nullptr, wit);
    if (wit) out->witness_n = body;
    ctx->tend(tf);
    ctx->launches += 3;
    MLCK_CUDA(cudaEventRecord(ctx->ev_pushed[0], ctx->side[0]));
    MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_pushed[0], 0));  // record complete everywhere
    return ctx->stream;
  }
  if (trailer && (mode == 1 || mode == 4) && !out->replicas.empty() && body) {
    // pack the local record in pieces; the copy engines push each piece to
    // every replica (NVLink for peers) on the side stream as soon as it is
    // packed, beside the rest of the pack and the FNV kernel (mode 4,
    // ablation: the whole push after the hash); the 8-byte trailer follows
    // the hash.
    pack::Dsts local{};
    local.p[0] = out->dev;
    local.n = 1;
    // replica r streams on side[r]: each copy-engine queue sees one
    // destination's pieces in order (alternating destinations on one queue
    // cost 30 % at N=4 with 16 pieces)
    const int n_rep = static_cast<int>(out->replicas.size());
    cudaStream_t side = ctx->side[0];
    const int pieces = mode == 1 ? static_cast<int>(std::min<uint64_t>(mlck_ctx::kPieces, div_up(body, 64ull << 20))) : 1;
    const uint64_t piece = align_up(div_up(body, pieces), 64ull << 10);  // tile- and copy-engine friendly
    TrailerDsts t{};
    t.p[0] = out->dev + body;
    t.n = 1;
    uint32_t* scratch = ctx->fnv_scratch_for(body);
    auto hash = [&] {
      const int tf = ctx->tbegin("fnv");
      uint32_t* wit = out->witness_for(body);
      launch_fnv(out->dev, body, kFnvOffset, scratch, ctx->next_epoch(), ctx->results, t, ctx->stream, nullptr,
                 nullptr, nullptr, ctx->hash_reserve, nullptr, wit);
      if (wit) out->witness_n = body;
      ctx->tend(tf);
      MLCK_CUDA(cudaEventRecord(ctx->ev_hashed, ctx->stream));
    };
    const int tp = ctx->tbegin("pack");
    int tq = -1;
    for (int q = 0; q < pieces; ++q) {
      const uint64_t lo = std::min<uint64_t>(body, q * piece), hi = std::min<uint64_t>(body, lo + piece);
      if (hi <= lo) break;
      launch_pack(segs, n_segs, hi, local, ctx->stream, lo);
      ctx->launches += 1;
      if (mode == 1) {
        MLCK_CUDA(cudaEventRecord(ctx->ev_piece[q], ctx->stream));
        for (int r = 0; r < n_rep; ++r) {
          MLCK_CUDA(cudaStreamWaitEvent(ctx->side[r % mlck_ctx::kPushStreams], ctx->ev_piece[q], 0));
          if (q == 0 && r == 0) tq = ctx->tbegin("push", side);
          ce_copy(out->replicas[r].first + lo, out->dev + lo, hi - lo, cudaMemcpyDefault, ctx->side[r % mlck_ctx::kPushStreams]);
        }
      }
    }
    ctx->tend(tp);
    if (mode == 4) {
      hash();
      MLCK_CUDA(cudaStreamWaitEvent(side, ctx->ev_hashed, 0));
      tq = ctx->tbegin("push", side);
      for (int r = 0; r < n_rep; ++r) {
        if (r) MLCK_CUDA(cudaStreamWaitEvent(ctx->side[r % mlck_ctx::kPushStreams], ctx->ev_hashed, 0));
        ce_copy(out->replicas[r].first, out->dev, body, cudaMemcpyDefault, ctx->side[r % mlck_ctx::kPushStreams]);
      }
    }
    // the push timing covers every replica stream
    for (int r = 1; r < n_rep; ++r) {
      MLCK_CUDA(cudaEventRecord(ctx->ev_pushed[r % mlck_ctx::kPushStreams], ctx->side[r % mlck_ctx::kPushStreams]));
      MLCK_CUDA(cudaStreamWaitEvent(side, ctx->ev_pushed[r % mlck_ctx::kPushStreams], 0));
    }
    ctx->tend(tq, side);
    if (mode == 1) hash();
    ctx->launches += 1;
    for (int r = 0; r < n_rep; ++r) {
      MLCK_CUDA(cudaStreamWaitEvent(ctx->side[r % mlck_ctx::kPushStreams], ctx->ev_hashed, 0));
      MLCK_CUDA(cudaMemcpyAsync(out->replicas[r].first + body, out->dev + body, 8, cudaMemcpyDefault, ctx->side[r % mlck_ctx::kPushStreams]));
      MLCK_CUDA(cudaEventRecord(ctx->ev_pushed[r % mlck_ctx::kPushStreams], ctx->side[r % mlck_ctx::kPushStreams]));
      MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_pushed[r % mlck_ctx::kPushStreams], 0));  // record complete everywhere
    }
    return ctx->stream;
  }
  const int tp = ctx->tbegin("pack");
  launch_pack(segs, n_segs, body, d, ctx->stream);
  ctx->launches += body ? 1 : 0;
  ctx->tend(tp);
  if (!trailer) return ctx->stream;
  TrailerDsts t{};
  for (int r = 0; r < d.n; ++r) t.p[r] = d.p[r] + body;
  t.n = d.n;
  uint32_t* wit = out->witness_for(body);
  cudaStream_t hs = ctx->stream;
  uint32_t* scratch = nullptr;
  unsigned long long* res = ctx->results;
  if (ctx->hash_async) {  // the hash follows this pack on hstream; the ctx stream moves on
    MLCK_CUDA(cudaEventRecord(ctx->ev_packed_h, ctx->stream));
    MLCK_CUDA(cudaStreamWaitEvent(ctx->hstream, ctx->ev_packed_h, 0));
    hs = ctx->hstream;
    scratch = ctx->hscratch_for(body);
    res = ctx->hresult;
  } else {
    scratch = ctx->fnv_scratch_for(body);
  }
  const int tf = ctx->tbegin("fnv", hs);
  launch_fnv(out->dev, body, kFnvOffset, scratch, ctx->next_epoch(), res, t, hs, nullptr, nullptr, nullptr,
             ctx->hash_reserve, nullptr, wit);
  if (wit) out->witness_n = body;
  ctx->tend(tf, hs);
  ctx->launches += 1;
  if (ctx->hash_async) {
    MLCK_CUDA(cudaEventRecord(ctx->ev_hash_last, ctx->hstream));
    ctx->hash_pending = true;
  }
  return hs;
}

void build_state_image(const mlck_state* st, SegmentBuilder& b) {
  b.value<uint32_t>(0x4d4c5354u);  // "MLST"
  b.value<uint32_t>(1u);
  b.value<uint64_t>(st->iteration);
  b.value<uint64_t>(st->data_seed);
  b.value<uint32_t>(st->n_ops);
  for (uint32_t i = 0; i < st->n_ops; ++i) {
    const bool pr = st->present[i];
    b.value<uint64_t>(pr ? st->step[i] : 0);
    b.value<uint64_t>(pr ? st->P[i] : 0);
    if (pr) b.span(st->master(i), 12 * st->P[i]);
  }
}

struct SlotEntry {
  uint32_t id;
  uint8_t mode;
};

void build_record(const mlck_state* st, const std::vector<SlotEntry>& ents, uint8_t kind,
                  uint64_t iteration, uint64_t window_start, uint32_t wsparse, uint32_t slot,
                  uint64_t data_seed, SegmentBuilder& b) {
  // snapshot.hpp:120-141
  b.value<uint32_t>(kMagic);
  b.value<uint32_t>(1u);
  b.value<uint8_t>(kind);
  b.value<uint64_t>(iteration);
  b.value<uint64_t>(window_start);
  b.value<uint32_t>(wsparse);
  b.value<uint32_t>(slot);
  b.value<uint64_t>(data_seed);
  b.value<uint32_t>(static_cast<uint32_t>(ents.size()));
  for (const auto& e : ents) {
    const uint64_t P = st->P[e.id];
    b.value<uint32_t>(e.id);
    b.value<uint8_t>(e.mode);
    b.value<uint64_t>(P);
    if (e.mode == 0) {
      b.value<uint64_t>(st->step[e.id]);
      b.span(st->master(e.id), 12 * P);
    } else {
      b.span(st->codes(e.id), static_cast<uint64_t>(st->cb) * P);
    }
  }
}

std::vector<SlotEntry> slot_entries(const mlck_state* st, const uint32_t* active, uint32_t na,
                                    const uint32_t* co, uint32_t nc) {
  std::vector<SlotEntry> ents;
  ents.reserve(na + nc);
  for (uint32_t k = 0; k < na; ++k) {
    const uint32_t id = active[k];
    if (id >= st->n_ops)  // snapshot.hpp:212-216
      throw_invalid("snapshot slot references unknown operator " + std::to_string(id));
    if (!st->has_full[id])  // snapshot.hpp:220-222
      throw_runtime("snapshot: operator " + std::to_string(id) + " in active set has no full state");
    ents.push_back({id, 0});
  }
  for (uint32_t k = 0; k < nc; ++k) {
    const uint32_t id = co[k];
    if (id >= st->n_ops)
      throw_invalid("snapshot slot references unknown operator " + std::to_string(id));
    ents.push_back({id, 1});
  }
  std::stable_sort(ents.begin(), ents.end(),
                   [](const SlotEntry& a, const SlotEntry& b) { return a.id < b.id; });
  return ents;
}

adam::Opt to_opt(const mlck_optimizer* o) {
  adam::Opt r;
  r.kind = o ? o->kind : 0;
  r.lr = o ? o->lr : 1e-3f;
  r.b1 = o ? o->beta1 : 0.9f;
  r.b2 = o ? o->beta2 : 0.999f;
  r.eps = o ? o->eps : 1e-8f;
  r.omb1 = 1.0f - r.b1;
  r.omb2 = 1.0f - r.b2;
  return r;
}

// host libm, exactly the reference's std::pow(float, float) (engine.hpp:716-717)
float bias_correction(float beta, uint64_t step) {
  return 1.0f - std::pow(beta, static_cast<float>(step));
}

// Parsed view of a device record (parse_record): checksum, header, entries.
struct Parsed {
  WalkResult hdr;
  std::vector<WalkEntry> entries;
};

std::string walk_error(const WalkResult& r) {
  switch (r.status) {
    case kWalkTruncated: return "container truncated";
    case kWalkMagic: return "container: bad magic";
    case kWalkVersion: return "container: unsupported version " + std::to_string(r.version);
    case kWalkWidth: return "container: unsupported compute width";
    default: return "container: parse error";
  }
}

// parse_record over n device records in three phases, so the caller can
// overlap its own work with the checksum pass:
//   verify_begin: one FNV launch per record (trailer check, snapshot.hpp:
//     156-163), alternating between the ctx stream and vside; nothing waits;
//   walk: the header / entry walk of every record of >= 8 bytes (bounds
//     checked, so a corrupt record walks harmlessly) on the ctx stream, which
//     is synchronized -- entry tables sized from the records' own op counts;
//   verify_end: the ctx stream joins vside; errors[k] in the reference's
//     order: "container truncated" (< 8 bytes), "container checksum
//     mismatch", then the walk's magic / version / truncation error.
struct ParseJob {
  int witness_ctas = 0;  // 0 = one per SM
  mlck_ctx* ctx = nullptr;
  mlck_blob* const* blobs = nullptr;
  uint32_t n = 0;
  int cb = 2;
  std::vector<Parsed> out;
  std::vector<std::string> walk_err;
};

// the records' asynchronous hashes (trailer, witness) have landed
void wait_written(mlck_ctx* ctx, mlck_blob* const* blobs, uint32_t n) {
  for (uint32_t k = 0; k < n; ++k)
    if (blobs[k]->written) MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, blobs[k]->written, 0));
}

void verify_begin(ParseJob& j) {
  mlck_ctx* ctx = j.ctx;
  const uint32_t n = j.n;
  wait_written(ctx, j.blobs, n);
  ctx->results_for(3 * static_cast<size_t>(n));
  MLCK_CUDA(cudaMemsetAsync(ctx->results + 2 * static_cast<size_t>(n), 0, 8 * static_cast<size_t>(n), ctx->stream));
  MLCK_CUDA(cudaEventRecord(ctx->ev_vmain, ctx->stream));  // the records are complete
  for (int i = 0; i < 2; ++i) MLCK_CUDA(cudaStreamWaitEvent(ctx->vside[i], ctx->ev_vmain, 0));
  uint32_t launched = 0;
  for (uint32_t k = 0; k < n; ++k) {
    const mlck_blob* b = j.blobs[k];
    if (b->size < 8) continue;
    const int side = static_cast<int>(launched++ & 1u);  // (one side stream: 0.1 ms slower)
    cudaStream_t st = ctx->vside[side];
    uint32_t* scratch = ctx->vscratch_for(side, b->size - 8);
    TrailerDsts none{};
    if (ctx->witness && b->has_witness()) {  // exact re-hash against the record's witness (fnv.cuh)
      const int tf = ctx->tbegin("fnv_witness", st);
      launch_fnv_witness(b->dev, b->size - 8, kFnvOffset, b->witness, scratch, ctx->results + k,
                         ctx->results + 2 * static_cast<size_t>(n) + k, st, j.witness_ctas);
      ctx->tend(tf, st);
      ctx->witness_used += 1;
    } else {
      const int tf = ctx->tbegin("fnv_verify", st);
      launch_fnv(b->dev, b->size - 8, kFnvOffset, scratch, ctx->next_epoch(), ctx->results + k, none, st,
                 nullptr, nullptr, nullptr, ctx->hash_reserve);
      ctx->tend(tf, st);
    }
    ctx->launches += 1;
    MLCK_CUDA(cudaMemcpyAsync(ctx->results + n + k, b->dev + b->size - 8, 8, cudaMemcpyDeviceToDevice, st));
  }
  for (int i = 0; i < 2; ++i) MLCK_CUDA(cudaEventRecord(ctx->ev_vside[i], ctx->vside[i]));
}

void walk_records(ParseJob& j) {
  mlck_ctx* ctx = j.ctx;
  wait_written(ctx, j.blobs, j.n);
  j.out.assign(j.n, Parsed{});
  j.walk_err.assign(j.n, std::string());
  std::vector<uint32_t> idx;
  for (uint32_t k = 0; k < j.n; ++k)
    if (j.blobs[k]->size >= 8) idx.push_back(k);
  std::vector<uint32_t> cap(j.n, 1024);
  // pass 1 with 1024 entries per record; records with more run again with
  // their own op count (the walk validates every entry either way)
  for (int pass = 0; pass < 2 && !idx.empty(); ++pass) {
    const size_t nj = idx.size();
    const size_t res_bytes = align_up(nj * sizeof(WalkResult), 256);
    std::vector<size_t> ent_off(nj + 1, 0);
    for (size_t q = 0; q < nj; ++q) ent_off[q + 1] = ent_off[q] + align_up(cap[idx[q]] * sizeof(WalkEntry), 256);
    uint8_t* dscratch = nullptr;
    MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dscratch), res_bytes + ent_off[nj], ctx->stream));
    std::vector<WalkJob> jobs(nj);
    for (size_t q = 0; q < nj; ++q) {
      const mlck_blob* b = j.blobs[idx[q]];
      jobs[q] = WalkJob{b->dev, b->size, j.cb, cap[idx[q]], reinterpret_cast<WalkEntry*>(dscratch + res_bytes + ent_off[q]),
                        reinterpret_cast<WalkResult*>(dscratch) + q};
    }
    auto& stg = ctx->stage_for(nj * sizeof(WalkJob));
    std::memcpy(stg.host, jobs.data(), nj * sizeof(WalkJob));
    ctx->stage_upload(stg, nj * sizeof(WalkJob));
    const int tw = ctx->tbegin("walk");
    launch_walk(reinterpret_cast<const WalkJob*>(stg.dev), static_cast<int>(nj), ctx->stream);
    ctx->tend(tw);
    ctx->launches += 1;
    std::vector<WalkResult> res(nj);
    MLCK_CUDA(cudaMemcpyAsync(res.data(), dscratch, nj * sizeof(WalkResult), cudaMemcpyDeviceToHost, ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<uint32_t> again;
    for (size_t q = 0; q < nj; ++q) {
      const uint32_t k = idx[q];
      j.out[k].hdr = res[q];
      if (res[q].status != kWalkOk) {
        j.walk_err[k] = walk_error(res[q]);
        continue;
      }
      if (res[q].n_entries > cap[k]) {
        cap[k] = res[q].n_entries;
        again.push_back(k);
        continue;
      }
      j.out[k].entries.resize(res[q].n_entries);
      MLCK_CUDA(cudaMemcpyAsync(j.out[k].entries.data(), dscratch + res_bytes + ent_off[q],
                                res[q].n_entries * sizeof(WalkEntry), cudaMemcpyDeviceToHost, ctx->stream));
    }
    MLCK_CUDA(cudaFreeAsync(dscratch, ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    idx.swap(again);
  }
}

std::vector<std::string> verify_end(ParseJob& j) {
  mlck_ctx* ctx = j.ctx;
  const uint32_t n = j.n;
  for (int i = 0; i < 2; ++i) MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_vside[i], 0));
  MLCK_CUDA(cudaMemcpyAsync(ctx->host_results, ctx->results, 3 * static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
  MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->check_watchdog();
  // a witness that does not match its record's bytes: hash the record from
  // scratch (the witness path computed nothing usable)
  std::vector<uint32_t> redo;
  for (uint32_t k = 0; k < n; ++k)
    if (ctx->host_results[2 * static_cast<size_t>(n) + k]) redo.push_back(k);
  if (!redo.empty()) {
    std::vector<unsigned long long> full(n, 0);
    for (uint32_t k : redo) {
      const mlck_blob* b = j.blobs[k];
      TrailerDsts none{};
      uint32_t* scratch = ctx->fnv_scratch_for(b->size - 8);
      const int tf = ctx->tbegin("fnv_verify");
      launch_fnv(b->dev, b->size - 8, kFnvOffset, scratch, ctx->next_epoch(), ctx->results + k, none, ctx->stream,
                 nullptr, nullptr, nullptr, ctx->hash_reserve);
      ctx->tend(tf);
      ctx->launches += 1;
      ctx->witness_fallbacks += 1;
    }
    MLCK_CUDA(cudaMemcpyAsync(ctx->host_results, ctx->results, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost,
                              ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->check_watchdog();
  }
  std::vector<std::string> errors(n);
  for (uint32_t k = 0; k < n; ++k) {
    if (j.blobs[k]->size < 8)
      errors[k] = "container truncated";
    else if (ctx->host_results[k] != ctx->host_results[n + k])  // snapshot.hpp:158-163
      errors[k] = "container checksum mismatch";
    else
      errors[k] = j.walk_err[k];
    if (!errors[k].empty()) j.out[k].entries.clear();
  }
  return errors;
}

// All three phases: verified and walked records; errors[k] empty when blob k parsed.
std::vector<Parsed> parse_blobs(mlck_ctx* ctx, mlck_blob* const* blobs, uint32_t n, int cb,
                                std::vector<std::string>& errors) {
  ParseJob j;
  j.ctx = ctx;
  j.blobs = blobs;
  j.n = n;
  j.cb = cb;
  errors.assign(n, std::string());
  if (n == 0) return {};
  verify_begin(j);
  walk_records(j);
  errors = verify_end(j);
  return std::move(j.out);
}

}  // namespace

extern "C" {

const char* mlck_last_error(void) { return last_error().c_str(); }

// internal: used by log.cu
int mlck_ctx_device_stream_(mlck_ctx* c, int* device, void** stream) {
  *device = c->device;
  *stream = c->stream;
  return 0;
}

int mlck_ctx_create(int device, mlck_ctx** out) {
  return api([&] {
    auto* c = new mlck_ctx();
    c->device = device;
    c->activate();
    // highest priority: the hash kernel's CTAs must all become resident
    // (slot-major look-back), so they go ahead of other work queued on the GPU
    int least = 0, greatest = 0;
    MLCK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    MLCK_CUDA(cudaStreamCreateWithPriority(&c->own, cudaStreamNonBlocking, greatest));
    c->stream = c->own;
    for (auto& s : c->stage) MLCK_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    for (auto& sd : c->side) MLCK_CUDA(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      MLCK_CUDA(cudaStreamCreateWithPriority(&c->vside[i], cudaStreamNonBlocking, greatest));
      MLCK_CUDA(cudaEventCreateWithFlags(&c->ev_vside[i], cudaEventDisableTiming));
    }
    MLCK_CUDA(cudaEventCreateWithFlags(&c->ev_vmain, cudaEventDisableTiming));
    MLCK_CUDA(cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking));
    MLCK_CUDA(cudaEventCreateWithFlags(&c->ev_packed_h, cudaEventDisableTiming));
    MLCK_CUDA(cudaEventCreateWithFlags(&c->ev_hash_last, cudaEventDisableTiming));
    MLCK_CUDA(cudaMalloc(&c->hresult, 64));
    for (cudaEvent_t* e : {&c->ev_packed, &c->ev_hashed})
      MLCK_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (auto& e : c->ev_pushed) MLCK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->ev_piece) MLCK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->ev) MLCK_CUDA(cudaEventCreate(&e));
    c->results_for(64);
    // stream-ordered scratch (parse tables, staging) stays in the pool across
    // synchronizations instead of being returned to the OS every call
    cudaMemPool_t pool;
    MLCK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    MLCK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    init_constants();
    *out = c;
  });
}

int mlck_ctx_destroy(mlck_ctx* c) {
  return api([&] {
    if (!c) return;
    c->activate();
    cudaStreamSynchronize(c->stream);
    for (auto& s : c->stage) {
      if (s.host) cudaFreeHost(s.host);
      if (s.dev) cudaFree(s.dev);
      cudaEventDestroy(s.done);
    }
    for (auto& sd : c->side) {
      cudaStreamSynchronize(sd);
      cudaStreamDestroy(sd);
    }
    for (auto& e : c->ev) cudaEventDestroy(e);
    for (auto& e : c->ev_pushed) cudaEventDestroy(e);
    for (auto& e : c->ev_piece) cudaEventDestroy(e);
    cudaEventDestroy(c->ev_packed);
    cudaEventDestroy(c->ev_hashed);
    for (int i = 0; i < 2; ++i) {
      cudaStreamSynchronize(c->vside[i]);
      cudaStreamDestroy(c->vside[i]);
      cudaEventDestroy(c->ev_vside[i]);
      if (c->vscratch[i]) cudaFree(c->vscratch[i]);
    }
    cudaEventDestroy(c->ev_vmain);
    cudaStreamSynchronize(c->hstream);
    cudaStreamDestroy(c->hstream);
    cudaEventDestroy(c->ev_packed_h);
    cudaEventDestroy(c->ev_hash_last);
    if (c->hscratch) cudaFree(c->hscratch);
    cudaFree(c->hresult);
    if (c->fnv_scratch) cudaFree(c->fnv_scratch);
    if (c->patch) cudaFree(c->patch);
    cudaFree(c->results);
    cudaFreeHost(c->host_results);
    cudaStreamDestroy(c->own);
    delete c;
  });
}

int mlck_ctx_set_stream(mlck_ctx* c, void* stream) {
  return api([&] {
    c->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(c->stream));
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
  });
}
int mlck_ctx_synchronize(mlck_ctx* c) {
  return api([&] {
    c->activate();
    c->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(c->stream));
    c->check_watchdog();
  });
}
uint64_t mlck_ctx_kernel_launches(mlck_ctx* c) { return c ? c->launches : 0; }


int mlck_ctx_set_replica_mode(mlck_ctx* c, int mode) {
  return api([&] {
    if (mode < -1 || mode > 5)
      throw_invalid("replica mode must be -1 (auto), 0 (pack-kernel stores), 1 (copy engines), "
                    "2 (fused pack+hash+push), 3 (SM push beside the hash), 4 (copy engines "
                    "after the hash) or 5 (hash-kernel stores)");
    c->replica_mode = mode;
  });
}

int mlck_ctx_set_witness(mlck_ctx* c, int on) {
  return api([&] { c->witness = on != 0; });
}
int mlck_ctx_witness_stats(mlck_ctx* c, uint64_t* used, uint64_t* fallbacks) {
  return api([&] {
    if (used) *used = c->witness_used;
    if (fallbacks) *fallbacks = c->witness_fallbacks;
  });
}

int mlck_ctx_set_convert_overlap(mlck_ctx* c, int witness_sms) {
  return api([&] {
    if (witness_sms < 0) throw_invalid("convert overlap: SM count must be >= 0");
    c->convert_overlap = witness_sms;
  });
}

int mlck_ctx_set_hash_async(mlck_ctx* c, int on) {
  return api([&] {
    c->join_hash();
    c->hash_async = on != 0;
  });
}

int mlck_ctx_set_hash_reserve(mlck_ctx* c, int sms) {
  return api([&] {
    if (sms < 0) throw_invalid("hash reserve must be >= 0 SMs");
    c->hash_reserve = sms;
  });
}

int mlck_ctx_set_timing(mlck_ctx* c, int on) {
  return api([&] {
    c->timing = on != 0;
    c->timed.clear();
    c->ev_used = 0;
  });
}

int mlck_ctx_timings(mlck_ctx* c, char* labels, uint64_t labels_cap, float* ms, uint32_t cap,
                     uint32_t* n) {
  return api([&] {
    c->activate();
    c->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(c->stream));
    std::string csv;
    const uint32_t cnt = static_cast<uint32_t>(c->timed.size());
    for (uint32_t i = 0; i < cnt; ++i) {
      if (i < cap) MLCK_CUDA(cudaEventElapsedTime(ms + i, c->timed[i].a, c->timed[i].b));
      if (i) csv += ",";
      csv += c->timed[i].label;
    }
    if (labels && labels_cap) std::snprintf(labels, labels_cap, "%s", csv.c_str());
    if (n) *n = cnt;
    c->timed.clear();
    c->ev_used = 0;
  });
}

// ------------------------------------------------------------------ state
int mlck_state_create(mlck_ctx* ctx, uint32_t n_ops, const uint64_t* pc, int cb, mlck_state** out) {
  return api([&] {
    if (cb != 1 && cb != 2 && cb != 4)  // tensor.hpp:107-109
      throw_invalid("quantize: unsupported width " + std::to_string(cb));
    ctx->activate();
    auto* st = new mlck_state();
    st->ctx = ctx;
    st->n_ops = n_ops;
    st->cb = cb;
    st->P.assign(pc, pc + n_ops);
    st->step.assign(n_ops, 0);
    st->has_full.assign(n_ops, 1);
    st->present.assign(n_ops, 1);
    uint64_t off = 0;
    for (uint32_t i = 0; i < n_ops; ++i) {
      st->full_off.push_back(off);
      off += align_up(12 * st->P[i] + 16, kAlign);
    }
    for (uint32_t i = 0; i < n_ops; ++i) {
      st->code_off.push_back(off);
      off += align_up(static_cast<uint64_t>(cb) * st->P[i] + 16, kAlign);
    }
    st->arena_bytes = std::max<uint64_t>(off, kAlign);
    dev_malloc(reinterpret_cast<void**>(&st->arena), st->arena_bytes);
    MLCK_CUDA(cudaMemsetAsync(st->arena, 0, st->arena_bytes, ctx->stream));
    *out = st;
  });
}

int mlck_state_destroy(mlck_state* st) {
  return api([&] {
    if (!st) return;
    st->ctx->activate();
    cudaStreamSynchronize(st->ctx->stream);
    cudaFree(st->arena);
    delete st;
  });
}

int mlck_state_set_meta(mlck_state* st, uint64_t it, uint64_t seed) {
  return api([&] {
    st->iteration = it;
    st->data_seed = seed;
  });
}
int mlck_state_get_meta(mlck_state* st, uint64_t* it, uint64_t* seed) {
  return api([&] {
    if (it) *it = st->iteration;
    if (seed) *seed = st->data_seed;
  });
}

int mlck_state_upload_op(mlck_state* st, uint32_t id, const float* master, const float* m,
                         const float* v, uint64_t step, int has_full) {
  return api([&] {
    st->check_id(id);
    st->ctx->activate();
    const uint64_t P = st->P[id];
    float* d = st->master(id);
    cudaStream_t s = st->ctx->stream;
    if (P) {
      MLCK_CUDA(cudaMemcpyAsync(d, master, 4 * P, cudaMemcpyHostToDevice, s));
      MLCK_CUDA(cudaMemcpyAsync(d + P, m, 4 * P, cudaMemcpyHostToDevice, s));
      MLCK_CUDA(cudaMemcpyAsync(d + 2 * P, v, 4 * P, cudaMemcpyHostToDevice, s));
      launch_encode(d, st->codes(id), P, st->cb, s);  // refresh_compute
      st->ctx->launches += 1;
    }
    MLCK_CUDA(cudaStreamSynchronize(s));  // host arrays are caller-owned
    st->step[id] = step;
    st->has_full[id] = has_full ? 1 : 0;
    st->present[id] = 1;
  });
}

int mlck_state_download_op(mlck_state* st, uint32_t id, float* master, float* m, float* v,
                           uint64_t* step, float* compute, int* has_full) {
  return api([&] {
    st->check_id(id);
    st->ctx->activate();
    const uint64_t P = st->P[id];
    float* d = st->master(id);
    cudaStream_t s = st->ctx->stream;
    if (P) {
      if (master) MLCK_CUDA(cudaMemcpyAsync(master, d, 4 * P, cudaMemcpyDeviceToHost, s));
      if (m) MLCK_CUDA(cudaMemcpyAsync(m, d + P, 4 * P, cudaMemcpyDeviceToHost, s));
      if (v) MLCK_CUDA(cudaMemcpyAsync(v, d + 2 * P, 4 * P, cudaMemcpyDeviceToHost, s));
      if (compute) {
        float* tmp = nullptr;
        MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), 4 * P, s));
        launch_decode(st->codes(id), tmp, P, st->cb, s);
        st->ctx->launches += 1;
        MLCK_CUDA(cudaMemcpyAsync(compute, tmp, 4 * P, cudaMemcpyDeviceToHost, s));
        MLCK_CUDA(cudaFreeAsync(tmp, s));
      }
    }
    MLCK_CUDA(cudaStreamSynchronize(s));
    if (step) *step = st->step[id];
    if (has_full) *has_full = st->has_full[id];
  });
}

int mlck_state_set_step(mlck_state* st, uint32_t id, uint64_t step, int has_full) {
  return api([&] {
    st->check_id(id);
    st->step[id] = step;
    st->has_full[id] = has_full ? 1 : 0;
  });
}

int mlck_state_op_ptrs(mlck_state* st, uint32_t id, float** master, float** m, float** v,
                       void** compute) {
  return api([&] {
    st->check_id(id);
    float* d = st->master(id);
    if (master) *master = d;
    if (m) *m = d + st->P[id];
    if (v) *v = d + 2 * st->P[id];
    if (compute) *compute = st->codes(id);
  });
}

int mlck_state_fill_synthetic(mlck_state* st, uint64_t seed, uint64_t step) {
  return api([&] {
    st->ctx->activate();
    cudaStream_t s = st->ctx->stream;
    for (uint32_t i = 0; i < st->n_ops; ++i) {
      const uint64_t P = st->P[i];
      float* d = st->master(i);
      launch_synth(d, P, seed, 3ull * i + 0, -0.25f, 0.25f, s);
      launch_synth(d + P, P, seed, 3ull * i + 1, -1e-3f, 1e-3f, s);
      launch_synth(d + 2 * P, P, seed, 3ull * i + 2, 0.0f, 1e-6f, s);
      launch_encode(d, st->codes(i), P, st->cb, s);
      st->ctx->launches += P ? 4 : 0;
      st->step[i] = step;
      st->has_full[i] = 1;
      st->present[i] = 1;
    }
  });
}

int mlck_state_serialize_blob(mlck_state* st, mlck_blob* out) {
  return api([&] {
    st->ctx->activate();
    SegmentBuilder b;
    build_state_image(st, b);
    run_pack(st->ctx, b, out, /*trailer=*/false);
  });
}

int mlck_state_serialize(mlck_state* st, uint8_t* host_out, uint64_t cap, uint64_t* size) {
  return api([&] {
    const uint64_t n = state_mlst_size(st);
    if (size) *size = n;
    if (!host_out) return;
    if (cap < n) throw_invalid("serialize_state: buffer too small");
    st->ctx->activate();
    mlck_blob tmp;
    tmp.ctx = st->ctx;
    SegmentBuilder b;
    build_state_image(st, b);
    run_pack(st->ctx, b, &tmp, false);
    ce_copy(host_out, tmp.dev, n, cudaMemcpyDeviceToHost, st->ctx->stream);
    MLCK_CUDA(cudaStreamSynchronize(st->ctx->stream));
    MLCK_CUDA(cudaFree(tmp.dev));
  });
}

// ------------------------------------------------------------------ blobs
int mlck_blob_create(mlck_ctx* ctx, uint64_t capacity, mlck_blob** out) {
  return api([&] {
    ctx->activate();
    auto* b = new mlck_blob();
    b->ctx = ctx;
    b->reserve(std::max<uint64_t>(capacity, kAlign));
    ctx->blobs.push_back(b);
    *out = b;
  });
}
int mlck_blob_destroy(mlck_blob* b) {
  return api([&] {
    if (!b) return;
    b->ctx->activate();
    if (b->written) cudaEventSynchronize(b->written);
    cudaStreamSynchronize(b->ctx->stream);
    if (b->dev && !b->external) cudaFree(b->dev);
    if (b->witness && !b->external_witness) cudaFree(b->witness);
    if (b->written) cudaEventDestroy(b->written);
    auto& v = b->ctx->blobs;
    v.erase(std::remove(v.begin(), v.end(), b), v.end());
    delete b;
  });
}
int mlck_blob_from_host(mlck_ctx* ctx, const uint8_t* bytes, uint64_t n, mlck_blob** out) {
  return api([&] {
    ctx->activate();
    auto* b = new mlck_blob();
    b->ctx = ctx;
    b->reserve(std::max<uint64_t>(n, kAlign));
    if (n) MLCK_CUDA(cudaMemcpyAsync(b->dev, bytes, n, cudaMemcpyHostToDevice, ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    b->size = n;
    ctx->blobs.push_back(b);
    *out = b;
  });
}
uint64_t mlck_blob_size(const mlck_blob* b) { return b ? b->size : 0; }
void* mlck_blob_device_ptr(const mlck_blob* b) { return b ? b->dev : nullptr; }
void* mlck_blob_witness_ptr(const mlck_blob* b) { return b && b->has_witness() ? b->witness : nullptr; }
int mlck_blob_to_host(const mlck_blob* b, uint8_t* host, uint64_t cap) {
  return api([&] {
    if (cap < b->size) throw_invalid("blob_to_host: buffer too small");
    b->ctx->activate();
    if (b->written) MLCK_CUDA(cudaStreamWaitEvent(b->ctx->stream, b->written, 0));
    if (b->size)
      ce_copy(host, b->dev, b->size, cudaMemcpyDeviceToHost, b->ctx->stream);
    MLCK_CUDA(cudaStreamSynchronize(b->ctx->stream));
    b->ctx->check_watchdog();
  });
}
int mlck_blob_add_replica(mlck_blob* b, void* ptr, uint64_t capacity) {
  return api([&] {
    if (b->replicas.size() + 1 >= static_cast<size_t>(pack::kMaxDst))
      throw_invalid("at most " + std::to_string(pack::kMaxDst - 1) + " replicas per blob");
    if (reinterpret_cast<uintptr_t>(ptr) % 16)
      throw_invalid("replica buffers must be 16-byte aligned");
    // a replica inside a peer's IPC mapping must fit in it: the pack kernel and
    // the copy engines would otherwise write past the peer's allocation
    const uint64_t a = reinterpret_cast<uint64_t>(ptr);
    bool ipc = false;
    for (const auto& r : b->ctx->ipc_ranges)
      if (a >= r.first && a < r.first + r.second) {
        ipc = true;
        if (capacity > r.first + r.second - a)
          throw_invalid("replica capacity " + std::to_string(capacity) + " exceeds its IPC mapping (" +
                        std::to_string(r.first + r.second - a) + " bytes from the replica pointer)");
      }
    // any other device pointer (local, peer access): against its allocation
    uint64_t base = 0, bytes = 0;
    if (!ipc && alloc_range(ptr, &base, &bytes) && capacity > base + bytes - a)
      throw_invalid("replica capacity " + std::to_string(capacity) + " exceeds its allocation (" +
                    std::to_string(base + bytes - a) + " bytes from the replica pointer)");
    b->replicas.push_back({static_cast<uint8_t*>(ptr), capacity});
  });
}
int mlck_blob_clear_replicas(mlck_blob* b) {
  return api([&] {
    b->replicas.clear();
    b->witness_dsts.clear();
  });
}
int mlck_blob_add_replica_witness(mlck_blob* b, void* ptr, uint64_t capacity) {
  return api([&] {
    if (b->witness_dsts.size() + 1 >= static_cast<size_t>(pack::kMaxDst))
      throw_invalid("at most " + std::to_string(pack::kMaxDst - 1) + " replica witnesses per blob");
    if (reinterpret_cast<uintptr_t>(ptr) % 16) throw_invalid("replica witness buffers must be 16-byte aligned");
    uint64_t base = 0, bytes = 0;
    const uint64_t a = reinterpret_cast<uint64_t>(ptr);
    if (alloc_range(ptr, &base, &bytes) && capacity > base + bytes - a)
      throw_invalid("replica witness capacity " + std::to_string(capacity) + " exceeds its allocation (" +
                    std::to_string(base + bytes - a) + " bytes from the pointer)");
    b->witness_dsts.push_back({static_cast<uint8_t*>(ptr), capacity});
  });
}
uint64_t mlck_witness_bytes(uint64_t record_bytes) {
  return 4 * witness_alloc_words(record_bytes >= 8 ? record_bytes - 8 : 0);
}
int mlck_blob_wrap(mlck_ctx* ctx, void* record, uint64_t n, const void* witness, mlck_blob** out) {
  return api([&] {
    ctx->activate();
    if (!record && n) throw_invalid("blob wrap: null record");
    // the record and the witness (with the verifier's whole-chunk over-read)
    // must lie inside the allocations they point into
    uint64_t base = 0, bytes = 0;
    const uint64_t r = reinterpret_cast<uint64_t>(record), w = reinterpret_cast<uint64_t>(witness);
    if (n && alloc_range(record, &base, &bytes) && r + n > base + bytes)
      throw_invalid("blob wrap: " + std::to_string(n) + " record bytes run past their allocation (" +
                    std::to_string(base + bytes - r) + " bytes from the record pointer)");
    const uint64_t wneed = n >= 8 ? 4 * witness_alloc_words(n - 8) : 0;
    if (witness && n >= 8 && alloc_range(witness, &base, &bytes) && w + wneed > base + bytes)
      throw_invalid("blob wrap: witness buffer of " + std::to_string(base + bytes - w) + " bytes < " +
                    std::to_string(wneed) + " (mlck_witness_bytes)");
    auto* b = new mlck_blob();
    b->ctx = ctx;
    b->external = true;
    b->dev = static_cast<uint8_t*>(record);
    b->cap = b->size = n;
    if (witness && n >= 8) {
      b->external_witness = true;
      b->witness = static_cast<uint32_t*>(const_cast<void*>(witness));
      b->witness_cap = witness_alloc_words(n - 8);
      b->witness_n = n - 8;
    }
    ctx->blobs.push_back(b);
    *out = b;
  });
}

// ---- window lifecycle and durability ----------------------
int mlck_blob_replication(mlck_blob* b, uint32_t* done) {
  return api([&] {
    *done = 0;
    if (!b->written) return;
    const cudaError_t e = cudaEventQuery(b->written);
    if (e == cudaErrorNotReady) return;
    MLCK_CUDA(e);
    // a record whose hash the look-back watchdog cut short carries a poisoned
    // trailer: it is not a replica of anything (the error, not a count)
    b->ctx->activate();
    b->ctx->check_watchdog();
    *done = b->written_replicas;
  });
}

namespace {
// Double-buffered pinned staging for file I/O: the copy of one piece
// overlaps the file operation on the other.
constexpr uint64_t kIoPiece = 64ull << 20;
struct IoStage {
  uint8_t* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  IoStage() {
    for (int i = 0; i < 2; ++i) {
      MLCK_CUDA(cudaMallocHost(&buf[i], kIoPiece));
      MLCK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~IoStage() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};
struct File {
  std::FILE* f;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};
}  // namespace

int mlck_blob_save(mlck_blob* b, const char* path, uint64_t* written) {
  return api([&] {
    b->ctx->activate();
    if (b->written) MLCK_CUDA(cudaStreamWaitEvent(b->ctx->stream, b->written, 0));
    File file(path, "wb");
    if (!file.f) throw_runtime(std::string("persist: cannot open ") + path);
    IoStage io;
    const uint64_t n = b->size, pieces = div_up(n, kIoPiece);
    cudaStream_t s = b->ctx->stream;
    auto piece_len = [&](uint64_t i) { return std::min(kIoPiece, n - i * kIoPiece); };
    for (uint64_t i = 0; i <= pieces; ++i) {
      if (i < pieces) {  // D2H of piece i into buffer i % 2
        MLCK_CUDA(cudaMemcpyAsync(io.buf[i & 1], b->dev + i * kIoPiece, piece_len(i), cudaMemcpyDeviceToHost, s));
        MLCK_CUDA(cudaEventRecord(io.ev[i & 1], s));
      }
      if (i >= 1) {  // write piece i - 1 while piece i is in flight
        const uint64_t j = i - 1;
        MLCK_CUDA(cudaEventSynchronize(io.ev[j & 1]));
        if (std::fwrite(io.buf[j & 1], 1, piece_len(j), file.f) != piece_len(j))
          throw_runtime(std::string("persist: short write to ") + path);
      }
    }
    if (std::fflush(file.f) != 0 || fsync(fileno(file.f)) != 0)
      throw_runtime(std::string("persist: cannot flush ") + path);
    if (written) *written = n;
  });
}

int mlck_blob_load(mlck_ctx* ctx, const char* path, mlck_blob** out) {
  return api([&] {
    ctx->activate();
    File file(path, "rb");
    if (!file.f) throw_runtime(std::string("persist: cannot open ") + path);
    if (std::fseek(file.f, 0, SEEK_END) != 0) throw_runtime(std::string("persist: cannot seek ") + path);
    const long len = std::ftell(file.f);
    if (len < 0) throw_runtime(std::string("persist: cannot size ") + path);
    std::rewind(file.f);
    const uint64_t n = static_cast<uint64_t>(len), pieces = div_up(n, kIoPiece);
    auto* b = new mlck_blob();
    b->ctx = ctx;
    try {
      b->reserve(std::max<uint64_t>(n, kAlign));
      IoStage io;
      cudaStream_t s = ctx->stream;
      for (uint64_t i = 0; i < pieces; ++i) {
        const uint64_t len_i = std::min(kIoPiece, n - i * kIoPiece);
        MLCK_CUDA(cudaEventSynchronize(io.ev[i & 1]));  // the buffer's previous H2D is done
        if (std::fread(io.buf[i & 1], 1, len_i, file.f) != len_i)
          throw_runtime(std::string("persist: short read from ") + path);
        MLCK_CUDA(cudaMemcpyAsync(b->dev + i * kIoPiece, io.buf[i & 1], len_i, cudaMemcpyHostToDevice, s));
        MLCK_CUDA(cudaEventRecord(io.ev[i & 1], s));
      }
      MLCK_CUDA(cudaStreamSynchronize(s));
      b->size = n;
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      if (b->dev) cudaFree(b->dev);
      delete b;
      throw;
    }
    ctx->blobs.push_back(b);
    *out = b;
  });
}

// ------------------------------------------------------------------ snapshot
int mlck_snapshot_record(mlck_state* st, const uint32_t* active, uint32_t na, const uint32_t* co,
                         uint32_t nc, uint32_t slot_index, uint8_t kind, uint64_t window_start,
                         uint32_t wsparse, mlck_blob* out) {
  return api([&] {
    st->ctx->activate();
    const auto ents = slot_entries(st, active, na, co, nc);
    SegmentBuilder b;
    build_record(st, ents, kind, st->iteration, window_start, wsparse, slot_index, st->data_seed, b);
    run_pack(st->ctx, b, out, true);
  });
}

int mlck_snapshot_record_host(mlck_state* st, const uint32_t* active, uint32_t na,
                              const uint32_t* co, uint32_t nc, uint32_t slot_index, uint8_t kind,
                              uint64_t window_start, uint32_t wsparse, mlck_blob* scratch,
                              uint8_t* host_out, uint64_t cap, uint64_t* size) {
  return api([&] {
    st->ctx->activate();
    const auto ents = slot_entries(st, active, na, co, nc);
    SegmentBuilder b;
    build_record(st, ents, kind, st->iteration, window_start, wsparse, slot_index, st->data_seed, b);
    const uint64_t n = b.pos + 8;
    if (size) *size = n;
    if (!host_out) return;
    if (cap < n) throw_invalid("snapshot: host buffer too small");
    // the host buffer is one more replica of the record, pushed piece by
    // piece by the copy engines as the pack kernel produces it (transport 1)
    mlck_ctx* ctx = st->ctx;
    struct Restore {
      mlck_ctx* c;
      mlck_blob* b;
      int mode;
      ~Restore() {
        c->replica_mode = mode;
        b->replicas.pop_back();
      }
    } restore{ctx, scratch, ctx->replica_mode};
    scratch->replicas.emplace_back(host_out, cap);
    ctx->replica_mode = 1;
    run_pack(ctx, b, scratch, true);
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->check_watchdog();
  });
}

int mlck_dense_checkpoint(mlck_state* st, mlck_blob* out) {
  return api([&] {
    std::vector<SlotEntry> ents;
    for (uint32_t id = 0; id < st->n_ops; ++id) {
      if (!st->has_full[id])  // snapshot.hpp:283-285
        throw_runtime("dense checkpoint: operator " + std::to_string(id) + " is frozen");
      ents.push_back({id, 0});
    }
    st->ctx->activate();
    SegmentBuilder b;
    build_record(st, ents, 0, st->iteration, st->iteration, 1, 0, st->data_seed, b);
    run_pack(st->ctx, b, out, true);
  });
}

int mlck_fastmath_check(mlck_ctx* ctx, uint64_t n_div, uint64_t seed, uint64_t* mismatches) {
  return api([&] {
    ctx->activate();
    unsigned long long* d = nullptr;
    MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 16, ctx->stream));
    MLCK_CUDA(cudaMemsetAsync(d, 0, 16, ctx->stream));
    launch_fastmath_check(n_div, seed, d, ctx->stream);
    unsigned long long h[2] = {0, 0};
    MLCK_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, ctx->stream));
    MLCK_CUDA(cudaFreeAsync(d, ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    mismatches[0] = h[0];
    mismatches[1] = h[1];
  });
}

int mlck_fnv1a64(mlck_ctx* ctx, const void* ptr, uint64_t n, uint64_t seed, uint64_t* out) {
  return api([&] {
    ctx->activate();
    ctx->join_hash();
    TrailerDsts none{};
    uint32_t* scratch = ctx->fnv_scratch_for(n);
    launch_fnv(static_cast<const uint8_t*>(ptr), n, seed, scratch, ctx->next_epoch(), ctx->results,
               none, ctx->stream);
    ctx->launches += 1;
    MLCK_CUDA(cudaMemcpyAsync(ctx->host_results, ctx->results, 8, cudaMemcpyDeviceToHost,
                              ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->check_watchdog();
    *out = ctx->host_results[0];
  });
}

// FNV with the kernel's profile counters (development aid): 24 counters, see
// fnv::Scratch::prof (fnv.cuh).
int mlck_fnv1a64_profile(mlck_ctx* ctx, const void* ptr, uint64_t n, uint64_t seed, uint64_t* out,
                         uint64_t* counters, uint64_t* trace_host) {
  return api([&] {
    ctx->activate();
    unsigned long long* prof = nullptr;
    MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prof), 24 * 8, ctx->stream));
    MLCK_CUDA(cudaMemsetAsync(prof, 0, 24 * 8, ctx->stream));
    TrailerDsts none{};
    unsigned long long* trace = nullptr;
    const uint64_t tb = fnv_chunks(n) * 12 * 8;
    if (trace_host) {
      MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&trace), tb, ctx->stream));
      MLCK_CUDA(cudaMemsetAsync(trace, 0, tb, ctx->stream));
    }
    uint32_t* scratch = ctx->fnv_scratch_for(n);
    launch_fnv(static_cast<const uint8_t*>(ptr), n, seed, scratch, ctx->next_epoch(), ctx->results,
               none, ctx->stream, prof, trace);
    ctx->launches += 1;
    if (trace_host) {
      MLCK_CUDA(cudaMemcpyAsync(trace_host, trace, tb, cudaMemcpyDeviceToHost, ctx->stream));
      MLCK_CUDA(cudaFreeAsync(trace, ctx->stream));
    }
    MLCK_CUDA(cudaMemcpyAsync(ctx->host_results, ctx->results, 8, cudaMemcpyDeviceToHost,
                              ctx->stream));
    MLCK_CUDA(cudaMemcpyAsync(counters, prof, 24 * 8, cudaMemcpyDeviceToHost, ctx->stream));
    MLCK_CUDA(cudaFreeAsync(prof, ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = ctx->host_results[0];
  });
}

// ------------------------------------------------------------------ parse
int mlck_parse_record(mlck_blob* b, int cb, mlck_record_info* info, mlck_entry_info* entries,
                      uint32_t cap, uint32_t* n_entries) {
  return api([&] {
    b->ctx->activate();
    std::vector<std::string> errs;
    auto p = parse_blobs(b->ctx, &b, 1, cb, errs);
    if (!errs[0].empty()) throw_runtime(errs[0]);
    const auto& h = p[0].hdr;
    if (info) *info = {h.kind, h.iteration, h.window_start, h.wsparse, h.slot, h.data_seed, h.op_count};
    if (n_entries) *n_entries = static_cast<uint32_t>(p[0].entries.size());
    for (uint32_t i = 0; i < std::min<uint32_t>(cap, p[0].entries.size()); ++i) {
      const auto& e = p[0].entries[i];
      entries[i] = {e.id, e.mode, e.param_count, e.step, e.payload_offset};
    }
  });
}

int mlck_read_entry(mlck_blob* b, const mlck_entry_info* e, int cb, float* master, float* m,
                    float* v, float* compute) {
  return api([&] {
    mlck_ctx* ctx = b->ctx;
    ctx->activate();
    if (b->written) MLCK_CUDA(cudaStreamWaitEvent(ctx->stream, b->written, 0));
    const uint64_t P = e->param_count;
    const uint8_t* src = b->dev + e->payload_offset;
    if (e->mode == 0) {
      if (master) MLCK_CUDA(cudaMemcpyAsync(master, src, 4 * P, cudaMemcpyDeviceToHost, ctx->stream));
      if (m) MLCK_CUDA(cudaMemcpyAsync(m, src + 4 * P, 4 * P, cudaMemcpyDeviceToHost, ctx->stream));
      if (v) MLCK_CUDA(cudaMemcpyAsync(v, src + 8 * P, 4 * P, cudaMemcpyDeviceToHost, ctx->stream));
    } else if (compute && P) {
      // codes at an arbitrary offset: stage aligned, decode on device
      void* codes = nullptr;
      float* tmp = nullptr;
      MLCK_CUDA(cudaMallocAsync(&codes, cb * P, ctx->stream));
      MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), 4 * P, ctx->stream));
      MLCK_CUDA(cudaMemcpyAsync(codes, src, cb * P, cudaMemcpyDeviceToDevice, ctx->stream));
      launch_decode(codes, tmp, P, cb, ctx->stream);
      ctx->launches += 1;
      MLCK_CUDA(cudaMemcpyAsync(compute, tmp, 4 * P, cudaMemcpyDeviceToHost, ctx->stream));
      MLCK_CUDA(cudaFreeAsync(codes, ctx->stream));
      MLCK_CUDA(cudaFreeAsync(tmp, ctx->stream));
    }
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mlck_check_coverage(mlck_blob* const* blobs, uint32_t n, uint64_t op_count, int cb) {
  return api([&] {
    if (n == 0) {
      if (op_count) throw_runtime("window coverage violated for operator 0: 0 full payloads");
      return;
    }
    mlck_ctx* ctx = blobs[0]->ctx;
    ctx->activate();
    std::vector<std::string> errs;
    auto p = parse_blobs(ctx, blobs, n, cb, errs);
    std::vector<int> seen(op_count, 0);
    for (uint32_t k = 0; k < n; ++k) {
      if (!errs[k].empty()) throw_runtime(errs[k]);
      for (const auto& e : p[k].entries)
        if (e.mode == 0) {
          if (e.id >= op_count) throw_runtime("window coverage: operator id out of range");
          seen[e.id] += 1;
        }
    }
    for (uint64_t id = 0; id < op_count; ++id)  // snapshot.hpp:329-333
      if (seen[id] != 1)
        throw_runtime("window coverage violated for operator " + std::to_string(id) + ": " +
                      std::to_string(seen[id]) + " full payloads");
  });
}

int mlck_conversion_plan(mlck_blob* const* blobs, uint32_t n, int cb, uint32_t* activating, uint64_t cap,
                         uint64_t* counts, uint64_t* total) {
  return api([&] {
    if (total) *total = 0;
    if (n == 0) return;
    mlck_ctx* ctx = blobs[0]->ctx;
    ctx->activate();
    std::vector<std::string> errs;
    auto p = parse_blobs(ctx, blobs, n, cb, errs);
    uint64_t w = 0;
    for (uint32_t k = 0; k < n; ++k) {  // recovery.hpp:127-134, in slot order
      if (!errs[k].empty()) throw_runtime(errs[k]);
      uint64_t c = 0;
      for (const auto& e : p[k].entries)
        if (e.mode == 0) {
          if (activating && w < cap) activating[w] = e.id;
          ++w;
          ++c;
        }
      if (counts) counts[k] = c;
    }
    if (total) *total = w;
  });
}

// ------------------------------------------------------------------ gradients
int mlck_gradlog_create(mlck_ctx* ctx, uint32_t n_ops, const uint64_t* pc, uint32_t cap,
                        mlck_gradlog** out) {
  return api([&] {
    if (cap == 0) throw_invalid("gradient log: capacity must be >= 1");
    ctx->activate();
    auto* g = new mlck_gradlog();
    g->ctx = ctx;
    g->n_ops = n_ops;
    g->P.assign(pc, pc + n_ops);
    for (uint32_t i = 0; i < n_ops; ++i) {
      g->off.push_back(g->per_iter);
      g->per_iter += align_up(g->P[i], 64);  // 256-byte aligned slots
    }
    g->per_iter = std::max<uint64_t>(g->per_iter, 64);
    g->cap = cap;
    dev_malloc(reinterpret_cast<void**>(&g->pool), 4 * g->per_iter * cap);
    g->ring_iter.assign(cap, -1);
    g->present.assign(cap, std::vector<uint8_t>(n_ops, 0));
    *out = g;
  });
}
int mlck_gradlog_destroy(mlck_gradlog* g) {
  return api([&] {
    if (!g) return;
    g->ctx->activate();
    cudaStreamSynchronize(g->ctx->stream);
    cudaFree(g->pool);
    delete g;
  });
}
int mlck_gradlog_put(mlck_gradlog* g, uint64_t it, uint32_t op, const float* host) {
  return api([&] {
    g->ctx->activate();
    float* d = g->slot(it, op);
    if (g->P[op])
      MLCK_CUDA(cudaMemcpyAsync(d, host, 4 * g->P[op], cudaMemcpyHostToDevice, g->ctx->stream));
    MLCK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}
int mlck_gradlog_capture(mlck_gradlog* g, uint64_t it, uint32_t op, const float* src) {
  return api([&] {
    g->ctx->activate();
    float* d = g->slot(it, op);
    if (!g->P[op]) return;
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {  // slots are 256-byte aligned: SM copy at HBM speed
      launch_copy16(d, src, 4 * g->P[op], g->ctx->stream);
      g->ctx->launches += 1;
    } else {
      ce_copy(d, src, 4 * g->P[op], cudaMemcpyDeviceToDevice, g->ctx->stream);
    }
  });
}
uint64_t mlck_gradlog_bytes(const mlck_gradlog* g) { return g ? 4 * g->per_iter * g->cap : 0; }
int mlck_gradlog_slot(mlck_gradlog* g, uint64_t it, uint32_t op, float** ptr) {
  return api([&] { *ptr = g->slot(it, op); });
}
int mlck_gradlog_fill_synthetic(mlck_gradlog* g, uint64_t first, uint32_t n_it, uint64_t seed) {
  return api([&] {
    g->ctx->activate();
    for (uint32_t k = 0; k < n_it; ++k)
      for (uint32_t op = 0; op < g->n_ops; ++op) {
        const uint64_t it = first + k;
        launch_synth(g->slot(it, op), g->P[op], seed, 1000000ull + it * g->n_ops + op, -1e-2f,
                     1e-2f, g->ctx->stream);
        g->ctx->launches += g->P[op] ? 1 : 0;
      }
  });
}

// ------------------------------------------------------------------ Adam
int mlck_optimizer_step_adam(mlck_ctx* ctx, float* w, float* m, float* v, uint64_t* step,
                             const float* g, uint64_t n, const mlck_optimizer* opt) {
  return api([&] {
    ctx->activate();
    const adam::Opt o = to_opt(opt);
    *step += 1;  // engine.hpp:745
    launch_adam_arrays(w, m, v, g, n, o, bias_correction(o.b1, *step), bias_correction(o.b2, *step),
                       ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}

namespace {
// Launch the fused replay over `ops` (host vectors) with their gradient
// pointers and bias corrections.
void run_replay(mlck_ctx* ctx, std::vector<adam::ConvOp>& ops, const std::vector<const float*>& gptr,
                const std::vector<float2>& bc, const adam::Opt& o, int cb) {
  uint64_t units = 0;  // CTAs: each operator's units round up to whole CTAs
  for (auto& op : ops) {
    op.unit_begin = units;
    units += div_up(div_up(op.P, static_cast<uint64_t>(replay_unit_elems())), static_cast<uint64_t>(replay_cta_threads()));
  }
  const size_t ob = ops.size() * sizeof(adam::ConvOp);
  const size_t go = align_up(ob, 16), gb = gptr.size() * sizeof(float*);
  const size_t bo = align_up(go + gb, 16), bb = bc.size() * sizeof(float2);
  const size_t so = align_up(bo + bb, 16), sb = bc.size() * sizeof(adam::StepConst);
  auto& s = ctx->stage_for(so + sb + 16);  // the StepConst table is filled on the device
  std::memcpy(s.host, ops.data(), ob);
  std::memcpy(s.host + go, gptr.data(), gb);
  std::memcpy(s.host + bo, bc.data(), bb);
  ctx->stage_upload(s, bo + bb);
  const int tr = ctx->tbegin("replay");
  launch_replay(reinterpret_cast<const adam::ConvOp*>(s.dev), static_cast<int>(ops.size()),
                reinterpret_cast<const float* const*>(s.dev + go), reinterpret_cast<const float2*>(s.dev + bo),
                static_cast<uint32_t>(bc.size()), reinterpret_cast<adam::StepConst*>(s.dev + so), o, cb, units,
                ctx->stream);
  ctx->tend(tr);
  ctx->launches += units ? 1 : 0;
}
}  // namespace

int mlck_state_apply_updates(mlck_state* st, const uint32_t* ids, uint32_t n_ids, mlck_gradlog* g,
                             uint64_t iteration, const mlck_optimizer* opt) {
  return api([&] {
    st->ctx->activate();
    const adam::Opt o = to_opt(opt);
    std::vector<adam::ConvOp> ops;
    std::vector<const float*> gptr;
    std::vector<float2> bc;
    for (uint32_t k = 0; k < n_ids; ++k) {
      const uint32_t id = ids[k];
      st->check_id(id);
      adam::ConvOp c{};
      c.src = reinterpret_cast<const uint8_t*>(st->master(id));
      c.dst = st->master(id);
      c.codes = st->codes(id);
      c.P = st->P[id];
      c.n_steps = 1;
      c.grad_base = static_cast<uint32_t>(gptr.size());
      c.bc_base = static_cast<uint32_t>(bc.size());
      gptr.push_back(g->lookup(iteration, id));
      const uint64_t s1 = st->step[id] + 1;  // engine.hpp:713/715
      bc.push_back(make_float2(bias_correction(o.b1, s1), bias_correction(o.b2, s1)));
      st->step[id] = s1;
      ops.push_back(c);
    }
    run_replay(st->ctx, ops, gptr, bc, o, st->cb);
  });
}

// ------------------------------------------------------------------ K3
}  // extern "C"

namespace {
// Merge + Adam replay over the window's records (sparse_to_dense_convert,
// recovery.hpp:180-227) or, with a scope, localized recovery
// (localized_recover, recovery.hpp:240-289): every in-scope operator takes
// its (last) Full payload of the window -- slot k -- and replays the Adam
// steps of iterations a+k+1 .. end from the gradient log, end = a+W for a
// conversion and max(a+W, target) for a localized recovery (the reference
// re-executes the lost iterations after the window from the boundary logs;
// the logged weight gradients are those iterations' gradients).  A W = 1
// conversion returns the record's own state (no replay, recovery.hpp:192-200);
// a W = 1 localized recovery replays iteration a+1 like the reference loop.
void convert_impl(mlck_state* out, mlck_blob* const* blobs, uint32_t n_blobs, uint64_t window_start,
                  uint32_t W, uint64_t data_seed, mlck_gradlog* g, const mlck_optimizer* opt,
                  const std::vector<uint8_t>* scope, uint64_t target) {
  const bool localized = scope != nullptr;
  if (n_blobs != W) {
    if (localized) throw_runtime("sparse checkpoint incomplete");  // recovery.hpp:250-251
    throw_runtime("sparse checkpoint incomplete: " + std::to_string(n_blobs) + " of " +  // 184-187
                  std::to_string(W) + " records");
  }
  mlck_ctx* ctx = out->ctx;
  ctx->activate();
  const uint32_t n_parse = (W == 1 && !localized) ? 1 : W;
  // The entry walk runs first (microseconds), then the records' checksums
  // are verified on the two side streams while the host builds the replay
  // table; the replay follows the verification (run concurrently, the
  // ALU-bound hash and the issue-bound replay only slowed each other down:
  // 13.0 ms vs 12.8 ms sequential, DESIGN 3.3).  Every error surfaces in the
  // reference's order -- a record's parse error (checksum first) before
  // anything the merge finds.
  ParseJob job;
  job.ctx = ctx;
  job.blobs = blobs;
  job.n = n_parse;
  job.cb = out->cb;
  walk_records(job);
  // the witnessed verification can run on a few SMs beside the replay
  bool all_witnessed = ctx->witness && ctx->convert_overlap > 0;
  for (uint32_t k = 0; k < n_parse && all_witnessed; ++k) all_witnessed = blobs[k]->has_witness();
  if (all_witnessed) job.witness_ctas = ctx->convert_overlap;
  verify_begin(job);
  bool verified = false;
  auto parse_errors = [&] {  // recovery.hpp:163-171
    if (verified) return;
    const auto errs = verify_end(job);
    verified = true;
    for (uint32_t k = 0; k < n_parse; ++k)
      if (!errs[k].empty())
        throw_runtime("sparse checkpoint record (slot " + std::to_string(k) + "): " + errs[k]);
  };
  for (uint32_t k = 0; k < n_parse; ++k)
    if (blobs[k]->size < 8 || !job.walk_err[k].empty()) parse_errors();
  const auto& parsed = job.out;
  struct Finish {  // an exception below still joins the side streams
    std::function<void()> f;
    ~Finish() {
      if (f) try { f(); } catch (...) {}
    }
  } join{[&] {
    if (!verified) {
      for (int i = 0; i < 2; ++i) cudaStreamWaitEvent(ctx->stream, ctx->ev_vside[i], 0);
    }
  }};
  auto in_scope = [&](uint32_t id) { return !localized || (id < scope->size() && (*scope)[id]); };
  // each operator's last Full payload in slot order (load_record overwrites)
  struct Src {
    int slot = -1;
    const WalkEntry* e = nullptr;
  };
  std::vector<Src> src(out->n_ops);
  for (uint32_t k = 0; k < n_parse; ++k)
    for (const auto& e : parsed[k].entries) {
      if (e.id >= out->n_ops) {
        parse_errors();
        throw_runtime("conversion: record operator id out of range");
      }
      if (e.mode == 0 && in_scope(e.id)) {
        if (e.param_count != out->P[e.id]) {
          parse_errors();
          throw_invalid("conversion: operator " + std::to_string(e.id) + " size mismatch");
        }
        src[e.id] = {static_cast<int>(k), &e};
      }
    }
  const adam::Opt o = to_opt(opt);
  std::vector<adam::ConvOp> ops;
  std::vector<const float*> gptr;
  std::vector<float2> bc;
  const bool replay = localized || W > 1;
  if (replay)
    for (uint32_t id = 0; id < out->n_ops; ++id)
      if (in_scope(id) && src[id].slot < 0) {
        parse_errors();
        throw_runtime(localized ? "localized recovery left operator " + std::to_string(id) + " frozen"  // 263-266
                                : "conversion finished with frozen operator " + std::to_string(id));  // 222-225
      }
  const uint64_t end = window_start + W + (localized && target > window_start + W ? target - window_start - W : 0);
  std::vector<uint64_t> new_step(out->n_ops, 0);
  for (uint32_t id = 0; id < out->n_ops; ++id) {
    if (!in_scope(id) || src[id].slot < 0) continue;
    const int k = src[id].slot;
    const WalkEntry& e = *src[id].e;
    adam::ConvOp c{};
    c.src = blobs[k]->dev + e.payload_offset;
    c.dst = out->master(id);
    c.codes = out->codes(id);
    c.P = e.param_count;
    c.n_steps = replay ? static_cast<uint32_t>(end - window_start - static_cast<uint64_t>(k)) : 0;
    c.grad_base = static_cast<uint32_t>(gptr.size());
    c.bc_base = static_cast<uint32_t>(bc.size());
    uint64_t stp = e.step;
    for (uint32_t s = 0; s < c.n_steps; ++s) {
      const uint64_t it = window_start + static_cast<uint64_t>(k) + 1 + s;
      if (!g) {
        parse_errors();
        throw_invalid("conversion: gradient log required for W > 1");
      }
      const float* gp = nullptr;
      try {
        gp = g->lookup(it, id);
      } catch (...) {
        parse_errors();
        throw;
      }
      gptr.push_back(gp);
      stp += 1;
      bc.push_back(make_float2(bias_correction(o.b1, stp), bias_correction(o.b2, stp)));
    }
    new_step[id] = stp;
    ops.push_back(c);
  }
  if (all_witnessed) {  // replay beside the verification; its errors still come first
    run_replay(ctx, ops, gptr, bc, o, out->cb);
    parse_errors();
  } else {
    parse_errors();
    run_replay(ctx, ops, gptr, bc, o, out->cb);
  }
  for (uint32_t id = 0; id < out->n_ops; ++id)
    if (in_scope(id)) {
      out->present[id] = src[id].slot >= 0 ? 1 : 0;
      out->has_full[id] = out->present[id];
      out->step[id] = new_step[id];
    }
  if (!replay) {
    out->iteration = parsed[0].hdr.iteration;
    out->data_seed = parsed[0].hdr.data_seed;
  } else {
    out->iteration = end;
    out->data_seed = data_seed;
  }
}
}  // namespace

extern "C" {

int mlck_sparse_to_dense_convert(mlck_state* out, mlck_blob* const* blobs, uint32_t n_blobs,
                                 uint64_t window_start, uint32_t W, uint64_t data_seed,
                                 mlck_gradlog* g, const mlck_optimizer* opt) {
  return api([&] { convert_impl(out, blobs, n_blobs, window_start, W, data_seed, g, opt, nullptr, 0); });
}

int mlck_localized_recover(mlck_state* out, const uint32_t* scope_ids, uint32_t n_scope,
                           mlck_blob* const* blobs, uint32_t n_blobs, uint64_t window_start, uint32_t W,
                           uint64_t data_seed, mlck_gradlog* g, uint64_t target_iteration,
                           const mlck_optimizer* opt) {
  return api([&] {
    std::vector<uint8_t> scope(out->n_ops, 0);
    for (uint32_t i = 0; i < n_scope; ++i) {
      if (scope_ids[i] >= out->n_ops) throw_invalid("unknown operator " + std::to_string(scope_ids[i]));
      scope[scope_ids[i]] = 1;
    }
    convert_impl(out, blobs, n_blobs, window_start, W, data_seed, g, opt, &scope, target_iteration);
  });
}

int mlck_localized_recover_segment(mlck_state* out, int32_t lo, int32_t hi, const int32_t* stage_of_op,
                                   int32_t n_stages, mlck_blob* const* blobs, uint32_t n_blobs,
                                   uint64_t window_start, uint32_t W, uint64_t data_seed, mlck_log* log,
                                   uint32_t n_gmb, mlck_gradlog* g, uint64_t target, const mlck_optimizer* opt) {
  return api([&] {
    if (n_stages < 1 || lo < 0 || hi < lo || hi >= n_stages)
      throw_invalid("recovery segment: stages [" + std::to_string(lo) + ", " + std::to_string(hi) +
                    "] outside 0.." + std::to_string(n_stages - 1));
    if (n_blobs != W) throw_runtime("sparse checkpoint incomplete");  // recovery.hpp:250-251
    // in_scope (recovery.hpp:253-256): Engine::stage_of_op in [stage_lo, stage_hi]
    std::vector<uint8_t> scope(out->n_ops, 0);
    for (uint32_t id = 0; id < out->n_ops; ++id) scope[id] = stage_of_op[id] >= lo && stage_of_op[id] <= hi;
    // run_scoped reads the segment's boundary inputs from the log for every
    // replayed iteration (engine.hpp:361-366 fwd, 393-400 bwd); the
    // replay from logged weight gradients needs none of them, but a log that
    // lacks one fails here as the reference's recovery would
    const uint64_t end = std::max<uint64_t>(window_start + W, target);
    if (lo > 0 || hi < n_stages - 1) {
      if (!log) throw_invalid("localized recovery: the segment needs its neighbours' boundary log");
      for (uint64_t it = window_start + 1; it <= end; ++it)
        for (uint32_t b = 0; b < n_gmb; ++b) {
          uint64_t nf = 0;
          if (lo > 0 && mlck_log_get(log, it, b, static_cast<uint32_t>(lo - 1), 0, nullptr, 0, &nf) != 0)
            throw_runtime(mlck_last_error());
          if (hi < n_stages - 1 && mlck_log_get(log, it, b, static_cast<uint32_t>(hi), 1, nullptr, 0, &nf) != 0)
            throw_runtime(mlck_last_error());
        }
    }
    convert_impl(out, blobs, n_blobs, window_start, W, data_seed, g, opt, &scope, target);
  });
}

// ------------------------------------------------------------------ codecs
}  // extern "C"
namespace {
void check_format(int eb, int mb) {
  if (eb < 2 || eb > 8 || mb < 1 || eb + mb > 15)
    throw_invalid("reduced format: unsupported widths e" + std::to_string(eb) + "m" + std::to_string(mb));
}
// n host values through a device kernel: H2D, launch, D2H on the ctx stream
template <typename In, typename Out, typename Launch>
void host_roundtrip(mlck_ctx* ctx, const In* in, Out* out, uint64_t n, Launch launch) {
  if (!n) return;
  ctx->activate();
  In* din = nullptr;
  Out* dout = nullptr;
  MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&din), sizeof(In) * n, ctx->stream));
  MLCK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), sizeof(Out) * n, ctx->stream));
  MLCK_CUDA(cudaMemcpyAsync(din, in, sizeof(In) * n, cudaMemcpyHostToDevice, ctx->stream));
  launch(din, dout);
  ctx->launches += 1;
  MLCK_CUDA(cudaMemcpyAsync(out, dout, sizeof(Out) * n, cudaMemcpyDeviceToHost, ctx->stream));
  MLCK_CUDA(cudaFreeAsync(din, ctx->stream));
  MLCK_CUDA(cudaFreeAsync(dout, ctx->stream));
  MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
}
}  // namespace
extern "C" {

int mlck_pack_reduced(mlck_ctx* ctx, const float* in, uint16_t* codes, uint64_t n, int eb, int mb) {
  return api([&] {
    check_format(eb, mb);
    ctx->activate();
    launch_pack_reduced(in, codes, n, eb, mb, ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}
int mlck_unpack_reduced(mlck_ctx* ctx, const uint16_t* codes, float* out, uint64_t n, int eb, int mb) {
  return api([&] {
    check_format(eb, mb);
    ctx->activate();
    launch_unpack_reduced(codes, out, n, eb, mb, ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}
int mlck_quantize_values(mlck_ctx* ctx, const float* in, float* out, uint64_t n, int cb) {
  return api([&] {
    if (cb != 1 && cb != 2 && cb != 4) throw_invalid("quantize: unsupported width " + std::to_string(cb));
    host_roundtrip(ctx, in, out, n, [&](const float* di, float* dout) { launch_quantize(di, dout, n, cb, ctx->stream); });
  });
}
int mlck_pack_reduced_values(mlck_ctx* ctx, const float* in, uint16_t* codes, uint64_t n, int eb, int mb) {
  return api([&] {
    check_format(eb, mb);
    host_roundtrip(ctx, in, codes, n,
                   [&](const float* di, uint16_t* dout) { launch_pack_reduced(di, dout, n, eb, mb, ctx->stream); });
  });
}
int mlck_unpack_reduced_values(mlck_ctx* ctx, const uint16_t* codes, float* out, uint64_t n, int eb, int mb) {
  return api([&] {
    check_format(eb, mb);
    host_roundtrip(ctx, codes, out, n,
                   [&](const uint16_t* di, float* dout) { launch_unpack_reduced(di, dout, n, eb, mb, ctx->stream); });
  });
}
int mlck_quantize(mlck_ctx* ctx, const float* in, float* out, uint64_t n, int cb) {
  return api([&] {
    if (cb != 1 && cb != 2 && cb != 4) throw_invalid("quantize: unsupported width " + std::to_string(cb));
    ctx->activate();
    launch_quantize(in, out, n, cb, ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}
int mlck_encode_compute(mlck_ctx* ctx, const float* in, void* codes, uint64_t n, int cb) {
  return api([&] {
    if (cb != 1 && cb != 2 && cb != 4) throw_invalid("container: unsupported compute width");
    ctx->activate();
    launch_encode(in, codes, n, cb, ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}
int mlck_decode_compute(mlck_ctx* ctx, const void* codes, float* out, uint64_t n, int cb) {
  return api([&] {
    if (cb != 1 && cb != 2 && cb != 4) throw_invalid("container: unsupported compute width");
    ctx->activate();
    launch_decode(codes, out, n, cb, ctx->stream);
    ctx->launches += n ? 1 : 0;
  });
}

// ------------------------------------------------------------------ IPC / peers
int mlck_ipc_export(mlck_ctx* ctx, void* ptr, uint8_t handle[64]) {
  return api([&] {
    ctx->activate();
    cudaIpcMemHandle_t h;
    MLCK_CUDA(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(handle, &h, 64);
  });
}
int mlck_ipc_open(mlck_ctx* ctx, const uint8_t handle[64], void** ptr) {
  return api([&] {
    ctx->activate();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    MLCK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
      cudaDriverEntryPointQueryResult q{};
      MLCK_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&get_range),
                                        cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !get_range) throw Error(kCuda, "cuMemGetAddressRange unavailable");
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(*ptr)) != CUDA_SUCCESS)
      throw Error(kCuda, "cuMemGetAddressRange failed on an IPC mapping");
    ctx->ipc_ranges.emplace_back(static_cast<uint64_t>(base), static_cast<uint64_t>(size));
  });
}
int mlck_ipc_close(mlck_ctx* ctx, void* ptr) {
  return api([&] {
    ctx->activate();
    const uint64_t a = reinterpret_cast<uint64_t>(ptr);
    auto& v = ctx->ipc_ranges;
    uint64_t end = a;
    for (const auto& r : v)
      if (r.first == a) end = r.first + r.second;
    v.erase(std::remove_if(v.begin(), v.end(), [&](const auto& r) { return r.first == a; }), v.end());
    // no blob keeps a replica inside the closed mapping (its next record
    // would be stored to unmapped memory): in-flight writes finish first
    ctx->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    for (mlck_blob* b : ctx->blobs)
      for (auto* reps : {&b->replicas, &b->witness_dsts})
        reps->erase(std::remove_if(reps->begin(), reps->end(),
                                   [&](const auto& r) {
                                     const uint64_t p = reinterpret_cast<uint64_t>(r.first);
                                     return p >= a && p < end;
                                   }),
                    reps->end());
    MLCK_CUDA(cudaIpcCloseMemHandle(ptr));
  });
}
int mlck_enable_peer_access(mlck_ctx* ctx, int peer) {
  return api([&] {
    ctx->activate();
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      return;
    }
    MLCK_CUDA(e);
  });
}

// ------------------------------------------------------------------ timing / memory
int mlck_event_record(mlck_ctx* ctx, int slot) {
  return api([&] {
    ctx->join_hash();
    if (slot < 0 || slot >= 16) throw_invalid("event slot out of range");
    MLCK_CUDA(cudaEventRecord(ctx->ev[slot], ctx->stream));
  });
}
int mlck_event_elapsed_ms(mlck_ctx* ctx, int a, int b, float* ms) {
  return api([&] {
    MLCK_CUDA(cudaEventSynchronize(ctx->ev[b]));
    MLCK_CUDA(cudaEventElapsedTime(ms, ctx->ev[a], ctx->ev[b]));
  });
}
int mlck_device_alloc(mlck_ctx* ctx, uint64_t bytes, void** ptr) {
  return api([&] {
    ctx->activate();
    dev_malloc(ptr, std::max<uint64_t>(bytes, 16));
  });
}
int mlck_device_free(mlck_ctx* ctx, void* ptr) {
  return api([&] {
    ctx->activate();
    ctx->join_hash();
    MLCK_CUDA(cudaStreamSynchronize(ctx->stream));
    MLCK_CUDA(cudaFree(ptr));
  });
}
int mlck_device_memset(mlck_ctx* ctx, void* ptr, int value, uint64_t bytes) {
  return api([&] {
    ctx->activate();
    ctx->join_hash();
    MLCK_CUDA(cudaMemsetAsync(ptr, value, bytes, ctx->stream));
  });
}
int mlck_host_alloc_pinned(mlck_ctx* ctx, uint64_t bytes, void** ptr) {
  return api([&] {
    ctx->activate();
    MLCK_CUDA(cudaMallocHost(ptr, std::max<uint64_t>(bytes, 16)));
  });
}
int mlck_host_free_pinned(mlck_ctx* ctx, void* ptr) {
  return api([&] {
    ctx->activate();
    MLCK_CUDA(cudaFreeHost(ptr));
  });
}
int mlck_memcpy_h2d(mlck_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  return api([&] {
    ctx->activate();
    ctx->join_hash();
    MLCK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  });
}
int mlck_memcpy_d2h(mlck_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  return api([&] {
    ctx->activate();
    ctx->join_hash();
    MLCK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  });
}

}  // extern "C"

// =========================================================================
// the GPU toy trainer (engine.cuh): run_iteration / replay_scoped_iteration
// and the recompute conversion / localized recovery
// =========================================================================
struct mlck_engine {
  mlck_ctx* ctx = nullptr;
  toy::Dims m{};
  uint32_t n_ops = 0;
  std::vector<uint64_t> P;
  mlck_optimizer opt{};
  float inv_tokens = 1.0f;
  // device scratch for a scope of every layer
  float *in_acts = nullptr, *targets = nullptr, *grad_in = nullptr, *fwd_out = nullptr, *bwd_out = nullptr;
  float *cache = nullptr, *work = nullptr, *terms = nullptr;
  void** codes_dev = nullptr;     // [n_ops] code pointers of the state in use
  uint8_t* active_dev = nullptr;  // [n_ops]
  float** grads_dev = nullptr;    // [n_ops] gradient destinations
  float* grads_own = nullptr;     // sum P floats: replay gradients (no log)
  std::vector<uint64_t> grads_off;

  int32_t layer_of(uint32_t id) const { return static_cast<int32_t>(id / m.ops_per_layer()); }
  int32_t stage_of_op(uint32_t id) const { return m.stage_of_layer(layer_of(id)); }
};

namespace {

void engine_free(mlck_engine* e) {
  for (void* p : {static_cast<void*>(e->in_acts), static_cast<void*>(e->targets), static_cast<void*>(e->grad_in),
                  static_cast<void*>(e->fwd_out), static_cast<void*>(e->bwd_out), static_cast<void*>(e->cache),
                  static_cast<void*>(e->work), static_cast<void*>(e->terms), static_cast<void*>(e->codes_dev),
                  static_cast<void*>(e->active_dev), static_cast<void*>(e->grads_dev),
                  static_cast<void*>(e->grads_own)})
    if (p) cudaFree(p);
}

// Optimizer steps of the listed operators with the gradients at gptr (one
// step each): Engine::apply_updates (engine.hpp:699-728), then codes refresh.
void apply_updates_ptrs(mlck_state* st, const std::vector<uint32_t>& ids, const std::vector<const float*>& gp,
                        const mlck_optimizer* opt) {
  const adam::Opt o = to_opt(opt);
  std::vector<adam::ConvOp> ops;
  std::vector<const float*> gptr;
  std::vector<float2> bc;
  for (size_t k = 0; k < ids.size(); ++k) {
    const uint32_t id = ids[k];
    adam::ConvOp c{};
    c.src = reinterpret_cast<const uint8_t*>(st->master(id));
    c.dst = st->master(id);
    c.codes = st->codes(id);
    c.P = st->P[id];
    c.n_steps = 1;
    c.grad_base = static_cast<uint32_t>(gptr.size());
    c.bc_base = static_cast<uint32_t>(bc.size());
    gptr.push_back(gp[k]);
    const uint64_t s1 = st->step[id] + 1;
    bc.push_back(make_float2(bias_correction(o.b1, s1), bias_correction(o.b2, s1)));
    st->step[id] = s1;
    ops.push_back(c);
  }
  run_replay(st->ctx, ops, gptr, bc, o, st->cb);
}

// run_scoped (engine.hpp:332-417) + apply_updates over [lo, hi]: frozen[id]
// = no weight gradient, no update.  grads[id]: where an active operator's
// gradient goes (null = the engine's own buffer).
void engine_step(mlck_engine* e, mlck_state* st, uint64_t it, int32_t lo, int32_t hi,
                 const std::vector<uint8_t>& frozen, mlck_log* log_in, mlck_log* log_out,
                 const std::vector<float*>* grads) {
  mlck_ctx* ctx = e->ctx;
  const toy::Dims& m = e->m;
  if (st->n_ops != e->n_ops) throw_invalid("engine: state has " + std::to_string(st->n_ops) + " operators, model " +
                                           std::to_string(e->n_ops));
  int32_t llo = m.layers, lhi = -1;
  for (int32_t l = 0; l < m.layers; ++l)
    if (m.stage_of_layer(l) >= lo && m.stage_of_layer(l) <= hi) {
      llo = std::min(llo, l);
      lhi = std::max(lhi, l);
    }
  if (lhi < llo) throw_runtime("stage range covers no layers");  // engine.hpp:349-350
  const int64_t T = m.tokens(), row = m.mb * m.d;
  const uint32_t n_gmb = static_cast<uint32_t>(m.dp) * static_cast<uint32_t>(m.M);
  cudaStream_t s = ctx->stream;
  // scope inputs: the data stream, or the upstream stage's logged activations
  if (lo == 0) {
    toy::launch_stream(e->in_acts, m, st->data_seed, it, 0, s);
    ctx->launches += 1;
  } else {
    for (uint32_t g = 0; g < n_gmb; ++g) {
      uint64_t nf = 0;
      if (!log_in) throw_invalid("engine: stages above 0 need a boundary log");
      if (mlck_log_get_device(log_in, it, g, static_cast<uint32_t>(lo - 1), 0, e->in_acts + g * row, row, &nf) != 0)
        throw_runtime(mlck_last_error());
    }
  }
  if (hi == m.stages - 1) {
    toy::launch_stream(e->targets, m, st->data_seed, it, 1, s);
    ctx->launches += 1;
  } else {
    for (uint32_t g = 0; g < n_gmb; ++g) {
      uint64_t nf = 0;
      if (!log_in) throw_invalid("engine: stages below the last need a boundary log");
      if (mlck_log_get_device(log_in, it, g, static_cast<uint32_t>(hi), 1, e->grad_in + g * row, row, &nf) != 0)
        throw_runtime(mlck_last_error());
    }
  }
  // per-operator tables: code pointers, active flags, gradient destinations
  std::vector<const void*> codes(e->n_ops);
  std::vector<uint8_t> active(e->n_ops, 0);
  std::vector<float*> gdst(e->n_ops, nullptr);
  std::vector<uint32_t> upd;
  std::vector<const float*> upd_g;
  for (uint32_t id = 0; id < e->n_ops; ++id) {
    codes[id] = st->codes(id);
    const int32_t sg = e->stage_of_op(id);
    if (sg < lo || sg > hi || frozen[id]) continue;
    active[id] = 1;
    gdst[id] = grads && (*grads)[id] ? (*grads)[id] : e->grads_own + e->grads_off[id];
    MLCK_CUDA(cudaMemsetAsync(gdst[id], 0, 4 * e->P[id], s));  // parameters the toy model never reads: 0
    upd.push_back(id);
    upd_g.push_back(gdst[id]);
  }
  const size_t tb = 8 * static_cast<size_t>(e->n_ops);
  auto& stg = ctx->stage_for(3 * tb);
  std::memcpy(stg.host, codes.data(), tb);
  std::memcpy(stg.host + tb, gdst.data(), tb);
  std::memcpy(stg.host + 2 * tb, active.data(), e->n_ops);
  ctx->stage_upload(stg, 2 * tb + e->n_ops);
  MLCK_CUDA(cudaMemcpyAsync(e->codes_dev, stg.dev, tb, cudaMemcpyDeviceToDevice, s));
  MLCK_CUDA(cudaMemcpyAsync(e->grads_dev, stg.dev + tb, tb, cudaMemcpyDeviceToDevice, s));
  MLCK_CUDA(cudaMemcpyAsync(e->active_dev, stg.dev + 2 * tb, e->n_ops, cudaMemcpyDeviceToDevice, s));
  toy::ScopeArgs a{};
  a.m = m;
  a.layer_lo = llo;
  a.layer_hi = lhi;
  a.stage_lo = lo;
  a.stage_hi = hi;
  a.codes = e->codes_dev;
  a.active = e->active_dev;
  a.in_acts = e->in_acts;
  a.targets = e->targets;
  a.grad_in = e->grad_in;
  a.fwd_out = log_out ? e->fwd_out : nullptr;
  a.bwd_out = log_out ? e->bwd_out : nullptr;
  a.cache = e->cache;
  a.work = e->work;
  a.terms = e->terms;
  a.inv_tokens = e->inv_tokens;
  toy::launch_scope(a, s);
  ctx->launches += 1;
  for (int32_t l = llo; l <= lhi; ++l) {
    toy::launch_reduce(a, l, e->grads_dev, s);
    ctx->launches += 1;
  }
  if (log_out)  // sender-side boundary copies (engine.hpp:383-385, 407-409)
    for (int32_t b = lo; b < hi; ++b)
      for (uint32_t g = 0; g < n_gmb; ++g) {
        const int64_t at = ((b - lo) * T + static_cast<int64_t>(g) * m.mb) * m.d;
        if (mlck_log_put(log_out, it, g, static_cast<uint32_t>(b), 0, e->fwd_out + at, row) != 0 ||
            mlck_log_put(log_out, it, g, static_cast<uint32_t>(b), 1, e->bwd_out + at, row) != 0)
          throw_runtime(mlck_last_error());
      }
  if (!upd.empty()) apply_updates_ptrs(st, upd, upd_g, &e->opt);
}

// load_record (recovery.hpp:144-161): Full payloads replace the operator's
// state (refresh_compute); compute-only payloads set the codes of operators
// still frozen.
void load_record_dev(mlck_state* st, mlck_blob* b, const Parsed& pr, const std::vector<uint8_t>& scope) {
  cudaStream_t s = st->ctx->stream;
  for (const auto& en : pr.entries) {
    const uint32_t id = en.id;
    if (id >= st->n_ops) throw_runtime("conversion: record operator id out of range");
    if (!scope[id]) continue;
    if (en.param_count != st->P[id]) throw_invalid("conversion: operator " + std::to_string(id) + " size mismatch");
    const uint64_t P = en.param_count;
    if (en.mode == 0) {
      if (P) {
        ce_copy(st->master(id), b->dev + en.payload_offset, 12 * P, cudaMemcpyDeviceToDevice, s);
        launch_encode(st->master(id), st->codes(id), P, st->cb, s);
        st->ctx->launches += 1;
      }
      st->step[id] = en.step;
      st->has_full[id] = 1;
      st->present[id] = 1;
    } else if (!st->has_full[id]) {
      if (P) ce_copy(st->codes(id), b->dev + en.payload_offset, static_cast<uint64_t>(st->cb) * P,
                     cudaMemcpyDeviceToDevice, s);
      st->present[id] = 1;
    }
  }
}

void convert_recompute(mlck_engine* e, mlck_state* out, mlck_blob* const* blobs, uint32_t n, uint64_t a,
                       uint32_t W, uint64_t data_seed, const int32_t* seg, mlck_log* logs, uint64_t target) {
  const bool localized = seg != nullptr;
  if (n != W) {
    if (localized) throw_runtime("sparse checkpoint incomplete");
    throw_runtime("sparse checkpoint incomplete: " + std::to_string(n) + " of " + std::to_string(W) + " records");
  }
  mlck_ctx* ctx = e->ctx;
  ctx->activate();
  if (out->n_ops != e->n_ops) throw_invalid("engine: state / model operator count mismatch");
  const int32_t lo = localized ? seg[0] : 0, hi = localized ? seg[1] : e->m.stages - 1;
  std::vector<uint8_t> scope(e->n_ops, 0);
  for (uint32_t id = 0; id < e->n_ops; ++id) scope[id] = e->stage_of_op(id) >= lo && e->stage_of_op(id) <= hi;
  std::vector<std::string> errs;
  const uint32_t n_parse = (W == 1 && !localized) ? 1 : W;
  auto parsed = parse_blobs(ctx, blobs, n_parse, out->cb, errs);
  for (uint32_t k = 0; k < n_parse; ++k)  // recovery.hpp:163-171
    if (!errs[k].empty()) throw_runtime("sparse checkpoint record (slot " + std::to_string(k) + "): " + errs[k]);
  for (uint32_t id = 0; id < e->n_ops; ++id)
    if (scope[id]) out->has_full[id] = 0;
  if (!localized && W == 1) {  // recovery.hpp:190-200
    load_record_dev(out, blobs[0], parsed[0], scope);
    out->iteration = parsed[0].hdr.iteration;
    out->data_seed = parsed[0].hdr.data_seed;
    return;
  }
  out->iteration = a;
  out->data_seed = data_seed;
  std::vector<uint8_t> frozen(e->n_ops, 1);
  uint64_t it = a;
  for (uint32_t k = 0; k < W; ++k) {
    load_record_dev(out, blobs[k], parsed[k], scope);
    for (uint32_t id = 0; id < e->n_ops; ++id)
      if (scope[id] && out->has_full[id]) frozen[id] = 0;
    it = a + k + 1;
    engine_step(e, out, it, lo, hi, frozen, localized ? logs : nullptr, nullptr, nullptr);
    out->iteration = it;
  }
  for (uint32_t id = 0; id < e->n_ops; ++id)
    if (scope[id] && !out->has_full[id])
      throw_runtime(localized ? "localized recovery left operator " + std::to_string(id) + " frozen"  // 263-266
                              : "conversion finished with frozen operator " + std::to_string(id));  // 222-225
  while (localized && it < target) {  // the lost iterations after the window (recovery.hpp:269-273)
    it += 1;
    engine_step(e, out, it, lo, hi, frozen, logs, nullptr, nullptr);
    out->iteration = it;
  }
}

}  // namespace

extern "C" {

int mlck_engine_create(mlck_ctx* ctx, const mlck_engine_config* c, mlck_engine** out) {
  return api([&] {
    if (c->layers < 1 || c->experts_per_layer < 1 || c->token_dim < 1 || c->pp_stages < 1 || c->dp_degree < 1 ||
        c->microbatches < 1 || c->microbatch_size < 1)
      throw_invalid("engine: every dimension must be >= 1");
    if (c->top_k + c->shared_experts > c->experts_per_layer)  // engine.hpp:111-112
      throw_invalid("engine: top_k + shared_experts > experts_per_layer");
    if (c->pp_stages > c->layers) throw_invalid("engine: more pipeline stages than layers");
    if (c->compute_bytes != 1 && c->compute_bytes != 2 && c->compute_bytes != 4)
      throw_invalid("quantize: unsupported width " + std::to_string(c->compute_bytes));
    ctx->activate();
    auto* e = new mlck_engine();
    e->ctx = ctx;
    toy::Dims& m = e->m;
    m.layers = c->layers;
    m.E = c->experts_per_layer;
    m.top_k = c->top_k;
    m.shared = c->shared_experts;
    m.d = c->token_dim;
    m.he = c->expert_hidden;
    m.hn = c->nonexpert_hidden;
    m.residual = c->residual;
    m.stages = c->pp_stages;
    m.dp = c->dp_degree;
    m.M = c->microbatches;
    m.mb = c->microbatch_size;
    m.cb = c->compute_bytes;
    // ModelSpec::derived_*_params (core.hpp:86-100)
    m.pe = c->expert_params >= 0 ? c->expert_params : toy::Dims::mlp_live(m.d, m.he);
    m.pn = c->nonexpert_params >= 0 ? c->nonexpert_params : toy::Dims::mlp_live(m.d, m.hn);
    m.pg = c->gate_params >= 0 ? c->gate_params : m.g_live();
    if (m.pe < m.e_live() || m.pn < m.ne_live() || m.pg < m.g_live())
      throw_invalid("engine: explicit parameter counts below the toy model's");
    e->opt = c->optimizer;
    e->n_ops = static_cast<uint32_t>(m.layers) * static_cast<uint32_t>(m.ops_per_layer());
    uint64_t tot = 0;
    for (uint32_t id = 0; id < e->n_ops; ++id) {
      const uint32_t j = id % m.ops_per_layer();
      const uint64_t p = j < static_cast<uint32_t>(m.E) ? m.pe : j == static_cast<uint32_t>(m.E) ? m.pn : m.pg;
      e->P.push_back(p);
      e->grads_off.push_back(tot);
      tot += align_up(p, 64);
    }
    e->inv_tokens = 1.0f / static_cast<float>(m.tokens());  // engine.hpp:341-342
    const int64_t T = m.tokens(), d = m.d;
    const toy::CacheLayout L(m);
    const toy::TermLayout TL(m);
    const int64_t hmax = std::max<int64_t>(1, std::max(m.he, m.hn));
    auto alloc = [&](auto** p, uint64_t bytes) { dev_malloc(reinterpret_cast<void**>(p), std::max<uint64_t>(bytes, 256)); };
    alloc(&e->in_acts, 4 * T * d);
    alloc(&e->targets, 4 * T * d);
    alloc(&e->grad_in, 4 * T * d);
    alloc(&e->fwd_out, 4 * T * d * std::max(1, m.stages - 1));
    alloc(&e->bwd_out, 4 * T * d * std::max(1, m.stages - 1));
    alloc(&e->cache, 4 * T * m.layers * L.stride);
    alloc(&e->work, 4 * T * (4 * d + 2 * m.nsel() + 2 * hmax));
    alloc(&e->terms, 4 * T * m.layers * TL.stride);
    alloc(&e->codes_dev, 8 * e->n_ops);
    alloc(&e->active_dev, e->n_ops);
    alloc(&e->grads_dev, 8 * e->n_ops);
    alloc(&e->grads_own, 4 * tot);
    *out = e;
  });
}

int mlck_engine_destroy(mlck_engine* e) {
  return api([&] {
    if (!e) return;
    e->ctx->activate();
    cudaStreamSynchronize(e->ctx->stream);
    engine_free(e);
    delete e;
  });
}

uint32_t mlck_engine_op_count(const mlck_engine* e) { return e ? e->n_ops : 0; }
int mlck_engine_param_counts(const mlck_engine* e, uint64_t* out) {
  return api([&] { std::copy(e->P.begin(), e->P.end(), out); });
}
int32_t mlck_engine_stage_of_op(const mlck_engine* e, uint32_t id) {
  return e && id < e->n_ops ? e->stage_of_op(id) : -1;
}

int mlck_engine_run_iteration(mlck_engine* e, mlck_state* st, const uint8_t* frozen, mlck_log* log_out,
                              mlck_gradlog* grads_out) {
  return api([&] {
    e->ctx->activate();
    const uint64_t it = st->iteration + 1;
    std::vector<uint8_t> fz(e->n_ops, 0);
    if (frozen) fz.assign(frozen, frozen + e->n_ops);
    std::vector<float*> gd(e->n_ops, nullptr);
    if (grads_out) {
      if (grads_out->n_ops != e->n_ops) throw_invalid("gradient log: operator count mismatch");
      for (uint32_t id = 0; id < e->n_ops; ++id)
        if (!fz[id]) gd[id] = grads_out->slot(it, id);  // zero-copy capture
    }
    engine_step(e, st, it, 0, e->m.stages - 1, fz, nullptr, log_out, &gd);
    st->iteration = it;
  });
}

int mlck_engine_replay_scoped_iteration(mlck_engine* e, mlck_state* ops, uint64_t it, int32_t lo, int32_t hi,
                                        const uint8_t* frozen, mlck_log* log_in) {
  return api([&] {
    if (lo < 0 || hi < lo || hi >= e->m.stages) throw_invalid("replay: stage range out of bounds");
    e->ctx->activate();
    std::vector<uint8_t> fz(e->n_ops, 0);
    if (frozen) fz.assign(frozen, frozen + e->n_ops);
    engine_step(e, ops, it, lo, hi, fz, log_in, nullptr, nullptr);
  });
}

int mlck_sparse_to_dense_convert_recompute(mlck_engine* e, mlck_state* out, mlck_blob* const* blobs, uint32_t n,
                                           uint64_t a, uint32_t W, uint64_t data_seed) {
  return api([&] { convert_recompute(e, out, blobs, n, a, W, data_seed, nullptr, nullptr, 0); });
}

int mlck_localized_recover_recompute(mlck_engine* e, mlck_state* out, int32_t lo, int32_t hi,
                                     mlck_blob* const* blobs, uint32_t n, uint64_t a, uint32_t W,
                                     uint64_t data_seed, mlck_log* logs, uint64_t target) {
  return api([&] {
    if (lo < 0 || hi < lo || hi >= e->m.stages) throw_invalid("recovery segment: stage range out of bounds");
    const int32_t seg[2] = {lo, hi};
    convert_recompute(e, out, blobs, n, a, W, data_seed, seg, logs, target);
  });
}

}  // extern "C"
