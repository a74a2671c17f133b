// moelab_b200/checkpoint.hpp -- C++ drop-in for the reference checkpoint API
// (/root/reference/proj/include/moelab: snapshot.hpp, recovery.hpp, the
// optimizer/log parts of engine.hpp, tensor.hpp codecs, digest.hpp FNV),
// implemented on the sm_100a kernels through the C ABI in mlck_b200.h.
//
// Same names, same argument meaning, same exception types and texts as the
// reference; the differences are where the data lives:
//   * Engine's TrainState  -> DeviceState (HBM arena, one per device)
//   * SnapshotRecord       -> a descriptor (no host copies of payloads)
//   * SparseCheckpoint::blobs -> device records (+ peer replicas)
//   * sparse_to_dense_convert replays Adam from a GradientLog instead of
//     re-running the toy model (bit-identical).
// Header-only; link with libmlck_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../mlck_b200.h"

namespace moelab_b200 {

// ---- errors: C-ABI status -> the reference's exception types -------------
inline void check(int rc) {
  if (rc == MLCK_OK) return;
  const std::string msg = mlck_last_error();
  if (rc == MLCK_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// ---- vocabulary (core.hpp:16-27, 202-220; engine.hpp:21-28) -------------
struct PrecisionPlan {
  int64_t compute_bytes = 2;
  int64_t master_bytes = 4;
  int64_t optimizer_bytes = 8;
  int64_t full_state_bytes() const { return master_bytes + optimizer_bytes; }
  void check() const {
    if (compute_bytes < 1 || master_bytes < 1 || optimizer_bytes < 1)
      throw std::invalid_argument("precision plan: all byte widths must be >= 1");
  }
};

enum class SnapshotMode : uint8_t { Full = 0, ComputeOnly = 1 };

struct ScheduleSlot {
  std::vector<uint32_t> active;
  std::vector<uint32_t> compute_only;
};

struct OptimizerConfig {
  enum class Kind : uint8_t { Adam = 0, Sgd = 1 };
  Kind kind = Kind::Adam;
  float lr = 1e-3f;
  float beta1 = 0.9f;
  float beta2 = 0.999f;
  float eps = 1e-8f;
  mlck_optimizer abi() const {
    return {kind == Kind::Adam ? 0 : 1, lr, beta1, beta2, eps};
  }
};

// The slices of ModelSpec / ParallelPlan / ClusterSpec (core.hpp:66-190)
// the checkpoint path reads: operator layout, pipeline shape, host budget.
struct ModelSpec {
  int32_t layers = 1;
  int32_t experts_per_layer = 1;
  int32_t token_dim = 4;
  int64_t operator_count() const { return static_cast<int64_t>(layers) * (experts_per_layer + 2); }
};
struct ParallelPlan {
  int32_t pp_stages = 1;
  int32_t dp_degree = 1;
  int32_t microbatches = 1;
  int64_t microbatch_size = 1;
  int32_t stage_of_layer(int32_t layer, int32_t layers) const {  // core.hpp:187-190
    return static_cast<int32_t>((static_cast<int64_t>(layer) * pp_stages) / layers);
  }
};
struct ClusterSpec {
  int32_t nodes = 1;
  double cpu_mem_per_node = 0.0;  // bytes; 0 = unchecked
};
// Engine::stage_of_op for every operator id (engine.hpp:170-172): ids are
// layer-major, E experts then the non-expert block and the gate per layer
// (ModelSpec::operators, core.hpp:105-134).
inline std::vector<int32_t> stage_of_ops(const ModelSpec& m, const ParallelPlan& p) {
  std::vector<int32_t> st(static_cast<size_t>(m.operator_count()));
  for (size_t id = 0; id < st.size(); ++id)
    st[id] = p.stage_of_layer(static_cast<int32_t>(id / (m.experts_per_layer + 2)), m.layers);
  return st;
}

// upstream_log_bytes / check_log_budget (recovery.hpp:296-317)
inline int64_t upstream_log_bytes(const ModelSpec& m, const ParallelPlan& p, int64_t wsparse) {
  return mlck_upstream_log_bytes(m.token_dim, p.pp_stages, p.microbatches, p.microbatch_size, p.dp_degree,
                                 wsparse);
}
inline void check_log_budget(const ModelSpec& m, const ParallelPlan& p, int64_t wsparse, const ClusterSpec& c) {
  check(mlck_check_log_budget(m.token_dim, p.pp_stages, p.microbatches, p.microbatch_size, p.dp_degree, wsparse,
                              c.cpu_mem_per_node, c.nodes));
}

// ---- device context -------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) { check(mlck_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) mlck_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mlck_ctx* get() const { return h_; }
  void synchronize() const { check(mlck_ctx_synchronize(h_)); }
  // SMs the hash kernel leaves to co-scheduled training work
  void set_hash_reserve(int sms) const { check(mlck_ctx_set_hash_reserve(h_, sms)); }
  // The context the scalar codec forms use when none is given (device 0).
  static Context& default_context() {
    thread_local Context c(0);
    return c;
  }

 private:
  mlck_ctx* h_ = nullptr;
};

// ---- codecs (tensor.hpp:99-183): the reference's scalar forms, computed by
// the device codec kernels (bit-identical to the bulk paths) ---------------
inline float quantize_value(Context& ctx, float x, int compute_bytes) {
  float y = 0.0f;
  check(mlck_quantize_values(ctx.get(), &x, &y, 1, compute_bytes));
  return y;
}
inline uint16_t pack_reduced(Context& ctx, float x, int ebits, int mbits) {
  uint16_t c = 0;
  check(mlck_pack_reduced_values(ctx.get(), &x, &c, 1, ebits, mbits));
  return c;
}
inline float unpack_reduced(Context& ctx, uint16_t code, int ebits, int mbits) {
  float y = 0.0f;
  check(mlck_unpack_reduced_values(ctx.get(), &code, &y, 1, ebits, mbits));
  return y;
}
inline float quantize_value(float x, int compute_bytes) {
  return quantize_value(Context::default_context(), x, compute_bytes);
}
inline uint16_t pack_reduced(float x, int ebits, int mbits) {
  return pack_reduced(Context::default_context(), x, ebits, mbits);
}
inline float unpack_reduced(uint16_t code, int ebits, int mbits) {
  return unpack_reduced(Context::default_context(), code, ebits, mbits);
}

// Host view of one operator (OperatorState, engine.hpp:33-45).
struct OperatorState {
  std::vector<float> master, m, v;
  uint64_t step = 0;
  std::vector<float> compute;
  bool has_full_state = false;
};

// ---- TrainState in HBM (engine.hpp:47-51) ---------------------------------
class DeviceState {
 public:
  DeviceState(Context& ctx, std::vector<uint64_t> param_counts, int compute_bytes)
      : ctx_(&ctx), pc_(std::move(param_counts)) {
    check(mlck_state_create(ctx.get(), static_cast<uint32_t>(pc_.size()), pc_.data(),
                            compute_bytes, &h_));
  }
  ~DeviceState() {
    if (h_) mlck_state_destroy(h_);
  }
  DeviceState(const DeviceState&) = delete;
  DeviceState& operator=(const DeviceState&) = delete;

  mlck_state* get() const { return h_; }
  Context& context() const { return *ctx_; }
  size_t op_count() const { return pc_.size(); }
  uint64_t param_count(uint32_t id) const { return pc_.at(id); }

  uint64_t iteration() const {
    uint64_t it = 0, seed = 0;
    check(mlck_state_get_meta(h_, &it, &seed));
    return it;
  }
  uint64_t data_seed() const {
    uint64_t it = 0, seed = 0;
    check(mlck_state_get_meta(h_, &it, &seed));
    return seed;
  }
  void set_meta(uint64_t iteration, uint64_t data_seed) {
    check(mlck_state_set_meta(h_, iteration, data_seed));
  }
  // Uploads one operator; compute = quantize(master) on the device.
  void set_op(uint32_t id, const OperatorState& op) {
    check(mlck_state_upload_op(h_, id, op.master.data(), op.m.data(), op.v.data(), op.step,
                               op.has_full_state ? 1 : 0));
  }
  OperatorState op(uint32_t id) const {
    OperatorState o;
    const uint64_t n = pc_.at(id);
    o.master.resize(n);
    o.m.resize(n);
    o.v.resize(n);
    o.compute.resize(n);
    int hf = 0;
    check(mlck_state_download_op(h_, id, o.master.data(), o.m.data(), o.v.data(), &o.step,
                                 o.compute.data(), &hf));
    o.has_full_state = hf != 0;
    return o;
  }
  void set_has_full_state(uint32_t id, uint64_t step, bool full) {
    check(mlck_state_set_step(h_, id, step, full ? 1 : 0));
  }
  // Engine::serialize_state (engine.hpp:246-261)
  std::vector<uint8_t> serialize_state() const {
    uint64_t n = 0;
    check(mlck_state_serialize(h_, nullptr, 0, &n));
    std::vector<uint8_t> out(n);
    check(mlck_state_serialize(h_, out.data(), n, &n));
    return out;
  }

 private:
  Context* ctx_;
  std::vector<uint64_t> pc_;
  mlck_state* h_ = nullptr;
};

// ---- records in HBM --------------------------------------------------------
class DeviceBlob {
 public:
  explicit DeviceBlob(Context& ctx, uint64_t capacity = 256) : ctx_(&ctx) {
    check(mlck_blob_create(ctx.get(), capacity, &h_));
  }
  DeviceBlob(Context& ctx, std::span<const uint8_t> bytes) : ctx_(&ctx) {
    check(mlck_blob_from_host(ctx.get(), bytes.data(), bytes.size(), &h_));
  }
  ~DeviceBlob() {
    if (h_) mlck_blob_destroy(h_);
  }
  DeviceBlob(DeviceBlob&& o) noexcept : ctx_(o.ctx_), h_(std::exchange(o.h_, nullptr)) {}
  DeviceBlob& operator=(DeviceBlob&& o) noexcept {
    std::swap(h_, o.h_);
    ctx_ = o.ctx_;
    return *this;
  }
  DeviceBlob(const DeviceBlob&) = delete;

  mlck_blob* get() const { return h_; }
  uint64_t size() const { return mlck_blob_size(h_); }
  std::vector<uint8_t> bytes() const {
    std::vector<uint8_t> out(size());
    check(mlck_blob_to_host(h_, out.data(), out.size()));
    return out;
  }
  // replica written by the same pack kernel (peer buffer via IPC or local)
  void add_replica(void* device_ptr, uint64_t capacity) {
    check(mlck_blob_add_replica(h_, device_ptr, capacity));
  }
  // each record's witness also goes to this buffer beside a replica
  // (capacity >= witness_bytes(record size)): a node recovering from the
  // replica wraps both and verifies on the witnessed path
  void add_replica_witness(void* device_ptr, uint64_t capacity) {
    check(mlck_blob_add_replica_witness(h_, device_ptr, capacity));
  }
  static uint64_t witness_bytes(uint64_t record_bytes) { return mlck_witness_bytes(record_bytes); }
  // a read-only view of `n` record bytes the caller owns in device memory (a
  // replica buffer) and its witness, if any: no copy
  static DeviceBlob wrap(Context& ctx, void* record, uint64_t n, const void* witness = nullptr) {
    DeviceBlob b(ctx, nullptr);
    check(mlck_blob_wrap(ctx.get(), record, n, witness, &b.h_));
    return b;
  }
  // replicas holding the complete last record (0 while its push is in flight)
  uint32_t replication() const {
    uint32_t n = 0;
    check(mlck_blob_replication(h_, &n));
    return n;
  }
  // the record bytes (MLCK v1 wire format) to / from a file
  void save(const std::string& path) const { check(mlck_blob_save(h_, path.c_str(), nullptr)); }
  static DeviceBlob load(Context& ctx, const std::string& path) {
    DeviceBlob b(ctx, nullptr);
    check(mlck_blob_load(ctx.get(), path.c_str(), &b.h_));
    return b;
  }

 private:
  DeviceBlob(Context& ctx, std::nullptr_t) : ctx_(&ctx) {}
  Context* ctx_;
  mlck_blob* h_ = nullptr;
};

// take_sparse_snapshot(engine, slot, slot_index) (snapshot.hpp:204-241): the
// GPU version keeps the payloads where they are; the record is what to pack.
struct SnapshotRecord {
  const DeviceState* state = nullptr;
  ScheduleSlot slot;
  uint32_t slot_index = 0;
  uint64_t iteration = 0;
  uint64_t data_seed = 0;
};

inline SnapshotRecord take_sparse_snapshot(const DeviceState& st, const ScheduleSlot& slot,
                                           uint32_t slot_index) {
  for (uint32_t id : slot.active)
    if (id >= st.op_count())
      throw std::invalid_argument("snapshot slot references unknown operator " +
                                  std::to_string(id));
  for (uint32_t id : slot.compute_only)
    if (id >= st.op_count())
      throw std::invalid_argument("snapshot slot references unknown operator " +
                                  std::to_string(id));
  return {&st, slot, slot_index, st.iteration(), st.data_seed()};
}

// serialize_record (snapshot.hpp:115-144) into a device record.
inline void serialize_record(const SnapshotRecord& rec, const PrecisionPlan& plan, uint8_t kind,
                             uint64_t window_start, uint32_t wsparse, DeviceBlob& out) {
  plan.check();
  const auto& s = rec.slot;
  check(mlck_snapshot_record(rec.state->get(), s.active.data(),
                             static_cast<uint32_t>(s.active.size()), s.compute_only.data(),
                             static_cast<uint32_t>(s.compute_only.size()), rec.slot_index, kind,
                             window_start, wsparse, out.get()));
}
// ... and the reference's by-value host bytes.
inline std::vector<uint8_t> serialize_record(const SnapshotRecord& rec, const PrecisionPlan& plan,
                                             uint8_t kind, uint64_t window_start,
                                             uint32_t wsparse) {
  DeviceBlob tmp(rec.state->context());
  serialize_record(rec, plan, kind, window_start, wsparse, tmp);
  return tmp.bytes();
}

// fnv1a64 (digest.hpp:18-25) over host bytes (uploaded) -- device kernel.
inline uint64_t fnv1a64(Context& ctx, std::span<const uint8_t> data,
                        uint64_t seed = 0xcbf29ce484222325ull) {
  DeviceBlob b(ctx, data);
  uint64_t h = 0;
  check(mlck_fnv1a64(ctx.get(), mlck_blob_device_ptr(b.get()), data.size(), seed, &h));
  return h;
}

// ---- parse (snapshot.hpp:146-197) ------------------------------------------
struct SnapshotPayload {
  SnapshotMode mode = SnapshotMode::Full;
  std::vector<float> master, m, v;
  uint64_t step = 0;
  std::vector<float> compute;
};
struct ParsedRecord {
  uint64_t iteration = 0;
  uint32_t slot = 0;
  uint64_t data_seed = 0;
  std::vector<std::pair<uint32_t, SnapshotPayload>> entries;
  uint64_t window_start = 0;
  uint32_t wsparse = 0;
  uint8_t kind = 0;
};

inline ParsedRecord parse_record(const DeviceBlob& blob, const PrecisionPlan& plan) {
  mlck_record_info info{};
  uint32_t n = 0;
  const int cb = static_cast<int>(plan.compute_bytes);
  check(mlck_parse_record(blob.get(), cb, &info, nullptr, 0, &n));
  std::vector<mlck_entry_info> ents(n);
  check(mlck_parse_record(blob.get(), cb, &info, ents.data(), n, &n));
  ParsedRecord pr;
  pr.iteration = info.iteration;
  pr.slot = info.slot;
  pr.data_seed = info.data_seed;
  pr.window_start = info.window_start;
  pr.wsparse = info.wsparse;
  pr.kind = info.kind;
  for (uint32_t i = 0; i < n; ++i) {
    SnapshotPayload p;
    const auto& e = ents[i];
    p.mode = e.mode == 0 ? SnapshotMode::Full : SnapshotMode::ComputeOnly;
    p.step = e.step;
    if (e.mode == 0) {
      p.master.resize(e.param_count);
      p.m.resize(e.param_count);
      p.v.resize(e.param_count);
      check(mlck_read_entry(blob.get(), &e, cb, p.master.data(), p.m.data(), p.v.data(), nullptr));
    } else {
      p.compute.resize(e.param_count);
      check(mlck_read_entry(blob.get(), &e, cb, nullptr, nullptr, nullptr, p.compute.data()));
    }
    pr.entries.emplace_back(e.id, std::move(p));
  }
  return pr;
}
inline ParsedRecord parse_record(Context& ctx, std::span<const uint8_t> blob,
                                 const PrecisionPlan& plan) {
  return parse_record(DeviceBlob(ctx, blob), plan);
}

// ---- SparseCheckpoint window (snapshot.hpp:297-335) ------------------------
struct SparseCheckpoint {
  uint64_t window_start = 0;
  uint32_t wsparse = 0;
  int32_t replication_target = 2;
  std::vector<DeviceBlob> blobs;       // one per record, slot order (device)
  std::vector<int32_t> replication;    // peer copies per record

  void add_record(const SnapshotRecord& rec, const PrecisionPlan& plan) {
    blobs.emplace_back(rec.state->context());
    serialize_record(rec, plan, /*kind=*/1, window_start, wsparse, blobs.back());
    replication.push_back(0);
  }
  bool complete() const { return blobs.size() == wsparse; }
  bool persisted() const {
    if (!complete()) return false;
    for (int32_t r : replication)
      if (r < replication_target) return false;
    return true;
  }
  void check_coverage(size_t op_count, const PrecisionPlan& plan) const {
    std::vector<mlck_blob*> hs;
    for (const auto& b : blobs) hs.push_back(b.get());
    check(mlck_check_coverage(hs.data(), static_cast<uint32_t>(hs.size()), op_count,
                              static_cast<int>(plan.compute_bytes)));
  }
  // Device-driven counters: a record's replicas count once its
  // push completed; a durable file copy (save) counts as one more.
  std::vector<int32_t> durable;
  void poll_replication() {
    durable.resize(blobs.size(), 0);
    for (size_t k = 0; k < blobs.size(); ++k)
      replication[k] = std::max<int32_t>(replication[k],
                                         static_cast<int32_t>(blobs[k].replication()) + durable[k]);
  }
  // Persist the window: record k as <dir>/window_<start>_slot_<k>.mlck (the
  // bytes of the reference's blobs[k]); the caller owns the directory.
  void save(const std::string& dir) {
    durable.resize(blobs.size(), 0);
    for (size_t k = 0; k < blobs.size(); ++k) {
      blobs[k].save(dir + "/window_" + std::to_string(window_start) + "_slot_" + std::to_string(k) + ".mlck");
      durable[k] += 1;
    }
    poll_replication();
  }
  static SparseCheckpoint load(Context& ctx, const std::string& dir, uint64_t window_start,
                               uint32_t wsparse) {
    SparseCheckpoint ck;
    ck.window_start = window_start;
    ck.wsparse = wsparse;
    for (uint32_t k = 0; k < wsparse; ++k) {
      ck.blobs.push_back(DeviceBlob::load(
          ctx, dir + "/window_" + std::to_string(window_start) + "_slot_" + std::to_string(k) + ".mlck"));
      ck.replication.push_back(0);
      ck.durable.push_back(1);
    }
    ck.poll_replication();
    return ck;
  }
};

// ---- conversion_plan (recovery.hpp:112-137) -------------------------------
struct ConversionStep {
  uint32_t record_index = 0;
  uint64_t replay_iteration = 0;
  std::vector<uint32_t> activating;
};
struct ConversionPlan {
  uint64_t window_start = 0;
  std::vector<ConversionStep> steps;
};
inline ConversionPlan conversion_plan(const SparseCheckpoint& ckpt, const PrecisionPlan& plan) {
  ConversionPlan cp;
  cp.window_start = ckpt.window_start;
  if (ckpt.blobs.size() < ckpt.wsparse)  // the reference's ckpt.blobs.at(k)
    throw std::out_of_range("vector::_M_range_check: __n (which is " + std::to_string(ckpt.blobs.size()) +
                            ") >= this->size() (which is " + std::to_string(ckpt.blobs.size()) + ")");
  std::vector<mlck_blob*> hs;
  for (uint32_t k = 0; k < ckpt.wsparse; ++k) hs.push_back(ckpt.blobs[k].get());
  std::vector<uint64_t> counts(hs.size());
  uint64_t total = 0;
  const int cb = static_cast<int>(plan.compute_bytes);
  check(mlck_conversion_plan(hs.data(), static_cast<uint32_t>(hs.size()), cb, nullptr, 0, counts.data(), &total));
  std::vector<uint32_t> ids(total);
  check(mlck_conversion_plan(hs.data(), static_cast<uint32_t>(hs.size()), cb, ids.data(), total, counts.data(),
                             &total));
  uint64_t at = 0;
  for (uint32_t k = 0; k < ckpt.wsparse; ++k) {
    ConversionStep st;
    st.record_index = k;
    st.replay_iteration = ckpt.window_start + k + 1;
    st.activating.assign(ids.begin() + static_cast<long>(at), ids.begin() + static_cast<long>(at + counts[k]));
    at += counts[k];
    cp.steps.push_back(std::move(st));
  }
  return cp;
}

// "One persisted checkpoint and another in flight, garbage-collecting the
// oldest after persisting a new one".  Records go to the window
// of their state index (capture_windows, verify.hpp:63-84).
class WindowRing {
 public:
  WindowRing(uint32_t wsparse, int32_t replication_target) : w_(wsparse), target_(replication_target) {}
  uint64_t window_of(uint64_t state_index) const { return state_index / w_ * w_; }
  SparseCheckpoint& add_record(uint64_t state_index, DeviceBlob blob) {
    const uint64_t ws = window_of(state_index);
    if (persisted_ && ws <= persisted_->window_start)
      throw std::runtime_error("record for window " + std::to_string(ws) +
                               " is older than the persisted window");
    auto it = in_flight_.find(ws);
    if (it == in_flight_.end()) {
      SparseCheckpoint ck;
      ck.window_start = ws;
      ck.wsparse = w_;
      ck.replication_target = target_;
      it = in_flight_.emplace(ws, std::move(ck)).first;
    }
    SparseCheckpoint& ck = it->second;
    if (ck.complete()) throw std::runtime_error("sparse checkpoint window is full");
    ck.blobs.push_back(std::move(blob));
    ck.replication.push_back(0);
    return ck;
  }
  // Returns the new persisted window start when a window persisted (the
  // caller's gc_logs point), after releasing the windows it replaces.
  std::optional<uint64_t> poll() {
    std::optional<uint64_t> newest;
    for (auto& [ws, ck] : in_flight_) {
      ck.poll_replication();
      if (ck.persisted()) newest = ws;
    }
    if (!newest) return std::nullopt;
    persisted_ = std::move(in_flight_.at(*newest));
    in_flight_.erase(in_flight_.begin(), in_flight_.upper_bound(*newest));
    return newest;
  }
  const SparseCheckpoint* persisted() const { return persisted_ ? &*persisted_ : nullptr; }
  size_t in_flight() const { return in_flight_.size(); }
  SparseCheckpoint* window(uint64_t window_start) {
    auto it = in_flight_.find(window_start);
    return it == in_flight_.end() ? nullptr : &it->second;
  }

 private:
  uint32_t w_;
  int32_t target_;
  std::optional<SparseCheckpoint> persisted_;
  std::map<uint64_t, SparseCheckpoint> in_flight_;
};

// ---- dense checkpoint (snapshot.hpp:245-295) --------------------------------
inline std::vector<uint8_t> take_dense_checkpoint_bytes(const DeviceState& st) {
  DeviceBlob b(st.context());
  check(mlck_dense_checkpoint(st.get(), b.get()));
  return b.bytes();
}

// ---- gradient log (Adam-replay input) ----------------------------------------
class GradientLog {
 public:
  GradientLog(Context& ctx, std::vector<uint64_t> param_counts, uint32_t capacity_iterations)
      : pc_(std::move(param_counts)) {
    check(mlck_gradlog_create(ctx.get(), static_cast<uint32_t>(pc_.size()), pc_.data(),
                              capacity_iterations, &h_));
  }
  ~GradientLog() {
    if (h_) mlck_gradlog_destroy(h_);
  }
  GradientLog(const GradientLog&) = delete;
  mlck_gradlog* get() const { return h_; }
  void put(uint64_t iteration, uint32_t op, std::span<const float> grad) {
    if (grad.size() != pc_.at(op)) throw std::invalid_argument("adam: shape mismatch");
    check(mlck_gradlog_put(h_, iteration, op, grad.data()));
  }

 private:
  std::vector<uint64_t> pc_;
  mlck_gradlog* h_ = nullptr;
};

// ---- sparse-to-dense conversion (recovery.hpp:180-227) ----------------------
// Result lands in `out` (a DeviceState sized like the model): the TrainState
// the reference returns by value.
inline void sparse_to_dense_convert(DeviceState& out, const SparseCheckpoint& ckpt,
                                    GradientLog* grads, uint64_t data_seed,
                                    const OptimizerConfig& oc = {}) {
  std::vector<mlck_blob*> hs;
  for (const auto& b : ckpt.blobs) hs.push_back(b.get());
  const mlck_optimizer o = oc.abi();
  check(mlck_sparse_to_dense_convert(out.get(), hs.data(), static_cast<uint32_t>(hs.size()),
                                     ckpt.window_start, ckpt.wsparse, data_seed,
                                     grads ? grads->get() : nullptr, &o));
}

// ---- localized recovery (recovery.hpp:240-289) ------------------------------
// The reference's RecoverySegment names the failed stages; the caller passes
// their operators (Engine::stage_of_op in [stage_lo, stage_hi]).  The
// recovered operators land in `out`; the result mirrors
// LocalizedRecoveryResult (the scope's operator states and the iteration).
struct LocalizedRecoveryResult {
  std::map<uint32_t, OperatorState> ops;
  uint64_t iteration = 0;
};
inline LocalizedRecoveryResult localized_recover(DeviceState& out, const std::vector<uint32_t>& scope_ops,
                                                 const SparseCheckpoint& ckpt, GradientLog* grads,
                                                 uint64_t data_seed, uint64_t target_iteration,
                                                 const OptimizerConfig& oc = {}) {
  std::vector<mlck_blob*> hs;
  for (const auto& b : ckpt.blobs) hs.push_back(b.get());
  const mlck_optimizer o = oc.abi();
  check(mlck_localized_recover(out.get(), scope_ops.data(), static_cast<uint32_t>(scope_ops.size()), hs.data(),
                               static_cast<uint32_t>(hs.size()), ckpt.window_start, ckpt.wsparse, data_seed,
                               grads ? grads->get() : nullptr, target_iteration, &o));
  LocalizedRecoveryResult r;
  uint64_t it = 0, seed = 0;
  check(mlck_state_get_meta(out.get(), &it, &seed));
  r.iteration = it;
  for (uint32_t id : scope_ops) r.ops.emplace(id, out.op(id));
  return r;
}

// ---- optimizer (engine.hpp:738-753) ---------------------------------------
// Device spans; `step` is incremented before the bias corrections.
inline void optimizer_step_adam(Context& ctx, float* master, float* m, float* v, uint64_t& step,
                                const float* grad, uint64_t n, const OptimizerConfig& oc) {
  const mlck_optimizer o = oc.abi();
  check(mlck_optimizer_step_adam(ctx.get(), master, m, v, &step, grad, n, &o));
}

// ---- upstream boundary log (engine.hpp:55-94) -------------------------------
struct LogKey {
  uint64_t iteration;
  uint32_t micro_batch;
  uint32_t boundary;
  uint8_t direction;
  auto operator<=>(const LogKey&) const = default;
};

class UpstreamLog {
 public:
  // kind 0: pinned host ring; 1: device ring on `device` (peer over NVLink)
  UpstreamLog(Context& ctx, uint64_t capacity_bytes, int kind = 0, int device = 0) {
    check(mlck_log_create(ctx.get(), kind, device, capacity_bytes, &h_));
  }
  ~UpstreamLog() {
    if (h_) mlck_log_destroy(h_);
  }
  UpstreamLog(const UpstreamLog&) = delete;
  mlck_log* get() const { return h_; }

  static int32_t owner_stage(const LogKey& k) {
    return k.direction == 0 ? static_cast<int32_t>(k.boundary)
                            : static_cast<int32_t>(k.boundary) + 1;
  }
  // entries[k] = tensor (engine.hpp:384-385, 408-409), device source
  void put(const LogKey& k, const float* device_src, uint64_t n) {
    check(mlck_log_put(h_, k.iteration, k.micro_batch, k.boundary, k.direction, device_src, n));
  }
  std::vector<float> at(const LogKey& k) const {
    uint64_t n = 0;
    check(mlck_log_get(h_, k.iteration, k.micro_batch, k.boundary, k.direction, nullptr, 0, &n));
    std::vector<float> out(n);
    check(mlck_log_get(h_, k.iteration, k.micro_batch, k.boundary, k.direction, out.data(), n, &n));
    return out;
  }
  size_t size() const { return mlck_log_count(h_); }
  size_t bytes() const { return mlck_log_bytes(h_); }
  std::map<LogKey, std::vector<float>> entries() const {
    std::map<LogKey, std::vector<float>> out;
    for (uint64_t i = 0; i < size(); ++i) {
      LogKey k{};
      uint64_t n = 0;
      check(mlck_log_entry(h_, i, &k.iteration, &k.micro_batch, &k.boundary, &k.direction, nullptr,
                           0, &n));
      std::vector<float> d(n);
      check(mlck_log_entry(h_, i, &k.iteration, &k.micro_batch, &k.boundary, &k.direction,
                           d.data(), n, &n));
      out.emplace(k, std::move(d));
    }
    return out;
  }
  void sync() const { check(mlck_log_sync(h_)); }
  // ASYNC mode: put() leaves the producer stream free; the caller fences the
  // stream that will overwrite a logged source (mlck_b200.h, mlck_log_put)
  void set_async(bool on) const { check(mlck_log_set_async(h_, on ? 1 : 0)); }
  void fence(void* stream = nullptr) const { check(mlck_log_fence(h_, stream)); }

 private:
  mlck_log* h_ = nullptr;
};

inline void gc_logs(UpstreamLog& log, uint64_t persisted_window_start) {
  check(mlck_gc_logs(log.get(), persisted_window_start));
}

// ---- the miniature MoE trainer on the GPU (engine.hpp:150-730) ----------------
// EngineConfig's fields as the C ABI's mlck_engine_config (params < 0 =
// derived).  run_iteration produces the boundary log and the weight-gradient
// log (zero-copy: the gradients land in the log's slots); the recompute
// conversion / localized recovery replay iterations by forward + backward.
class Engine {
 public:
  Engine(Context& ctx, const mlck_engine_config& cfg) : ctx_(&ctx) { check(mlck_engine_create(ctx.get(), &cfg, &h_)); }
  ~Engine() {
    if (h_) mlck_engine_destroy(h_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  mlck_engine* get() const { return h_; }
  std::vector<uint64_t> param_counts() const {
    std::vector<uint64_t> p(mlck_engine_op_count(h_));
    check(mlck_engine_param_counts(h_, p.data()));
    return p;
  }
  int32_t stage_of_op(uint32_t id) const { return mlck_engine_stage_of_op(h_, id); }
  // Engine::run_iteration(modes, log) (engine.hpp:189-207); frozen: n_ops flags or empty
  void run_iteration(DeviceState& st, const std::vector<uint8_t>& frozen = {}, UpstreamLog* log = nullptr,
                     GradientLog* grads = nullptr) {
    check(mlck_engine_run_iteration(h_, st.get(), frozen.empty() ? nullptr : frozen.data(),
                                    log ? log->get() : nullptr, grads ? grads->get() : nullptr));
  }
  // sparse_to_dense_convert(engine, ckpt) with the reference's recompute replay
  void sparse_to_dense_convert(DeviceState& out, const SparseCheckpoint& ckpt, uint64_t data_seed) {
    std::vector<mlck_blob*> hs;
    for (const auto& b : ckpt.blobs) hs.push_back(b.get());
    check(mlck_sparse_to_dense_convert_recompute(h_, out.get(), hs.data(), static_cast<uint32_t>(hs.size()),
                                                 ckpt.window_start, ckpt.wsparse, data_seed));
  }

 private:
  Context* ctx_;
  mlck_engine* h_ = nullptr;
};

// ---- localized_recover(engine, segment, ckpt, logs, target) ----------------
// (recovery.hpp:240-289) with the reference's own scope vocabulary: the
// failed stage range of one pipeline (RecoverySegment, recovery.hpp:29-41)
// and Engine::stage_of_op (stage_of_ops above).  The boundary tensors the
// segment consumes must be in `logs` (checked per replayed iteration and
// micro-batch, "upstream log missing entry: ..."); the optimizer steps come
// from the gradient log.
struct RecoverySegment {
  int32_t pipeline = 0;
  int32_t stage_lo = 0;
  int32_t stage_hi = 0;
  std::optional<int32_t> upstream_log_owner;
  std::optional<int32_t> downstream_log_owner;
};
inline LocalizedRecoveryResult localized_recover(DeviceState& out, const RecoverySegment& seg,
                                                 const SparseCheckpoint& ckpt, const UpstreamLog& logs,
                                                 GradientLog* grads, const std::vector<int32_t>& stage_of_op,
                                                 const ParallelPlan& plan, uint64_t data_seed,
                                                 uint64_t target_iteration, const OptimizerConfig& oc = {}) {
  if (stage_of_op.size() != out.op_count()) throw std::invalid_argument("stage_of_op: one entry per operator");
  std::vector<mlck_blob*> hs;
  for (const auto& b : ckpt.blobs) hs.push_back(b.get());
  const mlck_optimizer o = oc.abi();
  check(mlck_localized_recover_segment(out.get(), seg.stage_lo, seg.stage_hi, stage_of_op.data(), plan.pp_stages,
                                       hs.data(), static_cast<uint32_t>(hs.size()), ckpt.window_start, ckpt.wsparse,
                                       data_seed, logs.get(),
                                       static_cast<uint32_t>(plan.dp_degree * plan.microbatches),
                                       grads ? grads->get() : nullptr, target_iteration, &o));
  LocalizedRecoveryResult r;
  uint64_t it = 0, seed = 0;
  check(mlck_state_get_meta(out.get(), &it, &seed));
  r.iteration = it;
  for (uint32_t id = 0; id < out.op_count(); ++id)
    if (stage_of_op[id] >= seg.stage_lo && stage_of_op[id] <= seg.stage_hi) r.ops.emplace(id, out.op(id));
  return r;
}

}  // namespace moelab_b200
