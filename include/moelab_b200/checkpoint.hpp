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

 private:
  mlck_ctx* h_ = nullptr;
};

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
  std::vector<mlck_entry_info> ents(1 << 16);
  uint32_t n = 0;
  const int cb = static_cast<int>(plan.compute_bytes);
  check(mlck_parse_record(blob.get(), cb, &info, ents.data(),
                          static_cast<uint32_t>(ents.size()), &n));
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

 private:
  mlck_log* h_ = nullptr;
};

inline void gc_logs(UpstreamLog& log, uint64_t persisted_window_start) {
  check(mlck_gc_logs(log.get(), persisted_window_start));
}

}  // namespace moelab_b200
