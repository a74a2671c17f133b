// ref_shim.cpp -- C-ABI driver over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile straight from
// /root/reference/proj/include (never copied) into oracle/_ref/libmoelab_ref.so.
// It exposes the reference's own checkpoint functions to the Python tests,
// the golden-vector generator (tests/golden/make_golden.py) and bench.py's
// reference arm / cpu_baseline leg.  Nothing in paper_2412_15411_b200/ links it.
//
// Every entry point catches the reference's exceptions and returns -1 with the
// exception text in the caller's buffer, so tests can match the reference's
// error substrings.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "moelab/recovery.hpp"
#include "moelab/schedule.hpp"
#include "moelab/sim.hpp"
#include "moelab/snapshot.hpp"
#include "moelab/verify.hpp"

using namespace moelab;

extern "C" {

// Flat engine configuration (engine.hpp:96-124, core.hpp:66-191).
struct mlr_config {
  int32_t layers, experts_per_layer, top_k, shared_experts;
  int32_t token_dim, expert_hidden, nonexpert_hidden, residual;
  int64_t expert_params, nonexpert_params, gate_params;  // <0 = derived
  int64_t compute_bytes;
  int32_t pp_stages, dp_degree, microbatches;
  int64_t microbatch_size, global_batch;
  int32_t optimizer_kind;  // 0 adam 1 sgd
  float lr, beta1, beta2, eps;
  uint64_t seed;
};
}

namespace {

thread_local std::string g_err;

EngineConfig to_cfg(const mlr_config* c) {
  EngineConfig cfg;
  cfg.model.layers = c->layers;
  cfg.model.experts_per_layer = c->experts_per_layer;
  cfg.model.top_k = c->top_k;
  cfg.model.shared_experts = c->shared_experts;
  cfg.model.token_dim = c->token_dim;
  cfg.model.expert_hidden = c->expert_hidden;
  cfg.model.nonexpert_hidden = c->nonexpert_hidden;
  cfg.model.residual = c->residual != 0;
  if (c->expert_params >= 0) cfg.model.expert_params = c->expert_params;
  if (c->nonexpert_params >= 0) cfg.model.nonexpert_params = c->nonexpert_params;
  if (c->gate_params >= 0) cfg.model.gate_params = c->gate_params;
  cfg.precision.compute_bytes = c->compute_bytes;
  cfg.parallel.pp_stages = c->pp_stages;
  cfg.parallel.dp_degree = c->dp_degree;
  cfg.parallel.microbatches = c->microbatches;
  cfg.parallel.microbatch_size = c->microbatch_size;
  cfg.parallel.global_batch = c->global_batch;
  cfg.optimizer.kind = c->optimizer_kind == 0 ? OptimizerConfig::Kind::Adam
                                              : OptimizerConfig::Kind::Sgd;
  cfg.optimizer.lr = c->lr;
  cfg.optimizer.beta1 = c->beta1;
  cfg.optimizer.beta2 = c->beta2;
  cfg.optimizer.eps = c->eps;
  cfg.seed = c->seed;
  return cfg;
}

template <typename F>
int guarded(char* err, size_t cap, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  if (err && cap) std::snprintf(err, cap, "%s", g_err.c_str());
  return -1;
}

size_t copy_out(const std::vector<uint8_t>& v, uint8_t* out, size_t cap) {
  if (out && cap >= v.size()) std::memcpy(out, v.data(), v.size());
  return v.size();
}

}  // namespace

extern "C" {

const char* mlr_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- engine
void* mlr_engine_create(const mlr_config* c, char* err, size_t cap) {
  Engine* e = nullptr;
  if (guarded(err, cap, [&] { e = new Engine(to_cfg(c)); }) != 0) return nullptr;
  return e;
}
void mlr_engine_destroy(void* e) { delete static_cast<Engine*>(e); }

int mlr_engine_run_iteration(void* e, void* log, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    static_cast<Engine*>(e)->run_iteration(nullptr, static_cast<UpstreamLog*>(log));
  });
}
uint64_t mlr_engine_iteration(void* e) { return static_cast<Engine*>(e)->state().iteration; }
uint64_t mlr_engine_data_seed(void* e) { return static_cast<Engine*>(e)->state().data_seed; }
uint32_t mlr_engine_op_count(void* e) {
  return static_cast<uint32_t>(static_cast<Engine*>(e)->operators().size());
}
int64_t mlr_engine_param_count(void* e, uint32_t id) {
  return static_cast<Engine*>(e)->operators().at(id).param_count;
}
// Current vector length of an operator's state (differs from param_count
// after mlr_engine_set_op planted a synthetic payload).
uint64_t mlr_engine_op_size(void* e, uint32_t id) {
  return static_cast<Engine*>(e)->state().ops.at(id).master.size();
}
int32_t mlr_engine_stage_of_op(void* e, uint32_t id) {
  return static_cast<Engine*>(e)->stage_of_op(id);
}

// Copies one operator's state out; arrays sized param_count.
int mlr_engine_get_op(void* e, uint32_t id, float* master, float* m, float* v, uint64_t* step,
                      float* compute, int32_t* has_full) {
  const auto& op = static_cast<Engine*>(e)->state().ops.at(id);
  if (master) std::memcpy(master, op.master.data(), op.master.size() * 4);
  if (m) std::memcpy(m, op.m.data(), op.m.size() * 4);
  if (v) std::memcpy(v, op.v.data(), op.v.size() * 4);
  if (compute) std::memcpy(compute, op.compute.data(), op.compute.size() * 4);
  if (step) *step = op.step;
  if (has_full) *has_full = op.has_full_state ? 1 : 0;
  return 0;
}

// Overwrites one operator (sizes may change: used to plant large synthetic
// payloads into a small engine for timing).  compute = quantize(master).
int mlr_engine_set_op(void* e, uint32_t id, const float* master, const float* m, const float* v,
                      uint64_t n, uint64_t step, int32_t has_full) {
  auto* eng = static_cast<Engine*>(e);
  auto& op = eng->mutable_state().ops.at(id);
  op.master.assign(master, master + n);
  op.m.assign(m, m + n);
  op.v.assign(v, v + n);
  op.step = step;
  op.has_full_state = has_full != 0;
  op.refresh_compute(static_cast<int>(eng->config().precision.compute_bytes));
  return 0;
}

void mlr_engine_set_iteration(void* e, uint64_t it) {
  static_cast<Engine*>(e)->mutable_state().iteration = it;
}

size_t mlr_engine_serialize_state(void* e, uint8_t* out, size_t cap) {
  return copy_out(static_cast<Engine*>(e)->serialize_state(), out, cap);
}

// Per-operator gradients of iteration state.iteration+1 through the public
// API: clone the state into an engine with beta1 = 0 and
// lr = 0 and zeroed m, run one iteration, read m (== g; -0 reads as +0).
int mlr_engine_extract_grads(void* e, float** out_per_op, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto* src = static_cast<Engine*>(e);
    EngineConfig cfg = src->config();
    cfg.optimizer.kind = OptimizerConfig::Kind::Adam;
    cfg.optimizer.beta1 = 0.0f;
    cfg.optimizer.lr = 0.0f;
    Engine probe(cfg);
    probe.mutable_state() = src->state();
    for (auto& op : probe.mutable_state().ops) std::fill(op.m.begin(), op.m.end(), 0.0f);
    probe.run_iteration();
    for (size_t id = 0; id < probe.state().ops.size(); ++id) {
      const auto& m = probe.state().ops[id].m;
      std::memcpy(out_per_op[id], m.data(), m.size() * 4);
    }
  });
}

// ---------------------------------------------------------------- schedule
// order_operators(HardCount) + generate_schedule(W, O) (schedule.hpp:41-80,
// 153-172).  For slot k writes active ids then compute-only ids into
// ids[k*n_ops ...]; counts into n_active[k], n_co[k].
int mlr_schedule(void* e, int64_t wsparse, int64_t o_active, uint32_t* ids, uint32_t* n_active,
                 uint32_t* n_co, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto* eng = static_cast<Engine*>(e);
    const auto ordered = order_operators(eng->descriptors_with_popularity(),
                                         OrderingScheme::HardCount);
    const auto s = generate_schedule(ordered, wsparse, o_active, OrderingScheme::HardCount);
    const size_t n = eng->operators().size();
    for (size_t k = 0; k < s.slots.size(); ++k) {
      const auto& sl = s.slots[k];
      n_active[k] = static_cast<uint32_t>(sl.active.size());
      n_co[k] = static_cast<uint32_t>(sl.compute_only.size());
      uint32_t* dst = ids + k * n;
      for (uint32_t id : sl.active) *dst++ = id;
      for (uint32_t id : sl.compute_only) *dst++ = id;
    }
  });
}

// build_schedule (schedule.hpp:177-209) over explicit descriptors: cls[i]
// 0 expert / 1 non-expert / 2 gate, hard/soft/ema popularity, capacity.
// Writes W, O, fits and the slot layout like mlr_schedule (ids sized
// max_slots * n).
int mlr_build_schedule(uint32_t n, const uint8_t* cls, const int64_t* params, const double* hard,
                       const double* soft, const double* ema, const double* capacity, int64_t compute_bytes,
                       int64_t master_bytes, int64_t optimizer_bytes, double bandwidth, double t_iter,
                       int ordering, int allow_single, int64_t max_slots, int64_t* wsparse, int64_t* o_active,
                       int32_t* fits, uint32_t* ids, uint32_t* n_active, uint32_t* n_co, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    std::vector<OperatorDescriptor> ops(n);
    for (uint32_t i = 0; i < n; ++i) {
      ops[i].id = i;
      ops[i].cls = static_cast<OperatorClass>(cls[i]);
      ops[i].param_count = params[i];
      ops[i].capacity = capacity[i];
      ops[i].popularity.hard_count = hard[i];
      ops[i].popularity.soft_count = soft[i];
      ops[i].popularity.ema = ema[i];
    }
    PrecisionPlan plan;
    plan.compute_bytes = compute_bytes;
    plan.master_bytes = master_bytes;
    plan.optimizer_bytes = optimizer_bytes;
    const auto s = build_schedule(ops, plan, bandwidth, t_iter, static_cast<OrderingScheme>(ordering),
                                  allow_single != 0);
    *wsparse = s.wsparse;
    *o_active = s.o_active;
    *fits = s.fits_budget ? 1 : 0;
    if (static_cast<int64_t>(s.slots.size()) > max_slots) throw std::runtime_error("too many slots");
    for (size_t k = 0; k < s.slots.size(); ++k) {
      const auto& sl = s.slots[k];
      n_active[k] = static_cast<uint32_t>(sl.active.size());
      n_co[k] = static_cast<uint32_t>(sl.compute_only.size());
      uint32_t* dst = ids + k * n;
      for (uint32_t id : sl.active) *dst++ = id;
      for (uint32_t id : sl.compute_only) *dst++ = id;
    }
  });
}

// ---------------------------------------------------------------- snapshot
// serialize_record(take_sparse_snapshot(engine, slot, slot_index), ...)
// (snapshot.hpp:204-241, 115-144).  Returns the blob size (writes when cap
// suffices) or -1.
int64_t mlr_snapshot(void* e, const uint32_t* active, uint32_t n_active, const uint32_t* co,
                     uint32_t n_co, uint32_t slot_index, uint8_t kind, uint64_t window_start,
                     uint32_t wsparse, uint8_t* out, size_t cap, char* err, size_t ecap) {
  int64_t size = -1;
  guarded(err, ecap, [&] {
    auto* eng = static_cast<Engine*>(e);
    ScheduleSlot slot;
    slot.active.assign(active, active + n_active);
    slot.compute_only.assign(co, co + n_co);
    const SnapshotRecord rec = take_sparse_snapshot(*eng, slot, slot_index);
    const auto blob = serialize_record(rec, eng->config().precision, kind, window_start, wsparse);
    size = static_cast<int64_t>(copy_out(blob, out, cap));
  });
  return size;
}

// take_dense_checkpoint(engine).serialize(plan) (snapshot.hpp:245-295).
int64_t mlr_dense_checkpoint(void* e, uint8_t* out, size_t cap, char* err, size_t ecap) {
  int64_t size = -1;
  guarded(err, ecap, [&] {
    auto* eng = static_cast<Engine*>(e);
    const auto ck = take_dense_checkpoint(*eng);
    size = static_cast<int64_t>(copy_out(ck.serialize(eng->config().precision), out, cap));
  });
  return size;
}

// parse_record (snapshot.hpp:153-197); returns entry count or -1.
int64_t mlr_parse_record(const uint8_t* blob, size_t n, int64_t compute_bytes, uint64_t* iteration,
                         uint32_t* slot, char* err, size_t ecap) {
  int64_t count = -1;
  guarded(err, ecap, [&] {
    PrecisionPlan plan;
    plan.compute_bytes = compute_bytes;
    const auto pr = parse_record(std::span<const uint8_t>(blob, n), plan);
    if (iteration) *iteration = pr.record.iteration;
    if (slot) *slot = pr.record.slot;
    count = static_cast<int64_t>(pr.record.entries.size());
  });
  return count;
}

// ---------------------------------------------------------------- conversion
// sparse_to_dense_convert(Engine(cfg), ckpt) (recovery.hpp:180-227).  Writes
// serialize_state of the result.  blobs are W concatenated records.
int64_t mlr_convert(const mlr_config* c, uint64_t window_start, uint32_t wsparse,
                    const uint8_t* const* blobs, const uint64_t* sizes, uint32_t n_blobs,
                    uint8_t* out, size_t cap, char* err, size_t ecap) {
  int64_t size = -1;
  guarded(err, ecap, [&] {
    SparseCheckpoint ckpt;
    ckpt.window_start = window_start;
    ckpt.wsparse = wsparse;
    for (uint32_t k = 0; k < n_blobs; ++k) {
      ckpt.blobs.emplace_back(blobs[k], blobs[k] + sizes[k]);
      ckpt.replication.push_back(0);
    }
    Engine scratch(to_cfg(c));
    const TrainState st = sparse_to_dense_convert(scratch, ckpt);
    size = static_cast<int64_t>(copy_out(Engine::serialize_state(st), out, cap));
  });
  return size;
}

// localized_recover(Engine(cfg), {pipeline 0, stage_lo, stage_hi}, ckpt, log,
// target) (recovery.hpp:240-289).  Writes the "scope image": u64 iteration,
// u32 n_ops, then per recovered operator in id order: u32 id, u64 step,
// u64 P, f32 master[P], m[P], v[P].
int64_t mlr_localized_recover(const mlr_config* c, uint64_t window_start, uint32_t wsparse,
                              const uint8_t* const* blobs, const uint64_t* sizes, uint32_t n_blobs,
                              void* log, int32_t stage_lo, int32_t stage_hi, uint64_t target,
                              uint8_t* out, size_t cap, char* err, size_t ecap) {
  int64_t size = -1;
  guarded(err, ecap, [&] {
    SparseCheckpoint ckpt;
    ckpt.window_start = window_start;
    ckpt.wsparse = wsparse;
    for (uint32_t k = 0; k < n_blobs; ++k) {
      ckpt.blobs.emplace_back(blobs[k], blobs[k] + sizes[k]);
      ckpt.replication.push_back(0);
    }
    Engine scratch(to_cfg(c));
    RecoverySegment seg;
    seg.stage_lo = stage_lo;
    seg.stage_hi = stage_hi;
    const LocalizedRecoveryResult r =
        localized_recover(scratch, seg, ckpt, *static_cast<const UpstreamLog*>(log), target);
    ByteWriter w;
    w.value<uint64_t>(r.iteration);
    w.value<uint32_t>(static_cast<uint32_t>(r.ops.size()));
    for (const auto& [id, op] : r.ops) {
      w.value<uint32_t>(id);
      w.value<uint64_t>(op.step);
      w.value<uint64_t>(op.master.size());
      w.floats(op.master);
      w.floats(op.m);
      w.floats(op.v);
    }
    size = static_cast<int64_t>(copy_out(w.buf, out, cap));
  });
  return size;
}

// conversion_plan(ckpt, plan) (recovery.hpp:123-137): counts[k] = the
// activating ids of step k, concatenated into ids (cap entries); returns the
// total, -1 on error.
int64_t mlr_conversion_plan(uint64_t window_start, uint32_t wsparse, const uint8_t* const* blobs,
                            const uint64_t* sizes, uint32_t n_blobs, int64_t compute_bytes, uint32_t* ids,
                            size_t cap, uint64_t* counts, uint64_t* replay_iterations, char* err, size_t ecap) {
  int64_t total = -1;
  guarded(err, ecap, [&] {
    SparseCheckpoint ckpt;
    ckpt.window_start = window_start;
    ckpt.wsparse = wsparse;
    for (uint32_t k = 0; k < n_blobs; ++k) ckpt.blobs.emplace_back(blobs[k], blobs[k] + sizes[k]);
    PrecisionPlan plan;
    plan.compute_bytes = compute_bytes;
    const ConversionPlan cp = conversion_plan(ckpt, plan);
    size_t w = 0;
    for (size_t k = 0; k < cp.steps.size(); ++k) {
      counts[k] = cp.steps[k].activating.size();
      replay_iterations[k] = cp.steps[k].replay_iteration;
      for (uint32_t id : cp.steps[k].activating) {
        if (w < cap) ids[w] = id;
        ++w;
      }
    }
    total = static_cast<int64_t>(w);
  });
  return total;
}

// run_simulation (sim.hpp:246-597) for the sparse policy with Poisson
// failures: out[] = wsparse, t_iter, iterations, failures, useful, stall,
// recovery, idle, wall, ettr, overhead_s_per_iter, recovery_recompute_s,
// max_recovery_event_s, mean_recovery_event_s, checkpoint_never_persisted.
int mlr_run_simulation_sparse(int32_t layers, int32_t experts, int64_t expert_params, int64_t nonexpert_params,
                              int64_t gate_params, int64_t tokens_per_sample, int32_t nodes, double pcie,
                              double replication_bw, int32_t pp_stages, int32_t microbatches, int64_t global_batch,
                              const double* t_stage, int32_t n_stage, double t_sync, double t_update,
                              double t_iter_override, int32_t upstream_logging, int32_t savings, double mtbf,
                              double horizon, double t_restart, double detection_delay, int32_t replication_r,
                              uint64_t seed, double* out, char* err, size_t ecap) {
  return guarded(err, ecap, [&] {
    SimConfig cfg;
    cfg.model.layers = layers;
    cfg.model.experts_per_layer = experts;
    cfg.model.top_k = 1;
    cfg.model.expert_params = expert_params;
    cfg.model.nonexpert_params = nonexpert_params;
    cfg.model.gate_params = gate_params;
    cfg.model.tokens_per_sample = tokens_per_sample;
    cfg.cluster.nodes = nodes;
    cfg.cluster.pcie_bandwidth = pcie;
    cfg.cluster.replication_bandwidth = replication_bw;
    cfg.parallel.pp_stages = pp_stages;
    cfg.parallel.microbatches = microbatches;
    cfg.parallel.global_batch = global_batch;
    cfg.profile.t_stage.assign(t_stage, t_stage + n_stage);
    cfg.profile.t_sync = t_sync;
    cfg.profile.t_update = t_update;
    cfg.profile.t_iter_override = t_iter_override;
    cfg.policy.kind = PolicyKind::Sparse;
    cfg.policy.upstream_logging = upstream_logging != 0;
    cfg.policy.conversion_compute_savings = savings != 0;
    cfg.failures.kind = FailureProcess::Kind::Poisson;
    cfg.failures.mtbf = mtbf;
    cfg.horizon = horizon;
    cfg.t_restart = t_restart;
    cfg.detection_delay = detection_delay;
    cfg.replication_r = replication_r;
    cfg.seed = seed;
    const Metrics m = run_simulation(cfg);
    const double v[] = {m.wsparse_or_interval, m.t_iter, static_cast<double>(m.iterations),
                        static_cast<double>(m.failures), m.useful_s, m.stall_s, m.recovery_s, m.idle_s, m.wall_s,
                        m.ettr, m.overhead_s_per_iter, m.recovery_recompute_s, m.max_recovery_event_s,
                        m.mean_recovery_event_s, m.checkpoint_never_persisted ? 1.0 : 0.0};
    std::memcpy(out, v, sizeof(v));
  });
}

// check_log_budget(model, plan, wsparse, cluster) (recovery.hpp:308-317).
int mlr_check_log_budget(const mlr_config* c, int64_t wsparse, double cpu_mem_per_node, int32_t nodes,
                         char* err, size_t ecap) {
  return guarded(err, ecap, [&] {
    const EngineConfig cfg = to_cfg(c);
    ClusterSpec cl;
    cl.cpu_mem_per_node = cpu_mem_per_node;
    cl.nodes = nodes;
    check_log_budget(cfg.model, cfg.parallel, wsparse, cl);
  });
}

// SparseCheckpoint::check_coverage (snapshot.hpp:322-334).
int mlr_check_coverage(uint32_t wsparse, const uint8_t* const* blobs, const uint64_t* sizes,
                       uint32_t n_blobs, uint64_t op_count, int64_t compute_bytes, char* err,
                       size_t ecap) {
  return guarded(err, ecap, [&] {
    SparseCheckpoint ckpt;
    ckpt.wsparse = wsparse;
    for (uint32_t k = 0; k < n_blobs; ++k) ckpt.blobs.emplace_back(blobs[k], blobs[k] + sizes[k]);
    PrecisionPlan plan;
    plan.compute_bytes = compute_bytes;
    ckpt.check_coverage(op_count, plan);
  });
}

// ---------------------------------------------------------------- logging
void* mlr_log_create() { return new UpstreamLog(); }
void mlr_log_destroy(void* l) { delete static_cast<UpstreamLog*>(l); }
uint64_t mlr_log_count(void* l) { return static_cast<UpstreamLog*>(l)->entries.size(); }
uint64_t mlr_log_bytes(void* l) { return static_cast<UpstreamLog*>(l)->bytes(); }
// i-th entry in map order (LogKey ordering, engine.hpp:55-61).
int64_t mlr_log_entry(void* l, uint64_t i, uint64_t* iteration, uint32_t* micro_batch,
                      uint32_t* boundary, uint8_t* direction, float* data, size_t cap_floats) {
  auto* log = static_cast<UpstreamLog*>(l);
  if (i >= log->entries.size()) return -1;
  auto it = log->entries.begin();
  std::advance(it, static_cast<long>(i));
  *iteration = it->first.iteration;
  *micro_batch = it->first.micro_batch;
  *boundary = it->first.boundary;
  *direction = it->first.direction;
  if (data && cap_floats >= it->second.size())
    std::memcpy(data, it->second.data(), it->second.size() * 4);
  return static_cast<int64_t>(it->second.size());
}
void mlr_gc_logs(void* l, uint64_t persisted_window_start) {
  gc_logs(*static_cast<UpstreamLog*>(l), persisted_window_start);
}
int mlr_log_at(void* l, uint64_t iteration, uint32_t mb, uint32_t boundary, uint8_t dir,
               char* err, size_t ecap) {
  return guarded(err, ecap, [&] {
    (void)static_cast<UpstreamLog*>(l)->at({iteration, mb, boundary, dir});
  });
}
int64_t mlr_upstream_log_bytes(const mlr_config* c, int64_t wsparse) {
  const EngineConfig cfg = to_cfg(c);
  return upstream_log_bytes(cfg.model, cfg.parallel, wsparse);
}

// ---------------------------------------------------------------- primitives
uint64_t mlr_fnv1a64(const uint8_t* data, size_t n, uint64_t seed) {
  return fnv1a64(std::span<const uint8_t>(data, n), seed);
}
int mlr_quantize_value(float x, int compute_bytes, float* out, char* err, size_t ecap) {
  return guarded(err, ecap, [&] { *out = quantize_value(x, compute_bytes); });
}
// Array form (no float->double round trip through the caller: keeps
// signalling-NaN payloads exactly as quantize_value returns them).
int mlr_quantize_array(const float* in, size_t n, int compute_bytes, float* out, char* err,
                       size_t ecap) {
  return guarded(err, ecap, [&] {
    for (size_t i = 0; i < n; ++i) out[i] = quantize_value(in[i], compute_bytes);
  });
}
void mlr_unpack_array(const uint16_t* codes, size_t n, int ebits, int mbits, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = unpack_reduced(codes[i], ebits, mbits);
}
uint16_t mlr_pack_reduced(float x, int ebits, int mbits) { return pack_reduced(x, ebits, mbits); }
void mlr_pack_array(const float* x, size_t n, int ebits, int mbits, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = pack_reduced(x[i], ebits, mbits);
}
float mlr_unpack_reduced(uint16_t c, int ebits, int mbits) { return unpack_reduced(c, ebits, mbits); }

int mlr_optimizer_step_adam(float* master, float* m, float* v, uint64_t* step, const float* grad,
                            size_t n, float lr, float b1, float b2, float eps, char* err,
                            size_t ecap) {
  return guarded(err, ecap, [&] {
    std::vector<float> w(master, master + n), mm(m, m + n), vv(v, v + n), g(grad, grad + n);
    OptimizerConfig oc;
    oc.lr = lr;
    oc.beta1 = b1;
    oc.beta2 = b2;
    oc.eps = eps;
    optimizer_step_adam(w, mm, vv, *step, g, oc);
    std::memcpy(master, w.data(), n * 4);
    std::memcpy(m, mm.data(), n * 4);
    std::memcpy(v, vv.data(), n * 4);
  });
}

// ---------------------------------------------------------------- CPU timing
// Reference arm / cpu_baseline for the snapshot path: `threads` independent
// engines (SPEC.md:192 allows independent instances), each holding one shard
// of the slot: n_full operators with full_params params (Full payload) and
// n_co operators with co_params params (ComputeOnly).  Times
// serialize_record(take_sparse_snapshot(...)) `iters` times per thread after
// one warm-up.  Returns blob bytes produced per second (all threads), and the
// per-thread blob size in *blob_bytes.
double mlr_time_pack(uint32_t threads, uint32_t n_full, uint64_t full_params, uint32_t n_co,
                     uint64_t co_params, int64_t compute_bytes, uint32_t iters,
                     uint64_t* blob_bytes, double* seconds) {
  struct Shard {
    std::unique_ptr<Engine> eng;
    ScheduleSlot slot;
  };
  std::vector<Shard> shards(threads);
  auto build = [&](uint32_t t) {
    mlr_config c{};
    c.layers = 1;
    c.experts_per_layer = static_cast<int32_t>(std::max<uint32_t>(1, n_full + n_co));
    c.top_k = 1;
    c.token_dim = 4;
    c.expert_hidden = 4;
    c.nonexpert_hidden = 4;
    c.residual = 1;
    c.expert_params = c.nonexpert_params = c.gate_params = 8;
    c.compute_bytes = compute_bytes;
    c.pp_stages = c.dp_degree = c.microbatches = 1;
    c.microbatch_size = c.global_batch = 1;
    c.lr = 1e-3f;
    c.beta1 = 0.9f;
    c.beta2 = 0.999f;
    c.eps = 1e-8f;
    c.seed = 7 + t;
    shards[t].eng = std::make_unique<Engine>(to_cfg(&c));
    for (uint32_t i = 0; i < n_full + n_co; ++i) {
      const uint64_t n = i < n_full ? full_params : co_params;
      std::vector<float> w(n), mm(n), vv(n);
      for (uint64_t j = 0; j < n; ++j) {
        w[j] = 0.001f * static_cast<float>((j * 2654435761u + i) % 997) - 0.5f;
        mm[j] = 1e-4f * static_cast<float>(j % 13);
        vv[j] = 1e-7f * static_cast<float>(j % 7);
      }
      mlr_engine_set_op(shards[t].eng.get(), i, w.data(), mm.data(), vv.data(), n, 10, 1);
      (i < n_full ? shards[t].slot.active : shards[t].slot.compute_only).push_back(i);
    }
  };
  {
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(build, t);
    for (auto& th : ts) th.join();
  }
  std::vector<uint64_t> sizes(threads, 0);
  auto run = [&](uint32_t t, uint32_t n) {
    const PrecisionPlan& plan = shards[t].eng->config().precision;
    for (uint32_t k = 0; k < n; ++k) {
      const SnapshotRecord rec = take_sparse_snapshot(*shards[t].eng, shards[t].slot, 0);
      const auto blob = serialize_record(rec, plan, 1, 0, 1);
      sizes[t] = blob.size();
    }
  };
  {
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(run, t, 1u);
    for (auto& th : ts) th.join();
  }
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(run, t, iters);
    for (auto& th : ts) th.join();
  }
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t total = 0;
  for (auto s : sizes) total += s;
  if (blob_bytes) *blob_bytes = sizes.empty() ? 0 : sizes[0];
  if (seconds) *seconds = secs;
  return static_cast<double>(total) * iters / secs;
}

// Reference conversion cost on a synthetic window: `threads` independent
// shards, each an op of `params` params whose Full payload is replayed
// `steps` Adam steps via optimizer_step_adam after parse_record of its blob
// (the merge + logged-gradient replay the GPU kernel implements).  Returns
// element-steps per second.
double mlr_time_replay(uint32_t threads, uint64_t params, uint32_t steps, double* seconds) {
  auto work = [&](uint32_t t) {
    std::vector<float> w(params), m(params), v(params), g(params);
    for (uint64_t j = 0; j < params; ++j) {
      w[j] = 0.001f * static_cast<float>((j * 2654435761u + t) % 997) - 0.5f;
      m[j] = 1e-4f * static_cast<float>(j % 13);
      v[j] = 1e-7f * static_cast<float>(j % 7 + 1);
      g[j] = 1e-3f * static_cast<float>(static_cast<int>(j % 21) - 10);
    }
    uint64_t step = 10;
    OptimizerConfig oc;
    for (uint32_t s = 0; s < steps; ++s) optimizer_step_adam(w, m, v, step, g, oc);
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> ts;
  for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(work, t);
  for (auto& th : ts) th.join();
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (seconds) *seconds = secs;
  return static_cast<double>(threads) * params * steps / secs;
}

// Reference conversion on a window of the configs[3] shape, scaled: one
// layer of `experts` experts of expert_params, NE ne_params, G gate_params,
// W = wsparse with o_active Full operators per slot (generate_schedule on
// the id order, schedule.hpp:153-172), records captured the reference's way
// (capture_windows, verify.hpp:63-84) by `threads` independent engines
// (SPEC.md:192).  Times, per thread, after one warm-up:
//   [0] sparse_to_dense_convert(engine, ckpt)  (recovery.hpp:180-227, its
//       recompute replay included);
//   [1] the merge + logged-gradient replay the GPU kernel implements:
//       parse_record of every record, then each operator's Full payload
//       stepped with optimizer_step_adam on its W-k logged gradients.
// secs[0..1] = wall seconds of each (all threads at once); returns the
// Adam element-steps of one window per thread; *blob_bytes = its records.
double mlr_time_convert(uint32_t threads, int32_t experts, int64_t expert_params, int64_t ne_params,
                        int64_t gate_params, uint32_t wsparse, uint32_t o_active, double* secs,
                        uint64_t* blob_bytes) {
  struct Shard {
    std::unique_ptr<Engine> eng;
    SparseCheckpoint ckpt;
    std::vector<std::vector<std::vector<float>>> grads;  // [iteration k][op]
  };
  std::vector<Shard> shards(threads);
  double steps = 0;
  uint64_t bytes = 0;
  auto build = [&](uint32_t t) {
    mlr_config c{};
    c.layers = 1;
    c.experts_per_layer = experts;
    c.top_k = 2;
    c.token_dim = 4;
    c.expert_hidden = 4;
    c.nonexpert_hidden = 4;
    c.residual = 1;
    c.expert_params = expert_params;
    c.nonexpert_params = ne_params;
    c.gate_params = gate_params;
    c.compute_bytes = 2;
    c.pp_stages = c.dp_degree = 1;
    c.microbatches = 2;
    c.microbatch_size = 4;
    c.global_batch = 8;
    c.lr = 1e-3f;
    c.beta1 = 0.9f;
    c.beta2 = 0.999f;
    c.eps = 1e-8f;
    c.seed = 5 + t;
    Shard& sh = shards[t];
    sh.eng = std::make_unique<Engine>(to_cfg(&c));
    std::vector<uint32_t> ordered(sh.eng->operators().size());
    for (uint32_t i = 0; i < ordered.size(); ++i) ordered[i] = i;
    const SparseSchedule sched = generate_schedule(ordered, wsparse, o_active, OrderingScheme::HardCount);
    sh.ckpt.window_start = 0;
    sh.ckpt.wsparse = wsparse;
    const PrecisionPlan& plan = sh.eng->config().precision;
    for (uint32_t k = 0; k < wsparse; ++k) {  // state k -> slot k of window 0
      sh.ckpt.add_record(take_sparse_snapshot(*sh.eng, sched.slots[k], k), plan);
      // the iteration's weight gradients (the logged-replay input): the
      // beta1 = 0, lr = 0 probe of a clone
      mlr_config pc = c;
      pc.beta1 = 0.0f;
      pc.lr = 0.0f;
      Engine probe(to_cfg(&pc));
      probe.mutable_state() = sh.eng->state();
      for (auto& op : probe.mutable_state().ops) std::fill(op.m.begin(), op.m.end(), 0.0f);
      probe.run_iteration();
      std::vector<std::vector<float>> g;
      for (const auto& op : probe.state().ops) g.push_back(op.m);
      sh.grads.push_back(std::move(g));
      sh.eng->run_iteration();
    }
  };
  {
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(build, t);
    for (auto& th : ts) th.join();
  }
  {
    const auto& sh = shards[0];
    for (const auto& b : sh.ckpt.blobs) bytes += b.size();
    const auto ops = sh.eng->operators();
    for (uint32_t k = 0; k < wsparse; ++k) {
      const ParsedRecord pr = parse_record(sh.ckpt.blobs[k], sh.eng->config().precision);
      for (const auto& [id, p] : pr.record.entries)
        if (p.mode == SnapshotMode::Full) steps += static_cast<double>(p.master.size()) * (wsparse - k);
    }
  }
  auto convert = [&](uint32_t t) {
    Shard& sh = shards[t];
    Engine scratch(sh.eng->config());
    const TrainState st = sparse_to_dense_convert(scratch, sh.ckpt);
    (void)st;
  };
  auto replay = [&](uint32_t t) {
    Shard& sh = shards[t];
    const PrecisionPlan& plan = sh.eng->config().precision;
    const OptimizerConfig oc = sh.eng->config().optimizer;
    std::vector<OperatorState> ops(sh.eng->operators().size());
    std::vector<uint32_t> slot_of(ops.size(), 0);
    for (uint32_t k = 0; k < wsparse; ++k) {
      const ParsedRecord pr = parse_record(sh.ckpt.blobs[k], plan);
      for (const auto& [id, p] : pr.record.entries)
        if (p.mode == SnapshotMode::Full) {
          ops[id].master = p.master;
          ops[id].m = p.m;
          ops[id].v = p.v;
          ops[id].step = p.step;
          slot_of[id] = k;
        }
    }
    for (uint32_t id = 0; id < ops.size(); ++id) {
      for (uint32_t k = slot_of[id]; k < wsparse; ++k)
        optimizer_step_adam(ops[id].master, ops[id].m, ops[id].v, ops[id].step, sh.grads[k][id], oc);
      ops[id].refresh_compute(static_cast<int>(plan.compute_bytes));
    }
  };
  auto timed = [&](auto&& fn) {
    std::vector<std::thread> ts;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t t = 0; t < threads; ++t) ts.emplace_back(fn, t);
    for (auto& th : ts) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  timed(convert);  // warm-up
  secs[0] = timed(convert);
  timed(replay);
  secs[1] = timed(replay);
  if (blob_bytes) *blob_bytes = bytes;
  return steps;
}

}  // extern "C"
