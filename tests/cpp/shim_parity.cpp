// shim_parity.cpp -- drives the C++ drop-in (include/moelab_b200) the way the
// reference's own harness drives moelab (TrainRun, test_recovery.cpp:34-67):
// one window of sparse snapshots, coverage check, sparse-to-dense conversion.
// Inputs come from tests/test_cpp_shim.py (golden states/grads of the real
// reference); outputs are written for byte comparison, plus the reference's
// error texts for the failure paths.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "moelab_b200/checkpoint.hpp"

using namespace moelab_b200;

namespace {
struct Reader {
  std::vector<uint8_t> buf;
  size_t pos = 0;
  template <typename T>
  T get() {
    T v;
    std::memcpy(&v, buf.data() + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  void floats(std::vector<float>& v, size_t n) {
    v.resize(n);
    std::memcpy(v.data(), buf.data() + pos, 4 * n);
    pos += 4 * n;
  }
};

void write(const std::string& path, const std::vector<uint8_t>& b) {
  std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(b.data()), b.size());
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: shim_parity <case.bin> <outdir>\n");
    return 2;
  }
  Reader r;
  {
    std::ifstream f(argv[1], std::ios::binary);
    r.buf.assign(std::istreambuf_iterator<char>(f), {});
  }
  const std::string out = argv[2];
  const uint32_t n_ops = r.get<uint32_t>(), cb = r.get<uint32_t>(), W = r.get<uint32_t>();
  const uint64_t data_seed = r.get<uint64_t>(), ws = r.get<uint64_t>();
  OptimizerConfig oc;
  oc.kind = r.get<int32_t>() == 0 ? OptimizerConfig::Kind::Adam : OptimizerConfig::Kind::Sgd;
  oc.lr = r.get<float>();
  oc.beta1 = r.get<float>();
  oc.beta2 = r.get<float>();
  oc.eps = r.get<float>();
  std::vector<uint64_t> P(n_ops);
  for (auto& p : P) p = r.get<uint64_t>();
  PrecisionPlan plan;
  plan.compute_bytes = cb;

  Context ctx(0);
  SparseCheckpoint ckpt;
  ckpt.window_start = ws;
  ckpt.wsparse = W;
  // the same window recovered from replica buffers: each record's witness
  // travels beside its replica, the recovering side wraps both in place
  SparseCheckpoint from_replicas;
  from_replicas.window_start = ws;
  from_replicas.wsparse = W;
  std::vector<void*> rep_buffers;
  std::vector<ScheduleSlot> slots(W);
  for (uint32_t k = 0; k < W; ++k) {
    DeviceState st(ctx, P, static_cast<int>(cb));
    const uint64_t it = r.get<uint64_t>();
    for (uint32_t i = 0; i < n_ops; ++i) {
      OperatorState op;
      op.step = r.get<uint64_t>();
      r.floats(op.master, P[i]);
      r.floats(op.m, P[i]);
      r.floats(op.v, P[i]);
      op.has_full_state = true;
      st.set_op(i, op);
    }
    st.set_meta(it, data_seed);
    auto& sl = slots[k];
    sl.active.resize(r.get<uint32_t>());
    for (auto& id : sl.active) id = r.get<uint32_t>();
    sl.compute_only.resize(r.get<uint32_t>());
    for (auto& id : sl.compute_only) id = r.get<uint32_t>();
    // capture_windows (verify.hpp:75-76)
    ckpt.add_record(take_sparse_snapshot(st, sl, k), plan);
    {
      const uint64_t cap = 1 << 20, wcap = DeviceBlob::witness_bytes(cap);
      void *rep = nullptr, *wit = nullptr;
      check(mlck_device_alloc(ctx.get(), cap, &rep));
      check(mlck_device_alloc(ctx.get(), wcap, &wit));
      rep_buffers.push_back(rep);
      rep_buffers.push_back(wit);
      DeviceBlob sender(ctx, cap);
      sender.add_replica(rep, cap);
      sender.add_replica_witness(wit, wcap);
      serialize_record(take_sparse_snapshot(st, sl, k), plan, 1, ws, W, sender);
      from_replicas.blobs.push_back(DeviceBlob::wrap(ctx, rep, sender.size(), wit));
      from_replicas.replication.push_back(1);
      ctx.synchronize();
    }
    write(out + "/blob_" + std::to_string(k) + ".bin",
          serialize_record(take_sparse_snapshot(st, sl, k), plan, 1, ws, W));
    if (k == 0) {
      // reference error paths (test_snapshot.cpp:198-204, 133-143)
      try {
        ScheduleSlot bad;
        bad.active = {n_ops + 7};
        (void)take_sparse_snapshot(st, bad, 0);
      } catch (const std::invalid_argument& e) {
        std::cout << "ERR invalid_argument: " << e.what() << "\n";
      }
      auto bytes = ckpt.blobs[0].bytes();
      bytes[bytes.size() / 2] ^= 0x40;
      try {
        (void)parse_record(ctx, bytes, plan);
      } catch (const std::runtime_error& e) {
        std::cout << "ERR runtime_error: " << e.what() << "\n";
      }
      const ParsedRecord pr = parse_record(ctx, ckpt.blobs[0].bytes(), plan);
      std::cout << "PARSED iteration " << pr.iteration << " entries " << pr.entries.size() << "\n";
    }
  }
  ckpt.check_coverage(n_ops, plan);
  std::cout << "complete " << ckpt.complete() << " persisted " << ckpt.persisted() << "\n";

  // window durability: files back byte-exact; a window of the
  // ring persists once every record has its copies, here a durable file
  {
    std::filesystem::create_directories(out + "/window");
    ckpt.save(out + "/window");
    SparseCheckpoint back = SparseCheckpoint::load(ctx, out + "/window", ws, W);
    bool same = back.blobs.size() == W;
    for (uint32_t k = 0; same && k < W; ++k) same = back.blobs[k].bytes() == ckpt.blobs[k].bytes();
    back.check_coverage(n_ops, plan);
    std::cout << "SAVED same " << same << " durable_persisted " << back.persisted() << "\n";
    WindowRing ring(W, 1);
    for (uint32_t k = 0; k < W; ++k) ring.add_record(ws + k, DeviceBlob(ctx, ckpt.blobs[k].bytes()));
    const bool before = ring.poll().has_value();
    std::filesystem::create_directories(out + "/ring");
    ring.window(ws)->save(out + "/ring");
    const auto after = ring.poll();
    std::cout << "RING before " << before << " after " << (after ? static_cast<int64_t>(*after) : -1)
              << " in_flight " << ring.in_flight() << "\n";
  }

  GradientLog g(ctx, P, W);
  for (uint32_t s = 1; s <= W; ++s)
    for (uint32_t i = 0; i < n_ops; ++i) {
      std::vector<float> gr;
      r.floats(gr, P[i]);
      g.put(ws + s, i, gr);
    }
  DeviceState conv(ctx, P, static_cast<int>(cb));
  sparse_to_dense_convert(conv, ckpt, &g, data_seed, oc);
  write(out + "/conv.bin", conv.serialize_state());
  {
    uint64_t used0 = 0, fb0 = 0, used = 0, fb = 0;
    check(mlck_ctx_witness_stats(ctx.get(), &used0, &fb0));
    DeviceState conv_rep(ctx, P, static_cast<int>(cb));
    sparse_to_dense_convert(conv_rep, from_replicas, &g, data_seed, oc);
    check(mlck_ctx_witness_stats(ctx.get(), &used, &fb));
    std::cout << "REPLICA_WITNESS same " << (conv_rep.serialize_state() == conv.serialize_state())
              << " witnessed " << (used - used0) << " fallbacks " << (fb - fb0) << "\n";
    from_replicas.blobs.clear();
    for (void* p : rep_buffers) check(mlck_device_free(ctx.get(), p));
  }
  try {
    SparseCheckpoint partial;
    partial.wsparse = W + 1;
    sparse_to_dense_convert(conv, partial, &g, data_seed, oc);
  } catch (const std::runtime_error& e) {
    std::cout << "ERR runtime_error: " << e.what() << "\n";
  }
  // conversion_plan (recovery.hpp:123-137)
  {
    const ConversionPlan cp = conversion_plan(ckpt, plan);
    std::cout << "PLAN " << cp.window_start;
    for (const auto& st : cp.steps) {
      std::cout << " " << st.record_index << ":" << st.replay_iteration << ":";
      for (size_t i = 0; i < st.activating.size(); ++i) std::cout << (i ? "," : "") << st.activating[i];
    }
    std::cout << "\n";
  }
  // scalar codecs (tensor.hpp:99-183), the reference's known answers
  std::cout << "CODEC " << quantize_value(ctx, 65520.0f, 2) << " " << quantize_value(ctx, 300.0f, 1) << " "
            << pack_reduced(ctx, 1.0f, 5, 10) << " " << unpack_reduced(ctx, 0x3c00, 5, 10) << " "
            << pack_reduced(1.5f, 4, 3) << " " << unpack_reduced(static_cast<uint16_t>(0x77), 4, 3) << "\n";
  try {
    (void)quantize_value(ctx, 1.0f, 3);
  } catch (const std::invalid_argument& e) {
    std::cout << "ERR invalid_argument: " << e.what() << "\n";
  }
  // log budget (recovery.hpp:296-317): configs[4] needs 38.65 GB
  {
    ModelSpec m;
    m.token_dim = 2048;
    ParallelPlan pp;
    pp.pp_stages = 4;
    pp.dp_degree = 2;
    pp.microbatches = 8;
    pp.microbatch_size = 4096;
    ClusterSpec cl;
    cl.cpu_mem_per_node = 1e9;
    std::cout << "LOGBYTES " << upstream_log_bytes(m, pp, 6) << "\n";
    try {
      check_log_budget(m, pp, 6, cl);
    } catch (const std::invalid_argument& e) {
      std::cout << "ERR invalid_argument: " << e.what() << "\n";
    }
  }
  // the compiled gradient source: the GPU trainer runs the window itself,
  // its weight gradients landing in the gradient log (no copy); both
  // conversions rebuild its state bit for bit
  if (argc == 3 && n_ops == 18) {  // verify_toy: 3 layers x (4 experts + NE + gate)
    mlck_engine_config ec{};
    ec.layers = 3;
    ec.experts_per_layer = 4;
    ec.top_k = 2;
    ec.token_dim = 4;
    ec.expert_hidden = 4;
    ec.nonexpert_hidden = 4;
    ec.residual = 1;
    ec.expert_params = ec.nonexpert_params = ec.gate_params = -1;
    ec.pp_stages = 3;
    ec.dp_degree = 1;
    ec.microbatches = 2;
    ec.microbatch_size = 4;
    ec.compute_bytes = static_cast<int32_t>(cb);
    ec.optimizer = oc.abi();
    Engine eng(ctx, ec);
    DeviceState run(ctx, P, static_cast<int>(cb));
    for (uint32_t i = 0; i < n_ops; ++i) run.set_op(i, conv.op(i));
    run.set_meta(conv.iteration(), data_seed);
    const uint64_t ws2 = conv.iteration();
    SparseCheckpoint win;
    win.window_start = ws2;
    win.wsparse = W;
    GradientLog g2(ctx, P, W + 1);
    UpstreamLog blog(ctx, 1 << 20);
    for (uint32_t k = 0; k < W; ++k) {
      win.add_record(take_sparse_snapshot(run, slots[k], k), plan);
      eng.run_iteration(run, {}, &blog, &g2);
    }
    DeviceState a(ctx, P, static_cast<int>(cb)), b(ctx, P, static_cast<int>(cb));
    eng.sparse_to_dense_convert(a, win, data_seed);
    sparse_to_dense_convert(b, win, &g2, data_seed, oc);
    const auto want = run.serialize_state();
    std::cout << "ENGINE recompute " << (a.serialize_state() == want) << " logged " << (b.serialize_state() == want)
              << " log_entries " << blog.size() << "\n";
    // localized_recover(engine, RecoverySegment, ckpt, logs, target) for the
    // middle stage, boundary entries from the trainer's own log
    ModelSpec ms;
    ms.layers = 3;
    ms.experts_per_layer = 4;
    ms.token_dim = 4;
    ParallelPlan pp;
    pp.pp_stages = 3;
    pp.dp_degree = 1;
    pp.microbatches = 2;
    pp.microbatch_size = 4;
    const std::vector<int32_t> sop = stage_of_ops(ms, pp);
    RecoverySegment seg;
    seg.stage_lo = seg.stage_hi = 1;
    DeviceState rec(ctx, P, static_cast<int>(cb));
    const LocalizedRecoveryResult lr =
        localized_recover(rec, seg, win, blog, &g2, sop, pp, data_seed, ws2 + W, oc);
    bool same = lr.iteration == ws2 + W && !lr.ops.empty();
    for (const auto& [id, op] : lr.ops) {
      const OperatorState want_op = run.op(id);
      same = same && op.step == want_op.step && op.master == want_op.master && op.m == want_op.m && op.v == want_op.v;
    }
    std::cout << "SEGMENT ops " << lr.ops.size() << " same " << same << "\n";
    UpstreamLog empty_log(ctx, 1 << 16);
    try {
      DeviceState rec2(ctx, P, static_cast<int>(cb));
      (void)localized_recover(rec2, seg, win, empty_log, &g2, sop, pp, data_seed, ws2 + W, oc);
    } catch (const std::runtime_error& e) {
      std::cout << "ERR runtime_error: " << e.what() << "\n";
    }
  }
  std::cout << "OK\n";
  return 0;
}
