// engine.cuh -- the reference's miniature MoE trainer (moelab::Engine,
// engine.hpp:150-730) as sm_100a kernels: the recompute half of the
// checkpoint path.  Conversion and localized recovery can
// replay the window's iterations by re-running forward + backward, frozen
// operators producing input gradients only (engine.hpp:562/581/594), instead
// of reading logged weight gradients; and run_iteration is a GPU producer
// of both the upstream boundary log and the weight-gradient log.
//
// Layout.  One thread per token (the model has no cross-token coupling:
// routing is per token, no capacity limit), all layers of the scope in one
// pass, activations and caches in a per-token scratch row.  Each token's
// weight-gradient terms are kept apart and summed per parameter in the
// reference's canonical order (replica, micro-batch, token; engine.hpp:
// 143-147), so a replay is bit-identical to the GPU run it replays.  Float
// arithmetic follows the reference's operation order without contraction
// (--fmad=false); tanh / exp are evaluated in double and rounded once (the
// correctly rounded tanhf / expf), so parity with the CPU reference holds to
// the ulp where glibc's tanhf / expf round correctly -- a tolerance, stated
// in the tests.
#pragma once

#include "mlck_common.cuh"

namespace mlck {
namespace toy {

struct Dims {
  int32_t layers, E, top_k, shared, d, he, hn, residual;
  int32_t stages, dp, M;
  int64_t mb;
  int64_t pe, pn, pg;  // parameters per expert / non-expert block / gate
  int32_t cb;          // compute width (codes)
  __host__ __device__ int32_t nsel() const { return shared + top_k; }
  __host__ __device__ int32_t ops_per_layer() const { return E + 2; }
  __host__ __device__ int64_t tokens() const { return static_cast<int64_t>(dp) * M * mb; }
  __host__ __device__ static int64_t mlp_live(int64_t d, int64_t h) { return h > 0 ? 2 * d * h + h + d : d * d + d; }
  __host__ __device__ int64_t ne_live() const { return mlp_live(d, hn); }
  __host__ __device__ int64_t e_live() const { return mlp_live(d, he); }
  __host__ __device__ int64_t g_live() const { return static_cast<int64_t>(E) * d + E; }
  __host__ __device__ int32_t stage_of_layer(int32_t l) const {
    return static_cast<int32_t>((static_cast<int64_t>(l) * stages) / layers);
  }
};

// Per-token scratch of one layer of the scope (floats; selections as ints)
struct CacheLayout {
  int64_t x, nh, sc, sel, wt, eh, eo, stride;
  __host__ __device__ explicit CacheLayout(const Dims& m) {
    const int64_t hn = m.hn > 0 ? m.hn : 1, he = m.he > 0 ? m.he : 1, ns = m.shared + m.top_k;
    x = 0;
    nh = x + m.d;
    sc = nh + hn;
    sel = sc + m.E;
    wt = sel + ns;
    eh = wt + ns;
    eo = eh + ns * he;
    stride = eo + ns * m.d;
  }
};
// Per-token weight-gradient terms of one layer: NE, gate, each selected expert
struct TermLayout {
  int64_t ne, gate, ex, stride;
  __host__ __device__ explicit TermLayout(const Dims& m) {
    ne = 0;
    gate = ne + Dims::mlp_live(m.d, m.hn);
    ex = gate + static_cast<int64_t>(m.E) * m.d + m.E;
    stride = ex + static_cast<int64_t>(m.shared + m.top_k) * Dims::mlp_live(m.d, m.he);
  }
};

// Launchers (engine.cu).
// Data stream batch_tokens / batch_targets (engine.hpp:226-236, 302-314):
// out[(r * M + b) * mb * d + ...] for every replica r and micro-batch b.
void launch_stream(float* out, const Dims& m, uint64_t data_seed, uint64_t iteration, int targets,
                   cudaStream_t stream);
// Forward + backward of every token over layers [layer_lo, layer_hi]
// (run_scoped, engine.hpp:332-417).  codes[op] = compute codes of each
// operator (index op id); active[op] = 1 when its weight gradient is wanted.
// in_acts: [T, d] scope inputs; grad_in: [T, d] the loss-side gradient when
// stage_hi is the last stage is computed from `targets`, else given.
// fwd_out[s - stage_lo] / bwd_out[s - stage_lo]: [T, d] sender-side copies at
// the scope's inner boundaries (may be null).  terms: [T, nl, TermLayout].
struct ScopeArgs {
  Dims m;
  int32_t layer_lo, layer_hi, stage_lo, stage_hi;
  const void* const* codes;  // device array of n_ops code pointers
  const uint8_t* active;     // device [n_ops]
  const float* in_acts;
  const float* targets;      // [T, d] when stage_hi == stages - 1
  const float* grad_in;      // [T, d] otherwise
  float* fwd_out;            // [stage_hi - stage_lo][T][d]
  float* bwd_out;            // [stage_hi - stage_lo][T][d]
  float* cache;              // [T][nl][CacheLayout.stride]
  float* work;               // [T][4 d + 2 nsel + 2 max(h)]
  float* terms;              // [T][nl][TermLayout.stride]
  float inv_tokens;
};
void launch_scope(const ScopeArgs& a, cudaStream_t stream);
// Weight gradients of the active operators of layer l (ordered token sums):
// grads[op] (P floats, zeroed beyond the live parameters) for op in the
// layer, null entries skipped.
void launch_reduce(const ScopeArgs& a, int32_t layer, float* const* grads_dev, cudaStream_t stream);

}  // namespace toy
}  // namespace mlck
