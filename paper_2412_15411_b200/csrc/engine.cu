// engine.cu -- kernels of the GPU toy MoE engine (engine.cuh): the data
// stream, forward + backward of a stage scope, ordered weight-gradient sums.
// Follows moelab::Engine (engine.hpp) operation by operation.
#include "codec.cuh"
#include "engine.cuh"

namespace mlck {
namespace toy {
namespace {

// ---- xoshiro256++ with the reference's named substreams (rng.hpp:14-106)
struct Rng {
  uint64_t s[4];
  __device__ static uint64_t splitmix(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = splitmix(x);
  }
  __device__ uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  __device__ double uniform(double lo, double hi) {
    const double u = __dmul_rn(static_cast<double>(next() >> 11), 0x1.0p-53);
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
  }
  __device__ Rng substream(const char* label, uint64_t index) const {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](uint64_t v) {
      h ^= v;
      h *= 0x100000001b3ull;
    };
    for (const char* c = label; *c; ++c) mix(static_cast<uint8_t>(*c));
    mix(index);
    mix(s[0]);
    mix(s[2]);
    return Rng(h);
  }
};

// engine.hpp:302-314: micro-batch b of replica r at iteration it
__global__ void stream_kernel(float* out, Dims m, uint64_t seed, uint64_t it, int targets) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // r * M + b
  if (k >= static_cast<int64_t>(m.dp) * m.M) return;
  const int64_t r = k / m.M, b = k % m.M;
  const uint64_t idx = (it * static_cast<uint64_t>(m.dp) + r) * static_cast<uint64_t>(m.M) + b;
  Rng g = Rng(seed).substream(targets ? "targets" : "tokens", idx);
  const int64_t n = m.mb * m.d;
  for (int64_t i = 0; i < n; ++i) out[k * n + i] = static_cast<float>(g.uniform(-1.0, 1.0));
}

// tanhf / expf correctly rounded (double evaluation, one rounding)
__device__ __forceinline__ float tanh_f(float x) { return __double2float_rn(tanh(static_cast<double>(x))); }
__device__ __forceinline__ float exp_f(float x) { return __double2float_rn(exp(static_cast<double>(x))); }

struct Weights {
  const void* c;
  int cb;
  __device__ float operator()(int64_t i) const { return codec::load_code(c, static_cast<uint64_t>(i), cb); }
};

// out += W2 tanh(W1 x + b1) + b2 (h > 0); out += W x + b (h == 0)
// (mlp_forward, engine.hpp:608-639)
__device__ void mlp_forward(const Weights& w, int h, int d, const float* x, float* out, float* hid) {
  if (h > 0) {
    const int64_t b1 = static_cast<int64_t>(h) * d, W2 = b1 + h, b2 = W2 + static_cast<int64_t>(d) * h;
    for (int j = 0; j < h; ++j) {
      float s = w(b1 + j);
      for (int i = 0; i < d; ++i) s = __fadd_rn(s, __fmul_rn(w(static_cast<int64_t>(j) * d + i), x[i]));
      hid[j] = tanh_f(s);
    }
    for (int i = 0; i < d; ++i) {
      float s = w(b2 + i);
      for (int j = 0; j < h; ++j) s = __fadd_rn(s, __fmul_rn(w(W2 + static_cast<int64_t>(i) * h + j), hid[j]));
      out[i] = __fadd_rn(out[i], s);
    }
  } else {
    const int64_t b = static_cast<int64_t>(d) * d;
    for (int i = 0; i < d; ++i) {
      float s = w(b + i);
      for (int j = 0; j < d; ++j) s = __fadd_rn(s, __fmul_rn(w(static_cast<int64_t>(i) * d + j), x[j]));
      out[i] = __fadd_rn(out[i], s);
    }
  }
}

// Input gradients always; weight-gradient terms only with `term` (frozen
// operators skip them) -- mlp_backward, engine.hpp:643-696.  Each term is
// this token's addend of the reference's `+=` into the parameter's gradient.
__device__ void mlp_backward(const Weights& w, int h, int d, const float* x, const float* hid, const float* dy,
                             float* dx, float* dh, float* term) {
  if (h > 0) {
    const int64_t b1 = static_cast<int64_t>(h) * d, W2 = b1 + h, b2 = W2 + static_cast<int64_t>(d) * h;
    for (int j = 0; j < h; ++j) dh[j] = 0.0f;
    for (int i = 0; i < d; ++i) {
      const float g = dy[i];
      for (int j = 0; j < h; ++j) {
        dh[j] = __fadd_rn(dh[j], __fmul_rn(w(W2 + static_cast<int64_t>(i) * h + j), g));
        if (term) term[W2 + static_cast<int64_t>(i) * h + j] = __fmul_rn(hid[j], g);
      }
      if (term) term[b2 + i] = g;
    }
    for (int j = 0; j < h; ++j) {
      const float t = hid[j];
      dh[j] = __fmul_rn(dh[j], __fsub_rn(1.0f, __fmul_rn(t, t)));
    }
    for (int j = 0; j < h; ++j) {
      const float g = dh[j];
      for (int i = 0; i < d; ++i) {
        dx[i] = __fadd_rn(dx[i], __fmul_rn(w(static_cast<int64_t>(j) * d + i), g));
        if (term) term[static_cast<int64_t>(j) * d + i] = __fmul_rn(x[i], g);
      }
      if (term) term[b1 + j] = g;
    }
  } else {
    for (int i = 0; i < d; ++i) {
      const float g = dy[i];
      for (int j = 0; j < d; ++j) {
        dx[j] = __fadd_rn(dx[j], __fmul_rn(w(static_cast<int64_t>(i) * d + j), g));
        if (term) term[static_cast<int64_t>(i) * d + j] = __fmul_rn(x[j], g);
      }
      if (term) term[static_cast<int64_t>(d) * d + i] = g;
    }
  }
}

__device__ __forceinline__ int sel_at(const float* c, int k) { return __float_as_int(c[k]); }

// forward_layer (engine.hpp:420-530) for one token; acts in, acts out
__device__ void forward_layer(const ScopeArgs& a, int32_t l, float* acts, float* y, float* c) {
  const Dims& m = a.m;
  const int d = m.d, E = m.E, ns = m.nsel();
  const CacheLayout L(m);
  const int64_t base = static_cast<int64_t>(l) * m.ops_per_layer();
  const Weights ne{a.codes[base + E], m.cb}, gate{a.codes[base + E + 1], m.cb};
  for (int i = 0; i < d; ++i) {
    c[L.x + i] = acts[i];
    y[i] = m.residual ? acts[i] : 0.0f;
  }
  const float* x = c + L.x;
  mlp_forward(ne, m.hn, d, x, y, c + L.nh);
  float* sc = c + L.sc;
  for (int e = 0; e < E; ++e) {
    float s = gate(static_cast<int64_t>(E) * d + e);
    for (int i = 0; i < d; ++i) s = __fadd_rn(s, __fmul_rn(gate(static_cast<int64_t>(e) * d + i), x[i]));
    sc[e] = s;
  }
  // shared experts, then the top-k routed by (score desc, index asc) -- the
  // stable_sort of engine.hpp:467-472 -- in ascending index order
  float* sel = c + L.sel;
  for (int k = 0; k < m.shared; ++k) sel[k] = __int_as_float(k);
  int prev = -1;
  for (int k = 0; k < m.top_k; ++k) {
    int best = -1;
    for (int e = m.shared; e < E; ++e) {
      const bool after_prev = prev < 0 || sc[e] < sc[prev] || (sc[e] == sc[prev] && e > prev);
      if (after_prev && (best < 0 || sc[e] > sc[best])) best = e;
    }
    prev = best;
    int pos = m.shared + k;  // insertion into ascending order
    while (pos > m.shared && sel_at(sel, pos - 1) > best) {
      sel[pos] = sel[pos - 1];
      --pos;
    }
    sel[pos] = __int_as_float(best);
  }
  float* wt = c + L.wt;
  for (int k = 0; k < ns; ++k) wt[k] = 1.0f;
  {  // softmax over the routed selection (engine.hpp:478-488)
    float mx = -INFINITY;
    for (int k = m.shared; k < ns; ++k) {
      const float s = sc[sel_at(sel, k)];
      mx = mx < s ? s : mx;
    }
    float denom = 0.0f;
    for (int k = m.shared; k < ns; ++k) denom = __fadd_rn(denom, exp_f(__fsub_rn(sc[sel_at(sel, k)], mx)));
    for (int k = m.shared; k < ns; ++k) wt[k] = __fdiv_rn(exp_f(__fsub_rn(sc[sel_at(sel, k)], mx)), denom);
  }
  const int he = m.he > 0 ? m.he : 1;
  for (int k = 0; k < ns; ++k) {
    const Weights ex{a.codes[base + sel_at(sel, k)], m.cb};
    float* eo = c + L.eo + static_cast<int64_t>(k) * d;
    for (int i = 0; i < d; ++i) eo[i] = 0.0f;
    mlp_forward(ex, m.he, d, x, eo, c + L.eh + static_cast<int64_t>(k) * he);
    for (int i = 0; i < d; ++i) y[i] = __fadd_rn(y[i], __fmul_rn(wt[k], eo[i]));
  }
  for (int i = 0; i < d; ++i) acts[i] = y[i];
}

// backward_layer (engine.hpp:534-606) for one token; dy in, dx out (in dy)
__device__ void backward_layer(const ScopeArgs& a, int32_t l, float* dy, float* dx, float* de, float* dwt,
                               float* dh, const float* c, float* t) {
  const Dims& m = a.m;
  const int d = m.d, E = m.E, ns = m.nsel();
  const CacheLayout L(m);
  const TermLayout T(m);
  const int64_t base = static_cast<int64_t>(l) * m.ops_per_layer(), ne_id = base + E, gate_id = base + E + 1;
  const Weights ne{a.codes[ne_id], m.cb}, gate{a.codes[gate_id], m.cb};
  const float* x = c + L.x;
  for (int i = 0; i < d; ++i) dx[i] = m.residual ? __fadd_rn(0.0f, dy[i]) : 0.0f;
  mlp_backward(ne, m.hn, d, x, c + L.nh, dy, dx, dh, a.active[ne_id] ? t + T.ne : nullptr);
  const float* sel = c + L.sel;
  const float* wt = c + L.wt;
  const int he = m.he > 0 ? m.he : 1;
  const int64_t e_live = Dims::mlp_live(d, m.he);
  for (int k = 0; k < ns; ++k) {
    const int64_t eid = base + sel_at(sel, k);
    const float* eo = c + L.eo + static_cast<int64_t>(k) * d;
    dwt[k] = 0.0f;
    for (int i = 0; i < d; ++i) de[i] = __fmul_rn(wt[k], dy[i]);
    for (int i = 0; i < d; ++i) dwt[k] = __fadd_rn(dwt[k], __fmul_rn(dy[i], eo[i]));
    const Weights ex{a.codes[eid], m.cb};
    mlp_backward(ex, m.he, d, x, c + L.eh + static_cast<int64_t>(k) * he, de, dx, dh,
                 a.active[eid] ? t + T.ex + k * e_live : nullptr);
  }
  if (ns > m.shared) {  // softmax backward -> gate score gradients
    float dot = 0.0f;
    for (int k = m.shared; k < ns; ++k) dot = __fadd_rn(dot, __fmul_rn(dwt[k], wt[k]));
    for (int k = m.shared; k < ns; ++k) {
      const float ds = __fmul_rn(wt[k], __fsub_rn(dwt[k], dot));
      const int e = sel_at(sel, k);
      if (a.active[gate_id]) {
        for (int i = 0; i < d; ++i) t[T.gate + static_cast<int64_t>(e) * d + i] = __fmul_rn(ds, x[i]);
        t[T.gate + static_cast<int64_t>(E) * d + e] = ds;
      }
      for (int i = 0; i < d; ++i) dx[i] = __fadd_rn(dx[i], __fmul_rn(ds, gate(static_cast<int64_t>(e) * d + i)));
    }
  }
  for (int i = 0; i < d; ++i) dy[i] = dx[i];
}

__global__ void scope_kernel(ScopeArgs a) {
  const Dims& m = a.m;
  const int64_t tok = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t T = m.tokens();
  if (tok >= T) return;
  const int d = m.d, ns = m.nsel(), nl = a.layer_hi - a.layer_lo + 1;
  const int64_t hmax = (m.he > m.hn ? m.he : m.hn) > 0 ? (m.he > m.hn ? m.he : m.hn) : 1;
  const CacheLayout L(m);
  const TermLayout TL(m);
  float* cache = a.cache + tok * nl * L.stride;
  float* terms = a.terms + tok * nl * TL.stride;
  float* work = a.work + tok * (4 * static_cast<int64_t>(d) + 2 * ns + 2 * hmax);
  float *acts = work, *y = work + d, *dx = work + 2 * d, *de = work + 3 * d, *dwt = work + 4 * d,
        *dh = dwt + ns;
  for (int i = 0; i < d; ++i) acts[i] = a.in_acts[tok * d + i];
  int32_t cur = a.stage_lo;
  for (int32_t l = a.layer_lo; l <= a.layer_hi; ++l) {
    const int32_t ls = m.stage_of_layer(l);
    if (ls != cur) {  // sender-side copy at an inner boundary (engine.hpp:381-387)
      if (a.fwd_out)
        for (int i = 0; i < d; ++i) a.fwd_out[((ls - 1 - a.stage_lo) * T + tok) * d + i] = acts[i];
      cur = ls;
    }
    forward_layer(a, l, acts, y, cache + (l - a.layer_lo) * L.stride);
  }
  // loss head (engine.hpp:390-392) or the logged gradient
  if (a.stage_hi == m.stages - 1)
    for (int i = 0; i < d; ++i) acts[i] = __fmul_rn(__fsub_rn(acts[i], a.targets[tok * d + i]), a.inv_tokens);
  else
    for (int i = 0; i < d; ++i) acts[i] = a.grad_in[tok * d + i];
  cur = m.stage_of_layer(a.layer_hi);
  for (int32_t l = a.layer_hi; l >= a.layer_lo; --l) {
    const int32_t ls = m.stage_of_layer(l);
    if (ls != cur) {  // engine.hpp:404-411
      if (a.bwd_out)
        for (int i = 0; i < d; ++i) a.bwd_out[((ls - a.stage_lo) * T + tok) * d + i] = acts[i];
      cur = ls;
    }
    backward_layer(a, l, acts, dx, de, dwt, dh, cache + (l - a.layer_lo) * L.stride,
                   terms + (l - a.layer_lo) * TL.stride);
  }
}

// grads[op][p] = sum over tokens, in (replica, micro-batch, token) order, of
// their terms -- the reference's sequence of `+=` (engine.hpp:143-147)
__global__ void reduce_kernel(ScopeArgs a, int32_t l, float* const* grads) {
  const Dims& m = a.m;
  const int j = blockIdx.y;  // operator of the layer: experts, NE, gate
  const int64_t op = static_cast<int64_t>(l) * m.ops_per_layer() + j;
  float* g = grads[op];
  if (!g || !a.active[op]) return;
  const int64_t live = j < m.E ? Dims::mlp_live(m.d, m.he) : j == m.E ? Dims::mlp_live(m.d, m.hn) : m.g_live();
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= live) return;
  const CacheLayout L(m);
  const TermLayout TL(m);
  const int nl = a.layer_hi - a.layer_lo + 1, ci = l - a.layer_lo, ns = m.nsel();
  const int64_t T = m.tokens();
  const int ge = j == m.E + 1 ? static_cast<int>(p < static_cast<int64_t>(m.E) * m.d ? p / m.d : p - static_cast<int64_t>(m.E) * m.d) : 0;
  float s = 0.0f;
  for (int64_t tok = 0; tok < T; ++tok) {
    const float* c = a.cache + (tok * nl + ci) * L.stride;
    const float* t = a.terms + (tok * nl + ci) * TL.stride;
    if (j == m.E) {
      s = __fadd_rn(s, t[TL.ne + p]);
    } else if (j == m.E + 1) {
      for (int k = m.shared; k < ns; ++k)
        if (sel_at(c + L.sel, k) == ge) s = __fadd_rn(s, t[TL.gate + p]);
    } else {
      for (int k = 0; k < ns; ++k)
        if (sel_at(c + L.sel, k) == j) s = __fadd_rn(s, t[TL.ex + k * live + p]);
    }
  }
  g[p] = s;
}

}  // namespace

void launch_stream(float* out, const Dims& m, uint64_t seed, uint64_t it, int targets, cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(m.dp) * m.M;
  stream_kernel<<<static_cast<unsigned>((n + 63) / 64), 64, 0, stream>>>(out, m, seed, it, targets);
  MLCK_CUDA(cudaGetLastError());
}

void launch_scope(const ScopeArgs& a, cudaStream_t stream) {
  const int64_t T = a.m.tokens();
  scope_kernel<<<static_cast<unsigned>((T + 63) / 64), 64, 0, stream>>>(a);
  MLCK_CUDA(cudaGetLastError());
}

void launch_reduce(const ScopeArgs& a, int32_t l, float* const* grads, cudaStream_t stream) {
  const Dims& m = a.m;
  int64_t live = m.g_live();
  live = live > Dims::mlp_live(m.d, m.he) ? live : Dims::mlp_live(m.d, m.he);
  live = live > Dims::mlp_live(m.d, m.hn) ? live : Dims::mlp_live(m.d, m.hn);
  const dim3 grid(static_cast<unsigned>((live + 127) / 128), static_cast<unsigned>(m.ops_per_layer()));
  reduce_kernel<<<grid, 128, 0, stream>>>(a, l, grads);
  MLCK_CUDA(cudaGetLastError());
}

}  // namespace toy
}  // namespace mlck
