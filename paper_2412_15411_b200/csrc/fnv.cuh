// fnv.cuh -- parallel, bit-exact FNV-1a-64 for the MLCK container trailer.
//
// Replaces the byte-serial moelab::fnv1a64 (digest.hpp:18-25), which is on
// both the pack path (serialize_record trailer, snapshot.hpp:142) and the
// verify path (parse_record, snapshot.hpp:156-163).
//
// Decomposition (verified in tests/test_fnv_model.py):
//   h_{i+1} = (h_i ^ b_i) * P  ==  (h_i + d_i) * P,  d_i = (u_i ^ b_i) - u_i,
//   u_i = low byte of h_i, so  h_N = P^N h_0 + sum_i d_i P^(N-i)  (mod 2^64).
// The only sequential part is the 8-bit automaton u' = ((u ^ b) * 0xb3) & 255.
// It is a T-function: bit j of u' depends on bits <= j only, and
//   u'_j = u_j ^ b_j ^ R_j(y_0..y_{j-1}),   y = u ^ b,
// where R_j is the carry/sum of the lower columns of y*0xb3 (0xb3 = shifts
// {0,1,4,5,7}).  So each bit level is a prefix-XOR over positions once the
// lower levels are known.  Positions are bit-sliced 32 per word (an 8x8 bit
// transpose per byte lane), every level is a word-parallel prefix-XOR, and the
// chunk-to-chunk carry of each level is resolved with a decoupled look-back
// (one status word per chunk carries 8 aggregate bits and 8 inclusive bits).
// After the 8 levels every position knows u_i; d_i = b_i - 2 (u_i & b_i) and
// the polynomial sum is a per-thread Horner combined with precomputed powers.
#pragma once

#include "mlck_common.cuh"

namespace mlck {
namespace fnv {

constexpr uint64_t kPrime = 0x100000001b3ull;
constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
#ifndef MLCK_FNV_THREADS
#define MLCK_FNV_THREADS 1024
#endif
constexpr int kThreads = MLCK_FNV_THREADS;  // one CTA per SM at 64 regs/thread
constexpr int kBytesPerThread = 64;  // two 32-position groups
constexpr int kChunk = kThreads * kBytesPerThread;
constexpr int kWarps = kThreads / 32;

// One 64-bit look-back word per chunk, kStatusStride words apart (256 B): the
// ~600 in-flight chunks' words land in different L2 slices instead of a
// handful of hot lines.  The high half is the launch epoch, so the array is
// never cleared between launches (a word from an older launch reads as
// "nothing published").
constexpr int kStatusStride = 32;

struct Scratch {
  unsigned long long* status;  // [n_chunks * kStatusStride] epoch-tagged words
  uint32_t epoch;              // this launch's tag (>= 1)
  uint32_t* ticket;            // chunk dispatch counter (zeroed per launch)
  unsigned long long* accum;   // sum of chunk terms
  uint32_t* finished;          // completed-chunk counter
  unsigned long long* result;  // final 64-bit hash
  // optional profile counters (null = off): [0] look-back probes,
  // [1] spin re-reads, [2] cycles before look-backs, [3] cycles in
  // look-backs, [4] cycles in phase B, [5] chunks
  unsigned long long* prof;
  // optional per-chunk trace (null = off): 12 words per chunk, %globaltimer
  // ns at [0] start, [1+2r] map published, [2+2r] round resolved, [9] end,
  // [10] smid
  unsigned long long* trace;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// P^(64 k) for k = 0..kThreads-1, written by init_constants() (kernels.cu).
__constant__ unsigned long long c_pow64[kThreads];
// Q_k = P^(64-k) for a thread segment, split into 32-bit halves, and
// 512 * sum_k Q_k (the bias of the unsigned per-byte terms).
__constant__ uint32_t c_qlo[kBytesPerThread];
__constant__ uint32_t c_qhi[kBytesPerThread];
__constant__ unsigned long long c_qbias;
__host__ __device__ inline uint64_t mul_p(uint64_t x) { return x * kPrime; }

__host__ __device__ inline uint64_t pow_p(uint64_t e) {
  uint64_t r = 1, b = kPrime;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// ---- bit-slice transposes ----------------------------------------------
__device__ __forceinline__ void swapmove(uint32_t& a, uint32_t& b, uint32_t mask, int n) {
  const uint32_t t = ((a >> n) ^ b) & mask;
  b ^= t;
  a ^= t << n;
}
__device__ __forceinline__ void bit_transpose8(uint32_t x[8]) {
#pragma unroll
  for (int i = 0; i < 8; i += 2) swapmove(x[i], x[i + 1], 0x55555555u, 1);
#pragma unroll
  for (int i : {0, 1, 4, 5}) swapmove(x[i], x[i + 2], 0x33333333u, 2);
#pragma unroll
  for (int i = 0; i < 4; ++i) swapmove(x[i], x[i + 4], 0x0f0f0f0fu, 4);
}
// 32 bytes (word q byte k = position 4q+k) -> 8 planes (bit p = position p).
__device__ __forceinline__ void to_planes(const uint32_t w[8], uint32_t x[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int a = i >> 2, k = i & 3;
    const uint32_t sel = k | ((k + 4) << 4);
    const uint32_t lo = __byte_perm(w[a], w[a + 2], sel);
    const uint32_t hi = __byte_perm(w[a + 4], w[a + 6], sel);
    x[i] = __byte_perm(lo, hi, 0x5410);
  }
  bit_transpose8(x);
}
// inverse of to_planes
__device__ __forceinline__ void from_planes(uint32_t x[8], uint32_t w[8]) {
  bit_transpose8(x);
  // w[q] byte k = position 4q+k = x[(4q+k)&7] byte ((4q+k)>>3)
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int lane = q >> 1;            // (4q+k)>>3 for k=0..3
    const int i0 = (4 * q) & 7;         // x index of k=0
    const uint32_t s = lane | ((lane + 4) << 4);
    const uint32_t lo = __byte_perm(x[i0], x[i0 + 1], s);
    const uint32_t hi = __byte_perm(x[i0 + 2], x[i0 + 3], s);
    w[q] = __byte_perm(lo, hi, 0x5410);
  }
}

__device__ __forceinline__ uint32_t prefix_xor(uint32_t t) {
  t ^= t << 1;
  t ^= t << 2;
  t ^= t << 4;
  t ^= t << 8;
  t ^= t << 16;
  return t;
}
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (c & (a | b));
}
__device__ __forceinline__ uint32_t bcast(uint32_t bit) { return 0u - bit; }

// Column-carry state of y*0xb3 for one 32-position group.
struct Carries {
  uint32_t c1, c2, c3, c4a, c4b, k5a, k5b, k5c, m6a, m6b, m6c;
};

// R_j: contribution of y_0..y_{j-1} (and lower carries) to bit j of y*0xb3.
__device__ __forceinline__ uint32_t level_r(int j, const uint32_t y[8], const Carries& c) {
  switch (j) {
    case 0: return 0u;
    case 1: return y[0];
    case 2: return y[1] ^ c.c1;
    case 3: return y[2] ^ c.c2;
    case 4: return y[3] ^ y[0] ^ c.c3;
    case 5: return y[4] ^ y[1] ^ y[0] ^ c.c4a ^ c.c4b;
    case 6: return y[5] ^ y[2] ^ y[1] ^ c.k5a ^ c.k5b ^ c.k5c;
    default: return y[6] ^ y[3] ^ y[2] ^ y[0] ^ c.m6a ^ c.m6b ^ c.m6c;
  }
}
// After y_j is known: compress column j of y*0xb3 into carries for j+1.
__device__ __forceinline__ void level_carry(int j, const uint32_t y[8], Carries& c) {
  switch (j) {
    case 1: c.c1 = y[1] & y[0]; break;
    case 2: c.c2 = maj3(y[2], y[1], c.c1); break;
    case 3: c.c3 = maj3(y[3], y[2], c.c2); break;
    case 4: {
      const uint32_t s = y[4] ^ y[3] ^ y[0];
      c.c4a = maj3(y[4], y[3], y[0]);
      c.c4b = s & c.c3;
    } break;
    case 5: {
      const uint32_t s5a = y[5] ^ y[4] ^ y[1];
      const uint32_t s5b = y[0] ^ c.c4a ^ c.c4b;
      c.k5a = maj3(y[5], y[4], y[1]);
      c.k5b = maj3(y[0], c.c4a, c.c4b);
      c.k5c = s5a & s5b;
    } break;
    case 6: {
      const uint32_t s6a = y[6] ^ y[5] ^ y[2];
      const uint32_t s6b = y[1] ^ c.k5a ^ c.k5b;
      c.m6a = maj3(y[6], y[5], y[2]);
      c.m6b = maj3(y[1], c.k5a, c.k5b);
      c.m6c = maj3(s6a, s6b, c.k5c);
    } break;
    default: break;
  }
}

// Two bit levels (2r, 2r+1) are resolved per look-back round.  A chunk's
// effect on those two state bits, given its true lower start bits, is the map
//   s0' = s0 ^ a,   s1' = s1 ^ (s0 ? b1 : b0)
// packed as bits {a, b0, b1}; the family is closed under composition.
__device__ __forceinline__ uint32_t map_compose(uint32_t g, uint32_t f) {  // g o f
  const uint32_t af = f & 1u, b0f = (f >> 1) & 1u, b1f = (f >> 2) & 1u;
  const uint32_t ag = g & 1u, b0g = (g >> 1) & 1u, b1g = (g >> 2) & 1u;
  const uint32_t b0 = b0f ^ (af ? b1g : b0g);
  const uint32_t b1 = b1f ^ (af ? b0g : b1g);
  return (af ^ ag) | (b0 << 1) | (b1 << 2);
}
__device__ __forceinline__ uint32_t map_apply(uint32_t m, uint32_t s) {
  const uint32_t s0 = s & 1u, s1 = (s >> 1) & 1u;
  return (s0 ^ (m & 1u)) | ((s1 ^ ((m >> (1 + s0)) & 1u)) << 1);
}

// Status word of a chunk: bits [3r,3r+3) the round-r map, [12+2r,14+2r) the
// round-r inclusive end bits, [20,23) rounds with map published, [24,27)
// rounds with inclusive published.
constexpr int kRounds = 4;
__device__ __forceinline__ uint32_t st_nagg(uint32_t s) { return (s >> 20) & 7u; }
__device__ __forceinline__ uint32_t st_nincl(uint32_t s) { return (s >> 24) & 7u; }

struct SharedState {
  uint32_t sa[kWarps];      // level-2r thread-parity scan
  uint32_t sb[2][kWarps];   // level-2r+1 scan, per variant
  uint32_t start;           // resolved start bits of the round
  unsigned long long pc;    // P^(N - chunk_end); final hash in the last block
  unsigned long long red[kWarps];
};

// Look-back for round r, run by warp 0 alone: lane l probes the 8
// predecessors base-8l .. base-8l-7 with all 8 loads in flight, so one probe
// covers 256 chunks (more than the in-flight window) at one load latency.
// Returns the chunk's two start bits (in warp 0).
constexpr int kProbePerLane = 8;
__device__ __forceinline__ uint32_t look_back2_warp(const unsigned long long* status,
                                                    uint32_t epoch, int64_t chunk, int r,
                                                    uint32_t seed2, unsigned long long* prof) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;  // identity map
  int64_t base = chunk - 1;
  while (true) {
    if (prof && lane == 0) atomicAdd(prof + 0, 1ull);
    unsigned long long v[kProbePerLane];
#pragma unroll
    for (int q = 0; q < kProbePerLane; ++q) {
      const int64_t k = base - kProbePerLane * lane - q;
      v[q] = k < 0 ? 0ull : ld_relaxed_gpu_u64(status + k * kStatusStride);
    }
    // lane-local: nearest-first composition up to the first inclusive
    uint32_t m = 0, incl_val = 0;
    bool has_incl = false;
#pragma unroll
    for (int q = 0; q < kProbePerLane; ++q) {
      if (has_incl) continue;
      const int64_t k = base - kProbePerLane * lane - q;
      if (k < 0) {
        has_incl = true;
        incl_val = seed2;
        continue;
      }
      uint32_t s;
      uint32_t backoff = 32, spins = 0;
      // back off while the predecessor is behind (keeps pollers off L2)
      while (static_cast<uint32_t>(v[q] >> 32) != epoch ||
             st_nagg(s = static_cast<uint32_t>(v[q])) <= static_cast<uint32_t>(r)) {
        __nanosleep(backoff);
        backoff = backoff < 256 ? 2 * backoff : 256;
        v[q] = ld_relaxed_gpu_u64(status + k * kStatusStride);
        ++spins;
      }
      if (prof && spins) atomicAdd(prof + 1, static_cast<unsigned long long>(spins));
      if (st_nincl(s) > static_cast<uint32_t>(r)) {
        has_incl = true;
        incl_val = (s >> (12 + 2 * r)) & 3u;
      } else {
        m = map_compose(m, (s >> (3 * r)) & 7u);  // apply the farther map first
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, has_incl);
    const int first = bal ? __ffs(bal) - 1 : 32;
    // L_0 o L_1 o ... o L_first (lanes past the nearest inclusive: identity)
    uint32_t t = lane <= first ? m : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_down_sync(0xffffffffu, t, off);
      if (lane + off < 32) t = map_compose(t, o);
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    acc = map_compose(acc, t);
    if (bal) return map_apply(acc, __shfl_sync(0xffffffffu, incl_val, first));
    base -= 32 * kProbePerLane;
  }
}

constexpr int kGroups = kBytesPerThread / 32;

// 64 bytes at pos0 as 16 little-endian words, zero past n.
__device__ __forceinline__ void load_words64(const uint8_t* data, uint64_t n, uint64_t pos0,
                                             uint32_t (&w)[16]) {
  if (pos0 + 64 <= n && (reinterpret_cast<uintptr_t>(data) & 15u) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(data + pos0 + 16 * q);
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      uint32_t x = 0;
      for (int k = 0; k < 4; ++k) {
        const uint64_t p = pos0 + 4 * q + k;
        if (p < n) x |= static_cast<uint32_t>(data[p]) << (8 * k);
      }
      w[q] = x;
    }
  }
}

// Block-level FNV contribution of one kChunk-byte chunk of `data`; thread t
// owns bytes [chunk*kChunk + 64t, +64).  The chunk's term P^(N-end) * H is
// atomically accumulated into scr.accum; the last chunk to finish writes the
// final hash into scr.result (and sh.pc) and returns true in thread 0.
__device__ inline bool chunk_contribution(const uint8_t* data, int64_t chunk, uint64_t n,
                                          uint64_t seed, const Scratch& scr, uint64_t n_chunks,
                                          SharedState& sh) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t pos0 = static_cast<uint64_t>(chunk) * kChunk + static_cast<uint64_t>(tid) * kBytesPerThread;

  uint32_t B[kGroups][8], Y[kGroups][8];
  Carries car[kGroups];
  {
    uint32_t w[16];
    load_words64(data, n, pos0, w);
#pragma unroll
    for (int g = 0; g < kGroups; ++g) to_planes(w + 8 * g, B[g]);
  }
  // Positions past n are zero bytes; d_i is forced to zero for them below and
  // only the final chunk is padded, so its trailing states are never used.

  __syncthreads();  // previous chunk's readers of sh are done
  uint32_t status = 0;  // owner's view (thread 0)
  long long t_mark = scr.prof ? clock64() : 0;
  if (scr.trace && tid == 0) {
    scr.trace[chunk * 12 + 0] = gtimer();
    scr.trace[chunk * 12 + 10] = smid();
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int j0 = 2 * r, j1 = 2 * r + 1;
    // ---- level j0 (all lower start bits known): toggles and their prefix
    uint32_t T0[kGroups], I0[kGroups];
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      T0[g] = B[g][j0] ^ level_r(j0, Y[g], car[g]);
      I0[g] = prefix_xor(T0[g]);
      if (g) I0[g] ^= bcast(I0[g - 1] >> 31);
    }
    {
      const uint32_t bal = __ballot_sync(0xffffffffu, I0[kGroups - 1] >> 31);
      if (lane == 0) sh.sa[warp] = __popc(bal) & 1u;
      __syncthreads();
      // warp-parity bits of all warps in one ballot (lane q reads warp q)
      const uint32_t wb = __ballot_sync(0xffffffffu, lane < kWarps ? sh.sa[lane] : 0u);
      const uint32_t lt_w = (1u << warp) - 1u;
      const uint32_t agg = __popc(wb) & 1u;
      const uint32_t e0 = (__popc(wb & lt_w) ^ __popc(bal & lt)) & 1u;
      // ---- level j1 for both values v of the chunk's start bit j0
      uint32_t T1[2][kGroups];
      uint32_t pv[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        uint32_t x = 0;
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
          uint32_t yv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) yv[q] = Y[g][q];
          yv[j0] = I0[g] ^ T0[g] ^ bcast(e0 ^ static_cast<uint32_t>(v)) ^ B[g][j0];
          Carries cv = car[g];
          level_carry(j0, yv, cv);
          T1[v][g] = B[g][j1] ^ level_r(j1, yv, cv);
          x ^= T1[v][g];
        }
        pv[v] = __popc(x) & 1u;
      }
      const uint32_t bal0 = __ballot_sync(0xffffffffu, pv[0]);
      const uint32_t bal1 = __ballot_sync(0xffffffffu, pv[1]);
      if (lane == 0) {
        sh.sb[0][warp] = __popc(bal0) & 1u;
        sh.sb[1][warp] = __popc(bal1) & 1u;
      }
      __syncthreads();
      uint32_t wx1[2], tot[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const uint32_t w1 = __ballot_sync(0xffffffffu, lane < kWarps ? sh.sb[v][lane] : 0u);
        wx1[v] = __popc(w1 & lt_w) & 1u;
        tot[v] = __popc(w1) & 1u;
      }
      const uint32_t map = agg | (tot[0] << 1) | (tot[1] << 2);
      // The last warp owns the status word and runs the look-back: the
      // scheduler issues highest-warp-id first, so the critical-path warp is
      // not starved by compute warps of co-resident work.
      const bool lb_warp = warp == kWarps - 1;
      if (lb_warp && lane == 0) {
        status = (status & ~(7u << 20)) | (map << (3 * r)) | (static_cast<uint32_t>(r + 1) << 20);
        // atomic: performed at L2, visible to pollers immediately
        atomicExch(scr.status + chunk * kStatusStride,
                   (static_cast<unsigned long long>(scr.epoch) << 32) | status);
        if (scr.trace) scr.trace[chunk * 12 + 1 + 2 * r] = gtimer();
      }
      const uint32_t seed2 = static_cast<uint32_t>(seed >> j0) & 3u;
      if (scr.prof && tid == 0) {
        const long long t = clock64();
        atomicAdd(scr.prof + 2, static_cast<unsigned long long>(t - t_mark));
        t_mark = t;
      }
      if (lb_warp) {
        const uint32_t start = look_back2_warp(scr.status, scr.epoch, chunk, r, seed2, scr.prof);
        if (lane == 0) {
          status = (status & ~(7u << 24)) | (map_apply(map, start) << (12 + 2 * r)) |
                   (static_cast<uint32_t>(r + 1) << 24);
          atomicExch(scr.status + chunk * kStatusStride,
                     (static_cast<unsigned long long>(scr.epoch) << 32) | status);
          sh.start = start;
          if (scr.trace) scr.trace[chunk * 12 + 2 + 2 * r] = gtimer();
        }
      }
      __syncthreads();
      if (scr.prof && tid == 0) {
        const long long t = clock64();
        atomicAdd(scr.prof + 3, static_cast<unsigned long long>(t - t_mark));
        t_mark = t;
      }
      const uint32_t start = sh.start;
      const uint32_t s0 = start & 1u, s1 = (start >> 1) & 1u;
      // ---- finalize level j0 with the true start bit
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        Y[g][j0] = I0[g] ^ T0[g] ^ bcast(e0 ^ s0) ^ B[g][j0];
        level_carry(j0, Y[g], car[g]);
      }
      // ---- finalize level j1 (variant s0)
      const uint32_t e1 = (s0 ? wx1[1] : wx1[0]) ^ (__popc((s0 ? bal1 : bal0) & lt) & 1u);
      uint32_t Iprev = 0;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const uint32_t T = s0 ? T1[1][g] : T1[0][g];
        uint32_t I = prefix_xor(T);
        if (g) I ^= bcast(Iprev >> 31);
        Iprev = I;
        Y[g][j1] = I ^ T ^ bcast(e1 ^ s1) ^ B[g][j1];
        level_carry(j1, Y[g], car[g]);
      }
    }
  }

  if (scr.prof && tid == 0) {
    const long long t = clock64();
    atomicAdd(scr.prof + 2, static_cast<unsigned long long>(t - t_mark));
    t_mark = t;
  }
  // ---- phase B: d_i = b_i - 2 (u_i & b_i); z = u & b = b & ~y
  uint32_t zw[16];
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    uint32_t Z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) Z[j] = B[g][j] & ~Y[g][j];
    from_planes(Z, zw + 8 * g);
  }
  const uint64_t chunk_end = static_cast<uint64_t>(chunk + 1) * kChunk;
  uint64_t term = 0;
  {
    uint32_t w[16];  // reloaded (L1/L2 hit) instead of held live across the levels
    load_words64(data, n, pos0, w);
    uint64_t acc = 0;
    uint64_t seg_end = pos0 + kBytesPerThread;
    if (pos0 + kBytesPerThread <= n) {
      // acc = sum_k d_k P^(64-k) as independent products (no serial Horner):
      // with db = d + 512 >= 0, sum db*Q mod 2^64 = sum mad.wide(db, Q_lo)
      // + 2^32 sum mad.lo(db, Q_hi); the bias is removed once (c_qbias).
      uint64_t lo[4] = {0, 0, 0, 0};  // independent chains for ILP
      uint32_t hi[4] = {0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < 16; ++q) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t b = __byte_perm(w[q], 0, 0x4440 + k);
          const uint32_t z = __byte_perm(zw[q], 0, 0x4440 + k);
          const uint32_t db = b + 512u - 2u * z;
          lo[k] += static_cast<uint64_t>(db) * c_qlo[4 * q + k];  // mad.wide.u32
          hi[k] += db * c_qhi[4 * q + k];
        }
      }
      acc = (lo[0] + lo[1]) + (lo[2] + lo[3]) +
            (static_cast<uint64_t>((hi[0] + hi[1]) + (hi[2] + hi[3])) << 32) - c_qbias;
    } else {
      seg_end = pos0 < n ? n : pos0;
      for (int q = 0; q < 16; ++q)
        for (int k = 0; k < 4; ++k)
          if (pos0 + 4 * q + k < n) {
            const int32_t b = (w[q] >> (8 * k)) & 0xff;
            const int32_t z = (zw[q] >> (8 * k)) & 0xff;
            acc = (acc + static_cast<uint64_t>(static_cast<int64_t>(b - 2 * z))) * kPrime;
          }
    }
    // term = acc * P^(N - seg_end)
    if (chunk_end <= n) {
      if (tid == 0) sh.pc = pow_p(n - chunk_end);
      __syncthreads();
      term = acc * sh.pc * c_pow64[kThreads - 1 - tid];
    } else {
      term = acc * pow_p(n - seg_end);
    }
  }
  if (scr.prof && tid == 0) {
    atomicAdd(scr.prof + 4, static_cast<unsigned long long>(clock64() - t_mark));
    atomicAdd(scr.prof + 5, 1ull);
  }
  if (scr.trace && tid == 0) scr.trace[chunk * 12 + 9] = gtimer();
  // block reduction (mod 2^64, order-independent)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
  if (lane == 0) sh.red[warp] = term;
  __syncthreads();
  if (tid == 0) {
    uint64_t s = 0;
    for (int q = 0; q < kWarps; ++q) s += sh.red[q];
    atomicAdd(scr.accum, static_cast<unsigned long long>(s));
    __threadfence();
    const uint32_t done = atomicAdd(scr.finished, 1u) + 1;
    if (done == n_chunks) {
      const unsigned long long total = atomicAdd(scr.accum, 0ull);
      const unsigned long long h = pow_p(n) * seed + total;
      *scr.result = h;
      sh.pc = h;
      return true;
    }
  }
  return false;
}

}  // namespace fnv
}  // namespace mlck
