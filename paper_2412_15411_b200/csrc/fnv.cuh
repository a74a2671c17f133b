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
constexpr int kThreads = 256;
constexpr int kBytesPerThread = 64;  // two 32-position groups
constexpr int kChunk = kThreads * kBytesPerThread;
constexpr int kWarps = kThreads / 32;

struct Scratch {
  uint32_t* status;            // [n_chunks] look-back words (zeroed per launch)
  uint32_t* ticket;            // chunk dispatch counter (zeroed per launch)
  unsigned long long* accum;   // sum of chunk terms
  uint32_t* finished;          // completed-chunk counter
  unsigned long long* result;  // final 64-bit hash
};

// P^(64 k) for k = 0..kThreads-1, written by init_constants() (kernels.cu).
__constant__ unsigned long long c_pow64[kThreads];

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

// Look-back over predecessor chunks for bit level j.  Executed by one full
// warp; returns the start bit (state bit j before the chunk's first byte).
__device__ __forceinline__ uint32_t look_back(const uint32_t* status, int64_t chunk, int j,
                                              uint32_t seed_bit) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  int64_t base = chunk - 1;
  while (true) {
    const int64_t k = base - lane;
    bool incl;
    uint32_t bit;
    if (k < 0) {
      incl = true;
      bit = seed_bit;
    } else {
      uint32_t s;
      do {
        s = ld_relaxed_gpu(status + k);
      } while (((s >> 16) & 0xf) <= static_cast<uint32_t>(j));
      incl = ((s >> 20) & 0xf) > static_cast<uint32_t>(j);
      bit = incl ? (s >> (8 + j)) & 1u : (s >> j) & 1u;
    }
    const uint32_t incl_mask = __ballot_sync(0xffffffffu, incl);
    if (incl_mask) {
      const int first = __ffs(incl_mask) - 1;
      const uint32_t bits = __ballot_sync(0xffffffffu, bit && lane <= first);
      return acc ^ (__popc(bits) & 1u);
    }
    acc ^= __popc(__ballot_sync(0xffffffffu, bit)) & 1u;
    base -= 32;
  }
}

// Block-level FNV contribution of one kChunk-byte chunk.  Every thread
// passes its 64 bytes (16 little-endian words, positions thread*64 ..),
// already zero-padded past `n`.  The chunk's term P^(N-end) * H is
// atomically accumulated into scr.accum; the last chunk to finish writes the
// final hash into scr.result (and sh.pc) and returns true in thread 0.
struct SharedState {
  uint32_t warp_par[kWarps];
  uint32_t start_bit;
  unsigned long long pc;  // P^(N - chunk_end) for the chunk
  unsigned long long red[kWarps];
};

__device__ inline bool chunk_contribution(const uint32_t (&w)[16], int64_t chunk, uint64_t n,
                                          uint64_t seed, const Scratch& scr, uint64_t n_chunks,
                                          SharedState& sh) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  uint32_t B[2][8], Y[2][8];
  Carries car[2];
  to_planes(w, B[0]);
  to_planes(w + 8, B[1]);
  // Positions past n must not toggle: their bytes are zero, so B=0 there; the
  // automaton runs on but d_i is forced to zero below and nothing later reads
  // these states (only the final chunk is padded).

  uint32_t status = 0;  // owner's view (thread 0)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t T[2], I[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      T[g] = B[g][j] ^ level_r(j, Y[g], car[g]);
      I[g] = prefix_xor(T[g]);
    }
    I[1] ^= bcast(I[0] >> 31);
    const uint32_t par = I[1] >> 31;
    const uint32_t ballot = __ballot_sync(0xffffffffu, par);
    const uint32_t lane_excl = __popc(ballot & ((1u << lane) - 1u)) & 1u;
    if (lane == 0) sh.warp_par[warp] = __popc(ballot) & 1u;
    __syncthreads();
    uint32_t warp_excl = 0, agg = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const uint32_t p = sh.warp_par[q];
      warp_excl ^= (q < warp) ? p : 0u;
      agg ^= p;
    }
    if (warp == 0) {
      const uint32_t seed_bit = static_cast<uint32_t>(seed >> j) & 1u;
      // status word: [7:0] aggregate bits, [15:8] inclusive bits,
      // [19:16] levels with aggregate published, [23:20] levels inclusive
      if (lane == 0) {
        status = (status & ~(0xfu << 16)) | (agg << j) | (static_cast<uint32_t>(j + 1) << 16);
        st_relaxed_gpu(scr.status + chunk, status);
      }
      const uint32_t start = look_back(scr.status, chunk, j, seed_bit);
      if (lane == 0) {
        status = (status & ~(0xfu << 20)) | ((start ^ agg) << (8 + j)) |
                 (static_cast<uint32_t>(j + 1) << 20);
        st_relaxed_gpu(scr.status + chunk, status);
        sh.start_bit = start;
      }
    }
    __syncthreads();
    const uint32_t ts = bcast(sh.start_bit ^ warp_excl ^ lane_excl);
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const uint32_t U = I[g] ^ T[g] ^ ts;  // state bit j before each position
      Y[g][j] = U ^ B[g][j];
      level_carry(j, Y[g], car[g]);
    }
  }

  // ---- phase B: d_i = b_i - 2 (u_i & b_i); z = u & b = b & ~y
  uint32_t zw[16];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint32_t Z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) Z[j] = B[g][j] & ~Y[g][j];
    from_planes(Z, zw + 8 * g);
  }
  const uint64_t pos0 = static_cast<uint64_t>(chunk) * kChunk + static_cast<uint64_t>(tid) * kBytesPerThread;
  uint64_t acc = 0;
  uint64_t seg_end = pos0 + kBytesPerThread;
  if (pos0 + kBytesPerThread <= n) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t b = (w[q] >> (8 * k)) & 0xff;
        const int32_t z = (zw[q] >> (8 * k)) & 0xff;
        acc = (acc + static_cast<uint64_t>(static_cast<int64_t>(b - 2 * z))) * kPrime;
      }
    }
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
  const uint64_t chunk_end = static_cast<uint64_t>(chunk + 1) * kChunk;
  uint64_t term;
  if (chunk_end <= n) {
    if (tid == 0) sh.pc = pow_p(n - chunk_end);
    __syncthreads();
    term = acc * sh.pc * c_pow64[kThreads - 1 - tid];
  } else {
    term = acc * pow_p(n - seg_end);
  }
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
