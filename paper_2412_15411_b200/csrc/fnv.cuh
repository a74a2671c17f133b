// fnv.cuh -- parallel, bit-exact FNV-1a-64 for the MLCK container trailer.
//
// Replaces the byte-serial moelab::fnv1a64 (digest.hpp:18-25), which is on
// both the pack path (serialize_record trailer, snapshot.hpp:142) and the
// verify path (parse_record, snapshot.hpp:156-163).
//
// Algebra.  h_{i+1} = (h_i ^ b_i) * P with P = 2^40 + 0x1b3.  Since b_i < 256
// the xor only touches the low byte u_i of h_i, so over a segment of L bytes
//   FNV_seg(H) = FNV_seg(u) + P^L (H - u),      u = H & 0xff,
// i.e. once every segment knows the low byte of the hash at its start, the
// segments hash independently (the real recurrence, started from h = u) and
// combine linearly:  h_N = P^N (H_0 & ~0xff) + sum_s P^(N - end_s) (g_s & ~0xff)
// + u_N.  The only sequential part is the 8-bit automaton
//   u' = ((u ^ b) * 0xb3) & 0xff,
// a T-function (bit j of u' depends on bits <= j of u only).
//
// Resolving the automaton.  Four look-back rounds resolve two state bits
// each.  In round r every 32-byte segment already knows its start bits
// < 2r and runs the automaton itself -- byte-serial, several start variants
// packed in SIMD lanes of one register -- from start bit 2r = 0 and 1.  Its
// effect on bits (2r, 2r+1) is the map
//   s0' = s0 ^ a,   s1' = s1 ^ (s0 ? b1 : b0)            ({a,b0,b1}, 3 bits)
// a family closed under composition.  Maps are scanned across the segments
// of a chunk with three ballots per warp (a is xor-linear; the b toggles are
// xor-linear once the prefix of a is known), across the warps of the CTA by a
// dedicated look-back warp, and across chunks by a decoupled look-back over
// one status word per chunk.  Rounds 0-1 need only the low 2/4 bits (the
// multiplier is 3 mod 16), so four variants share one register in 8-bit
// lanes; rounds 2-3 use 16-bit lanes (two variants per register).  Cost:
// 1.5 + 1.5 + 2.5 + 2.5 integer ops per byte, then ~4.5 for the final pass,
// split between the ALU and FMA pipes.
//
// Latency.  Each CTA keeps kSlots chunks in flight (their bytes in shared
// memory, loaded by TMA -- from the record, or straight from the record's
// sources in the fused snapshot -- or by cp.async for unaligned inputs) and
// its compute warps visit them round-robin; each compute thread owns kSegs
// consecutive 32-byte segments of a chunk, so the per-round scan and
// hand-off amortise over 128 bytes.  Every slot has its own look-back warp,
// which folds the warp maps of the slot's round, publishes it and looks back
// while the compute warps work on the other slots: a look-back has kSlots-1
// slot turns to complete before its result is needed.  The same warp
// issues the slot's TMA loads and, for copies, its TMA stores.
#pragma once

#include <cuda.h>

#include <cstddef>

#include "mlck_common.cuh"
#include "pack.cuh"

namespace mlck {
namespace fnv {

constexpr uint64_t kPrime = 0x100000001b3ull;
constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
#ifndef MLCK_FNV_SLOTS
#define MLCK_FNV_SLOTS 3
#endif
#ifndef MLCK_FNV_WARPS
#define MLCK_FNV_WARPS 16
#endif
// MLCK_FNV_MMA: final pass as int8 tensor-core dot products (see mma_pass);
// 0 = the byte-serial 64-bit recurrence.  MLCK_FNV_NOSHIFT: rounds 2-3 keep
// segments B, D in the odd byte lanes (no shift of the data word).
#ifndef MLCK_FNV_MMA
#define MLCK_FNV_MMA 1
#endif
#ifndef MLCK_FNV_ROUND0_LINEAR
#define MLCK_FNV_ROUND0_LINEAR 1
#endif
// MLCK_FNV_PACKED_MAPS: a thread's four segment maps of a round as three
// 4-bit vectors (a, b0, b1), composed and applied with bit-parallel prefix
// xors instead of map by map.
#ifndef MLCK_FNV_PACKED_MAPS
#define MLCK_FNV_PACKED_MAPS 1
#endif
#ifndef MLCK_FNV_NOSHIFT
#define MLCK_FNV_NOSHIFT 1
#endif
constexpr int kSlots = MLCK_FNV_SLOTS;         // chunks in flight per CTA
constexpr int kComputeWarps = MLCK_FNV_WARPS;  // + one look-back warp per slot
constexpr int kWarps = kComputeWarps + kSlots;
constexpr int kThreads = 32 * kWarps;
constexpr int kComputeThreads = 32 * kComputeWarps;
constexpr int kBarThreads = kComputeThreads + 32;  // named barriers: compute warps + one look-back warp
constexpr int kSegs = 4;                           // 32-byte segments per thread
constexpr int kThreadBytes = 32 * kSegs;
constexpr int kThreadWords = kThreadBytes / 4;
constexpr int kChunk = kComputeThreads * kThreadBytes;  // 65,536 bytes by default
constexpr int kRounds = 4;
static_assert(kSegs % 2 == 0, "segments are processed in pairs");
// One 64-bit look-back word per chunk, kStatusStride words apart (128 B: one
// L2 line each, the in-flight chunks' words in different lines; 256 B was
// 2 % slower, 64 B equal, 32 B and 8 B 8 % and 60 % slower on the fused
// snapshot).  The high half is the launch epoch, so the array is never
// cleared between launches.
#ifndef MLCK_FNV_STATUS_STRIDE
#define MLCK_FNV_STATUS_STRIDE 16
#endif
constexpr int kStatusStride = MLCK_FNV_STATUS_STRIDE;
constexpr uint32_t kSpinLimit = 1u << 24;  // watchdog: never hang the GPU

struct Scratch {
  unsigned long long* status;  // [n_chunks * kStatusStride] epoch-tagged words
  uint32_t epoch;              // this launch's tag (>= 1)
  unsigned long long* ticket;  // next chunk to hand out (zeroed per launch)
  uint32_t* witness;           // null, or the segment starts of every 128-byte row (written)
  unsigned long long* accum;   // sum of chunk terms (inverse-power frame)
  uint32_t* finished;          // completed-CTA counter
  uint32_t* ulast;             // low byte of the final hash
  uint32_t* error;             // watchdog tripped (look-back never resolved)
  uint32_t* sticky;            // ... and stays set until the host reads it
  unsigned long long* result;  // final 64-bit hash
  // optional profile counters (null = off): [0] look-back probes, [1] spin
  // re-reads, compute thread 0 of each CTA: [2] cycles in rounds, [3] cycles
  // waiting for look-back results, [4] final passes + refills, [6] other;
  // [5] chunks; look-back warps (lane 0): [8] idle at PUB, [9] probe loads,
  // [10] spins, [11] compose, [12] publish + hand-off, [13] total
  unsigned long long* prof;
  // optional per-chunk trace (null = off): 12 words per chunk, %globaltimer
  // ns at [0] round-0 start, [1+2r] map published, [2+2r] round resolved,
  // [9] final pass done, [10] smid
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

__host__ __device__ constexpr uint64_t pow_u64(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
__host__ __device__ constexpr uint64_t pow_p(uint64_t e) { return pow_u64(kPrime, e); }
// P is odd, so it is a unit mod 2^64 (Newton: x <- x (2 - P x), 5 doublings).
__host__ __device__ constexpr uint64_t inv_odd(uint64_t a) {
  uint64_t x = a;  // correct to 3 bits
  for (int i = 0; i < 5; ++i) x *= 2 - a * x;
  return x;
}
constexpr uint64_t kPrimeInv = inv_odd(kPrime);
static_assert(kPrime * kPrimeInv == 1ull, "P^-1 mod 2^64");
constexpr uint64_t kPow32 = pow_p(32);

static_assert(kWarps <= 32, "one look-back warp per slot");
// MLCK_FNV_LB_FIRST: the look-back warps are the CTA's first warps (1) or
// its last (0); compute thread t is threadIdx.x - kComputeTidBase.
#ifndef MLCK_FNV_LB_FIRST
#define MLCK_FNV_LB_FIRST 0
#endif
__host__ __device__ constexpr int lookback_warp(int s) { return MLCK_FNV_LB_FIRST ? s : kComputeWarps + s; }
// index of a compute warp among the compute warps, -1 for a look-back warp
__host__ __device__ constexpr int compute_warp(int warp) {
  return MLCK_FNV_LB_FIRST ? (warp >= kSlots ? warp - kSlots : -1) : (warp < kComputeWarps ? warp : -1);
}
constexpr int kComputeTidBase = MLCK_FNV_LB_FIRST ? 32 * kSlots : 0;
// MLCK_FNV_LB_ONE_COPY: the look-back warps share one copy of their code
// (the slot a run-time value) instead of one inlined copy per slot.
#ifndef MLCK_FNV_LB_ONE_COPY
#define MLCK_FNV_LB_ONE_COPY 1
#endif
// MLCK_FNV_COMPUTE_ONE_COPY: the same for the compute warps' turn code
// (per-slot state in shared memory and packed registers, fnv_compute1; it
// has the tensor-core final pass only, so MLCK_FNV_MMA=0 builds keep the
// unrolled loop).
#ifndef MLCK_FNV_COMPUTE_ONE_COPY
#define MLCK_FNV_COMPUTE_ONE_COPY MLCK_FNV_MMA
#endif

// P^-(c * kChunk) as a product of three table entries (init_constants)
__constant__ unsigned long long c_wchunk[3][1024];
__device__ __forceinline__ uint64_t chunk_weight(int64_t c) {
  return c_wchunk[0][c & 1023] * c_wchunk[1][(c >> 10) & 1023] * c_wchunk[2][(c >> 20) & 1023];
}

// One step of the real recurrence on h = hi:lo (b < 256):
// lo' = lo*0x1b3, hi' = hi*0x1b3 + carry + (lo << 8).
__device__ __forceinline__ void fnv_byte(uint32_t& lo, uint32_t& hi, uint32_t b) {
  lo ^= b;
  const uint64_t t = static_cast<uint64_t>(lo) * 0x1b3u;
  uint32_t f;
  asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(f) : "r"(lo), "r"(static_cast<uint32_t>(t >> 32)));
  asm("mad.lo.u32 %0, %1, 0x1b3, %2;" : "=r"(hi) : "r"(hi), "r"(f));
  lo = static_cast<uint32_t>(t);
}

// ---- 2-bit maps {a, b0, b1} -----------------------------------------------
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
// Warp-wide exclusive scan of per-lane maps (lane 0 first).  Returns the
// lane's exclusive prefix map; *total = the composition of all 32.
__device__ __forceinline__ uint32_t map_scan_warp(uint32_t m, uint32_t* total) {
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  const uint32_t bal_a = __ballot_sync(0xffffffffu, m & 1u);
  const uint32_t ea = __popc(bal_a & lt) & 1u;
  const uint32_t b0 = (m >> 1) & 1u, b1 = (m >> 2) & 1u;
  // toggle of state bit 1 here, for chunk-start s0 = 0 and s0 = 1
  const uint32_t bal0 = __ballot_sync(0xffffffffu, ea ? b1 : b0);
  const uint32_t bal1 = __ballot_sync(0xffffffffu, ea ? b0 : b1);
  *total = (__popc(bal_a) & 1u) | ((__popc(bal0) & 1u) << 1) | ((__popc(bal1) & 1u) << 2);
  return ea | ((__popc(bal0 & lt) & 1u) << 1) | ((__popc(bal1 & lt) & 1u) << 2);
}

// ---- thread data layout.  A thread owns kSegs = 4 consecutive 32-byte
// segments A, B, C, D of the chunk.  Once its bytes land they are
// byte-interleaved in place: word k = {A_k, B_k, C_k, D_k}, so a round feeds
// byte k of all four segments to its SIMD lanes without any byte selects.
static_assert(kSegs == 4, "one byte lane per segment");
__device__ __forceinline__ void interleave(uint32_t (&w)[kThreadWords]) {
  uint32_t o[kThreadWords];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t r0 = w[j], r1 = w[8 + j], r2 = w[16 + j], r3 = w[24 + j];
    const uint32_t t0 = __byte_perm(r0, r1, 0x5140), t1 = __byte_perm(r2, r3, 0x5140);
    const uint32_t t2 = __byte_perm(r0, r1, 0x7362), t3 = __byte_perm(r2, r3, 0x7362);
    o[4 * j] = __byte_perm(t0, t1, 0x5410);
    o[4 * j + 1] = __byte_perm(t0, t1, 0x7632);
    o[4 * j + 2] = __byte_perm(t2, t3, 0x5410);
    o[4 * j + 3] = __byte_perm(t2, t3, 0x7632);
  }
#pragma unroll
  for (int k = 0; k < kThreadWords; ++k) w[k] = o[k];
}

// ---- round r of one thread: the maps of its four segments on state bits
// (2r, 2r+1), given their start bits < 2r (st byte i = segment i).
// Rounds 0-1 track the state mod 4 / mod 16 only (0xb3 = 3 mod 16): one
// register per start variant, 8-bit lanes {A, B, C, D} (each < 46 after the
// multiply).  Rounds 2-3 track the full byte in 16-bit lanes {A, C} and
// {B, D}, one register per (pair, variant).
__device__ __forceinline__ void round_maps_low(const uint32_t (&w)[kThreadWords], uint32_t st, int r,
                                               uint32_t (&map)[kSegs]) {
  const uint32_t bit = 1u << (2 * r);
  const uint32_t M = r == 0 ? 0x03030303u : 0x0f0f0f0fu;
  const uint32_t lo = st & ((bit - 1u) * 0x01010101u);
  uint32_t x0 = lo, x1 = lo | (bit * 0x01010101u);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    x0 = ((x0 ^ w[k]) & M) * 3u;
    x1 = ((x1 ^ w[k]) & M) * 3u;
  }
  const uint32_t e0 = x0 >> (2 * r), e1 = x1 >> (2 * r);  // lane bit 0 = a / bit 1 = b
#pragma unroll
  for (int i = 0; i < kSegs; ++i)
    map[i] = ((e0 >> (8 * i)) & 3u) | (((e1 >> (8 * i)) & 2u) << 1);
}
// Round 0 without the automaton: bits 0 and 1 of the state evolve linearly
// (0xb3 = 3 mod 4: u0' = u0 ^ b0, u1' = u1 ^ b1 ^ u0 ^ b0).  Over a 32-byte
// segment (even length, so the start bit 0 cancels in the bit-1 sum):
//   a = parity of the b0 bits,  b0 = b1 = parity of the b1 bits ^ parity of
//   the b0 bits at odd positions.
__device__ __forceinline__ void round0_maps(const uint32_t (&w)[kThreadWords], uint32_t (&map)[kSegs]) {
  uint32_t xe = 0, xo = 0;
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    xe ^= w[k];
    xo ^= w[k + 1];
  }
  const uint32_t xa = xe ^ xo;
  const uint32_t t = (xa >> 1) ^ xo;  // lane bit 0: the bit-1 toggle
#pragma unroll
  for (int i = 0; i < kSegs; ++i) map[i] = ((xa >> (8 * i)) & 1u) | (((t >> (8 * i)) & 1u) * 6u);
}
__device__ __forceinline__ void round_maps_high(const uint32_t (&w)[kThreadWords], uint32_t st, int r,
                                                uint32_t (&map)[kSegs]) {
  const uint32_t bit = 1u << (2 * r);
  constexpr uint32_t M = 0x00ff00ffu;
  const uint32_t lo = st & ((bit - 1u) * 0x01010101u);
#if MLCK_FNV_NOSHIFT
  // {A, C} in byte lanes 0 and 2, {B, D} in lanes 1 and 3 of their own
  // register: B's product spills into lane 2 (masked off by the next step)
  // and never carries into lane 3, D's high bits fall off the word.
  uint32_t ac0 = lo & M, bd0 = lo & ~M;
  uint32_t ac1 = ac0 | (bit * 0x00010001u), bd1 = bd0 | (bit * 0x01000100u);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t y = w[k];
    ac0 = ((ac0 ^ y) & M) * 0xb3u;
    ac1 = ((ac1 ^ y) & M) * 0xb3u;
    bd0 = ((bd0 ^ y) & ~M) * 0xb3u;
    bd1 = ((bd1 ^ y) & ~M) * 0xb3u;
  }
  const uint32_t a0 = ac0 >> (2 * r), a1 = ac1 >> (2 * r), b0 = bd0 >> (2 * r + 8), b1 = bd1 >> (2 * r + 8);
#else
  uint32_t ac0 = lo & M, bd0 = (lo >> 8) & M;
  uint32_t ac1 = ac0 | (bit * 0x00010001u), bd1 = bd0 | (bit * 0x00010001u);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t y = w[k];
    const uint32_t yb = __umulhi(y, 1u << 24);  // y >> 8 on the FMA pipe
    ac0 = ((ac0 ^ y) & M) * 0xb3u;
    ac1 = ((ac1 ^ y) & M) * 0xb3u;
    bd0 = ((bd0 ^ yb) & M) * 0xb3u;
    bd1 = ((bd1 ^ yb) & M) * 0xb3u;
  }
  const uint32_t a0 = ac0 >> (2 * r), a1 = ac1 >> (2 * r), b0 = bd0 >> (2 * r), b1 = bd1 >> (2 * r);
#endif
  map[0] = (a0 & 3u) | ((a1 & 2u) << 1);
  map[1] = (b0 & 3u) | ((b1 & 2u) << 1);
  map[2] = ((a0 >> 16) & 3u) | (((a1 >> 16) & 2u) << 1);
  map[3] = ((b0 >> 16) & 3u) | (((b1 >> 16) & 2u) << 1);
}

// ---- packed segment maps.  A round's per-segment maps arrive as two "lane
// words": byte lane i of e0 holds segment i's a (bit 0) and b0 (bit 1), byte
// lane i of e1 its b1 (bit 1).
__device__ __forceinline__ uint32_t gather4(uint32_t v) { return (v * 0x01020408u) >> 24; }  // bits 0,8,16,24 -> 0..3
__device__ __forceinline__ uint32_t scatter4(uint32_t v) { return (v * 0x00204081u) & 0x01010101u; }  // inverse
__device__ __forceinline__ uint32_t prefix_xor4_excl(uint32_t v) {  // bit i = xor of bits < i
  v ^= v << 1;
  v ^= v << 2;
  return (v << 1) & 0xfu;
}
// The thread's composed map (bits 0-2) and, in bits 3-14, what the segment
// starts need after the look-back: X (s0 entering each segment for a thread
// start s0 = 0) and the s1 toggles T0 / T1 for thread start s0 = 0 / 1.
__device__ __forceinline__ uint32_t compose_lanes(uint32_t e0, uint32_t e1, uint32_t* packed) {
  const uint32_t A = gather4(e0 & 0x01010101u), B0 = gather4((e0 >> 1) & 0x01010101u),
                 B1 = gather4((e1 >> 1) & 0x01010101u);
  const uint32_t X = prefix_xor4_excl(A);
  const uint32_t T0 = (X & B1) | (~X & B0 & 0xfu), T1 = (~X & B1 & 0xfu) | (X & B0);
  *packed = (X << 3) | (T0 << 7) | (T1 << 11);
  return (__popc(A) & 1u) | ((__popc(T0) & 1u) << 1) | ((__popc(T1) & 1u) << 2);
}
// Segment start bits (byte lane i: bits 0-1) from the thread's start state s.
__device__ __forceinline__ uint32_t starts_lanes(uint32_t packed, uint32_t s) {
  const uint32_t s0 = s & 1u, s1 = (s >> 1) & 1u;
  const uint32_t X = (packed >> 3) & 0xfu, T = s0 ? (packed >> 11) & 0xfu : (packed >> 7) & 0xfu;
  const uint32_t S0 = X ^ (0u - s0) & 0xfu, S1 = prefix_xor4_excl(T) ^ ((0u - s1) & 0xfu);
  return scatter4(S0) | (scatter4(S1) << 1);
}
// The rounds' lane words.
__device__ __forceinline__ void round0_lanes(const uint32_t (&w)[kThreadWords], uint32_t* e0, uint32_t* e1) {
  uint32_t xe = 0, xo = 0;
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    xe ^= w[k];
    xo ^= w[k + 1];
  }
  const uint32_t xa = xe ^ xo, t = ((xa >> 1) ^ xo) & 0x01010101u;
  *e0 = (xa & 0x01010101u) | (t << 1);
  *e1 = t << 1;
}
__device__ __forceinline__ void round_lanes_low(const uint32_t (&w)[kThreadWords], uint32_t st, int r, uint32_t* e0,
                                                uint32_t* e1) {
  const uint32_t bit = 1u << (2 * r);
  const uint32_t M = r == 0 ? 0x03030303u : 0x0f0f0f0fu;
  const uint32_t lo = st & ((bit - 1u) * 0x01010101u);
  uint32_t x0 = lo, x1 = lo | (bit * 0x01010101u);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    x0 = ((x0 ^ w[k]) & M) * 3u;
    x1 = ((x1 ^ w[k]) & M) * 3u;
  }
  *e0 = x0 >> (2 * r);
  *e1 = x1 >> (2 * r);
}
__device__ __forceinline__ void round_lanes_high(const uint32_t (&w)[kThreadWords], uint32_t st, int r, uint32_t* e0,
                                                 uint32_t* e1) {
  static_assert(MLCK_FNV_NOSHIFT, "packed maps expect the shift-free high rounds");
  const uint32_t bit = 1u << (2 * r);
  constexpr uint32_t M = 0x00ff00ffu;
  const uint32_t lo = st & ((bit - 1u) * 0x01010101u);
  uint32_t ac0 = lo & M, bd0 = lo & ~M;
  uint32_t ac1 = ac0 | (bit * 0x00010001u), bd1 = bd0 | (bit * 0x01000100u);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t y = w[k];
    ac0 = ((ac0 ^ y) & M) * 0xb3u;
    ac1 = ((ac1 ^ y) & M) * 0xb3u;
    bd0 = ((bd0 ^ y) & ~M) * 0xb3u;
    bd1 = ((bd1 ^ y) & ~M) * 0xb3u;
  }
  *e0 = ((ac0 >> (2 * r)) & 0x00030003u) | ((bd0 >> (2 * r)) & 0x03000300u);
  *e1 = ((ac1 >> (2 * r)) & 0x00020002u) | ((bd1 >> (2 * r)) & 0x02000200u);
}

// Look-back for round r of `chunk` (one warp): lane l reads the 8
// predecessors base-8l .. base-8l-7 with all loads in flight.  If an entry
// nearer than the nearest inclusive one is not published yet, the whole
// window is re-read (one round trip per retry, not one per stale entry).
// The window's aggregates are folded without shuffles: with s0 known before
// each entry (an xor of the farther entries' a bits), every entry's toggle of
// s1 is known, and both fold to parities (two ballots).  Returns the chunk's
// two start bits.
#ifndef MLCK_FNV_PROBE
#define MLCK_FNV_PROBE 1
#endif
constexpr int kProbePerLane = MLCK_FNV_PROBE;  // window = 32 * kProbePerLane chunks
static_assert(kProbePerLane >= 1 && kProbePerLane <= 16, "lane masks hold up to 16 entries");
constexpr uint32_t kLaneEntries = (1u << kProbePerLane) - 1u;
__device__ __forceinline__ uint32_t look_back2_warp(const Scratch& scr, int64_t chunk, int r,
                                                    uint32_t seed2, long long* lap = nullptr) {
  const int lane = threadIdx.x & 31;
  auto mark = [&](int bucket) {
    if (lap) {
      const long long now = clock64();
      lap[bucket] += now - lap[0];
      lap[0] = now;
    }
  };
  uint32_t acc = 0;  // identity map: the nearer windows, applied last
  int64_t base = chunk - 1;
  uint32_t retries = 0;
  while (true) {
    if (scr.prof && lane == 0) atomicAdd(scr.prof + 0, 1ull);
    uint32_t am, b0m, b1m, incl_val;  // bit q: entry q's map bits (aggregates to apply)
    int first;
    while (true) {
      unsigned long long v[kProbePerLane];
#pragma unroll
      for (int q = 0; q < kProbePerLane; ++q) {
        const int64_t k = base - kProbePerLane * lane - q;
        v[q] = k < 0 ? 0ull : ld_relaxed_gpu_u64(scr.status + k * kStatusStride);
      }
      // nearest-first up to the first inclusive entry; stop at an unpublished one
      am = b0m = b1m = incl_val = 0;
      bool has_incl = false, blocked = false;
#pragma unroll
      for (int q = 0; q < kProbePerLane; ++q) {
        if (has_incl || blocked) continue;
        const int64_t k = base - kProbePerLane * lane - q;
        if (k < 0) {
          has_incl = true;
          incl_val = seed2;
          continue;
        }
        const uint32_t s = static_cast<uint32_t>(v[q]);
        if (static_cast<uint32_t>(v[q] >> 32) != scr.epoch || ((s >> 20) & 7u) <= static_cast<uint32_t>(r)) {
          blocked = true;
        } else if (((s >> 24) & 7u) > static_cast<uint32_t>(r)) {
          has_incl = true;
          incl_val = (s >> (12 + 2 * r)) & 3u;
        } else {
          const uint32_t m = s >> (3 * r);
          am |= (m & 1u) << q;
          b0m |= ((m >> 1) & 1u) << q;
          b1m |= ((m >> 2) & 1u) << q;
        }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, has_incl);
      const uint32_t blk = __ballot_sync(0xffffffffu, blocked);
      first = bal ? __ffs(bal) - 1 : 32;
      const int first_blk = blk ? __ffs(blk) - 1 : 32;
      if (first_blk >= first) break;  // everything up to the inclusive entry is published
      if (++retries > kSpinLimit) {   // never resolves: flag it and stop waiting
        if (lane == 0) atomicExch(scr.error, 1u);
        first = 0;
        break;
      }
#ifndef MLCK_FNV_BACKOFF_NS
#define MLCK_FNV_BACKOFF_NS 32
#endif
      if (MLCK_FNV_BACKOFF_NS) __nanosleep(MLCK_FNV_BACKOFF_NS);
    }
    mark(3);
    if (scr.prof && lane == 0 && retries) atomicAdd(scr.prof + 1, static_cast<unsigned long long>(retries));
    if (lane > first) am = b0m = b1m = 0;
    // s0 before entry q of this lane = s0_far ^ far ^ (xor of am above q)
    const uint32_t bal_a = __ballot_sync(0xffffffffu, __popc(am) & 1u);
    const uint32_t far = __popc(bal_a & ~((2u << lane) - 1u)) & 1u;  // lanes farther than this one
    uint32_t suf = am;  // suf_q = xor of am_j for j >= q
    suf ^= suf >> 1;
    suf ^= suf >> 2;
    suf ^= suf >> 4;
    if (kProbePerLane > 8) suf ^= suf >> 8;
    const uint32_t x = (suf >> 1) ^ (far ? kLaneEntries : 0u);  // s0 before entry, for s0 = 0 at the far end
    const uint32_t t0 = (x & b1m) | (~x & b0m);  // toggles of s1, far-end s0 = 0
    const uint32_t t1 = (~x & b1m) | (x & b0m);  // far-end s0 = 1
    const uint32_t bal0 = __ballot_sync(0xffffffffu, __popc(t0) & 1u);
    const uint32_t bal1 = __ballot_sync(0xffffffffu, __popc(t1) & 1u);
    // the window's map (farthest entry first)
    const uint32_t wmap = (__popc(bal_a) & 1u) | ((__popc(bal0) & 1u) << 1) | ((__popc(bal1) & 1u) << 2);
    if (first < 32) {
      const uint32_t res = map_apply(acc, map_apply(wmap, __shfl_sync(0xffffffffu, incl_val, first)));
      mark(4);
      return res;
    }
    acc = map_compose(acc, wmap);
    base -= 32 * kProbePerLane;
    retries = 0;
  }
}

// ---- shared memory ----------------------------------------------------------
// Thread t's 128 bytes are row t of its slot (8 granules of 16 bytes) in the
// TMA 128-byte swizzle: granule q of row t sits at 16 * (8t + (q ^ (t & 7))),
// so a tensor-map load lands the chunk in place and the lanes of a
// quarter-warp hit 8 distinct bank groups for every access pattern below.
// A slot holds kComputeThreads + 8 rows: a fused snapshot lands a source
// window shifted by 0-127 bytes against the record's rows, one row longer
// (one more 1 KiB swizzle atom).
constexpr int kGranules = kThreadBytes / 16;  // 8
constexpr int kSlotRows = kComputeThreads + 8;
struct alignas(1024) Shared {
  uint4 data[kSlots][kSlotRows * kGranules];       // 1024-byte aligned rows (TMA swizzle atoms)
  unsigned long long mbar[kSlots][kComputeWarps];  // the slot's bytes landed (per warp; [s][0] under TMA)
  unsigned long long res[kSlots];                  // look-back result of the slot's round
  unsigned long long sres[kSlots];                 // copies: the TMA stores have read the slot's rows
  unsigned long long rd[kSlots][kComputeWarps];    // fused: warp w - 1 has read its window (overhang)
  int64_t next[kSlots];                            // the slot's next chunk (ticket), -1 = none
  uint32_t shift[kSlots];                          // fused: the landed window's byte shift (0-127)
  uint32_t* witness;                               // Scratch::witness (read at the final pass)
  uint32_t wmap[kSlots][32];    // warp maps of the round (compute -> look-back)
  uint32_t wstart[kSlots][32];  // warp start bits (look-back -> compute)
  unsigned long long red[32];
#if MLCK_FNV_COMPUTE_ONE_COPY
  int64_t cw[kSlots][kComputeWarps];        // each compute warp's chunk of the slot
  uint32_t cst[kSlots][kComputeThreads];    // segment start bits per thread
  uint32_t ckeep[kSlots][kComputeThreads];  // pending round's maps per thread
#endif
#if MLCK_FNV_MMA
  uint2 wfrag[2][4][32];        // mma_pass B fragments: [data | automaton][k-block][lane]
  unsigned long long kpos[32][4];  // mma_pass epilogue weights per lane
#endif
};
// + 1 KiB of slack: the kernel aligns Shared to 1 KiB inside its dynamic
// shared memory (the TMA swizzle pattern is anchored to 1 KiB boundaries)
constexpr size_t kSmemBytes = sizeof(Shared) + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");
static_assert(sizeof(uint4) * kSlotRows * kGranules % 1024 == 0, "slots keep the swizzle alignment");

__device__ __forceinline__ int granule(int t, int q) { return kGranules * t + (q ^ (t & 7)); }

// ---- copies (fused snapshot, replicas) ---------------------------------------
// The hash kernel can also write the bytes it hashes: every chunk's rows go
// from shared memory to up to pack::kMaxDst destinations by TMA tensor
// stores (record-row maps; rows past the last full row are clipped and the
// partial last row is stored by its thread), and, for a fused snapshot,
// arrive from the record's sources instead of the record: chunk c of run r
// is rows row0 + 512 (c - c0) ... of source map `map`, shifted by `delta`
// bytes (a source is not 128-aligned against the record), rows 512-519 of
// the slot taking the window's overhang.  Chunks that straddle segments
// (headers, entry boundaries, the record's partial last chunk) are
// pre-gathered whole into a patch buffer, which is one more source map.
constexpr int kMaxSrc = 6;
struct Run {
  int64_t c0, c1;  // record chunks [c0, c1)
  int64_t row0;    // source row of chunk c0
  int32_t map, delta;
};
struct Copy {
  CUtensorMap src[kMaxSrc][2];      // [map][0]: 256-row boxes, [map][1]: 8-row boxes
  CUtensorMap dst[pack::kMaxDst];   // record-row maps of the destinations (256-row boxes)
  uint8_t* dst_ptr[pack::kMaxDst];  // the same, for the partial last row
  int n_dst;                        // 0: hash only
  const Run* runs;                  // fused: sorted by c0, covering every chunk; null otherwise
  int n_runs;
};



__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared.b64 st, [%0]; }" ::"r"(smem_addr(m)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* m, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(tx) : "memory");
}
#ifndef MLCK_MBAR_SUSPEND_NS
#define MLCK_MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* m, uint32_t parity) {
#if MLCK_MBAR_SUSPEND_NS
  // the waiting warp is suspended until the phase completes (or the hint
  // expires) instead of spinning on issue slots the compute warps need
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1, %2; @!p bra W; }" ::"r"(
          smem_addr(m)),
      "r"(parity), "n"(MLCK_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
          smem_addr(m)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(unsigned long long* m) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_addr(m)) : "memory");
}

// Byte path (unaligned input, the record's tail, a thread straddling
// segments): thread t's bytes into its granules, zero past n.
template <typename ByteAt>
__device__ __forceinline__ void load_thread_bytes(Shared& sh, int slot, int t, ByteAt byte_at, bool arrive = true) {
  uint4* dst = sh.data[slot];
  for (int q = 0; q < kGranules; ++q) {
    uint32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x = 0;
      for (int k = 0; k < 4; ++k) x |= static_cast<uint32_t>(byte_at(16 * q + 4 * i + k)) << (8 * k);
      v[i] = x;
    }
    dst[granule(t, q)] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  if (arrive) mbar_arrive(&sh.mbar[slot][t >> 5]);
}

// Tensor-map load of `rows` x 128 bytes starting at record row `row` into
// swizzled rows at dst (rows past the tensor arrive as zeros).
// MLCK_FNV_L2HINT: TMA loads and stores of the streamed bytes carry an
// L2 evict-first policy (the look-back words and tables stay resident).
#ifndef MLCK_FNV_L2HINT
#define MLCK_FNV_L2HINT 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_rows(void* dst, const CUtensorMap* map, int32_t row,
                                              unsigned long long* mbar) {
#if MLCK_FNV_L2HINT
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(smem_addr(mbar)), "l"(l2_evict_first())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(smem_addr(mbar))
      : "memory");
#endif
}
#ifndef MLCK_FNV_BOX_ROWS
#define MLCK_FNV_BOX_ROWS 256
#endif
constexpr int kTmaBoxRows = MLCK_FNV_BOX_ROWS;  // rows per TMA box (a divisor of kComputeThreads)
static_assert(kComputeThreads % kTmaBoxRows == 0, "whole boxes per chunk");
// Tensor-map store of `rows` x 128 bytes of swizzled rows at src to record
// row `row` (rows past the tensor are clipped); bulk async-group.
__device__ __forceinline__ void tma_store_rows(const CUtensorMap* map, int32_t row, const void* src) {
#if MLCK_FNV_L2HINT
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::
                   "l"(reinterpret_cast<uint64_t>(map)),
               "r"(0), "r"(row), "r"(smem_addr(src)), "l"(l2_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(0), "r"(row), "r"(smem_addr(src))
               : "memory");
#endif
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Fused snapshot: chunk `chunk` of run `r` into `slot` (one thread; one
// mbarrier arrival with the byte count): 512 source rows, plus the 8-row atom
// of the overhang when the window is shifted.
__device__ __forceinline__ void tma_load_src(Shared& sh, int slot, const Copy& cp, const Run& r, int64_t chunk) {
  unsigned long long* mb = &sh.mbar[slot][0];
  const uint32_t delta = static_cast<uint32_t>(r.delta);
  const int32_t row = static_cast<int32_t>(r.row0 + static_cast<int64_t>(kComputeThreads) * (chunk - r.c0));
  sh.shift[slot] = delta;  // released to the waiters by the arrival below
  fence_async_shared();
  mbar_arrive_expect_tx(mb, (kComputeThreads + (delta ? 8 : 0)) * kThreadBytes);
  for (int b = 0; b < kComputeThreads / kTmaBoxRows; ++b)
    tma_load_rows(&sh.data[slot][kGranules * kTmaBoxRows * b], &cp.src[r.map][0], row + kTmaBoxRows * b, mb);
  if (delta) tma_load_rows(&sh.data[slot][kGranules * kComputeThreads], &cp.src[r.map][1], row + kComputeThreads, mb);
}
// The run holding record chunk c (warp-collective: a 32-ary search over the
// run starts, one load per lane per level).
__device__ __forceinline__ Run find_run(const Copy& cp, int64_t c) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = cp.n_runs;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) / 32;
    const int i = lo + lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, i < hi && cp.runs[i].c0 <= c);
    lo += (31 - __clz(m)) * step;  // lane 0's run starts at or before c
    hi = min(hi, lo + step);
  }
  return cp.runs[lo];
}
// The slot's chunk out to every destination (one thread; the caller waits
// for the TMA to have read the rows before the compute warps rewrite them).
__device__ __forceinline__ void tma_store_chunk(const Shared& sh, int slot, const Copy& cp, int64_t chunk,
                                                uint64_t rows_full) {
  const uint64_t row0 = static_cast<uint64_t>(chunk) * kComputeThreads;
  for (int d = 0; d < cp.n_dst; ++d)
    for (int b = 0; b < kComputeThreads / kTmaBoxRows; ++b)
      if (row0 + kTmaBoxRows * b < rows_full)
        tma_store_rows(&cp.dst[d], static_cast<int32_t>(row0 + kTmaBoxRows * b),
                       &sh.data[slot][kGranules * kTmaBoxRows * b]);
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// The chunk of `slot` by one thread: the 256-row boxes that start inside the
// map's rows_full full rows (the compute threads write the rest), one
// mbarrier arrival with their byte count.
__device__ __forceinline__ void tma_load_chunk(Shared& sh, int slot, const CUtensorMap* map, int64_t chunk,
                                               uint64_t rows_full) {
  unsigned long long* mb = &sh.mbar[slot][0];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint64_t row0 = static_cast<uint64_t>(chunk) * kComputeThreads;
  int boxes = 0;
#pragma unroll
  for (int b = 0; b < kComputeThreads / kTmaBoxRows; ++b) boxes += row0 + kTmaBoxRows * b < rows_full;
  mbar_arrive_expect_tx(mb, boxes * kTmaBoxRows * kThreadBytes);
  for (int b = 0; b < boxes; ++b)
    tma_load_rows(&sh.data[slot][kGranules * kTmaBoxRows * b], map, static_cast<int32_t>(row0 + kTmaBoxRows * b), mb);
}


// Thread t's bytes of `chunk` of a packed buffer into its slot granules,
// zero past n; one arrival on the warp's mbarrier when they have landed.
__device__ __forceinline__ void load_thread(Shared& sh, int slot, int t, const uint8_t* data,
                                            uint64_t n, int64_t chunk) {
  const uint64_t p = static_cast<uint64_t>(chunk) * kChunk + static_cast<uint64_t>(t) * kThreadBytes;
  if (p + kThreadBytes <= n && (reinterpret_cast<uintptr_t>(data) & 15u) == 0) {
    uint4* dst = sh.data[slot];
#pragma unroll
    for (int q = 0; q < kGranules; ++q) cp_async16(dst + granule(t, q), data + p + 16 * q);
    cp_async_arrive(&sh.mbar[slot][t >> 5]);
  } else {
    load_thread_bytes(sh, slot, t, [&](int i) -> uint32_t { return p + i < n ? data[p + i] : 0u; });
  }
}

__device__ __forceinline__ void write_thread_rows(uint4* rows, int t, const uint32_t (&w)[kThreadWords]) {
#pragma unroll
  for (int q = 0; q < kGranules; ++q) rows[granule(t, q)] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}
__device__ __forceinline__ void read_thread_rows(const uint4* rows, int t, uint32_t (&w)[kThreadWords]) {
#pragma unroll
  for (int q = 0; q < kGranules; ++q) {
    const uint4 v = rows[granule(t, q)];
    w[4 * q] = v.x;
    w[4 * q + 1] = v.y;
    w[4 * q + 2] = v.z;
    w[4 * q + 3] = v.w;
  }
}
__device__ __forceinline__ void write_thread(Shared& sh, int slot, int t, const uint32_t (&w)[kThreadWords]) {
#pragma unroll
  for (int q = 0; q < kGranules; ++q)
    sh.data[slot][granule(t, q)] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}
__device__ __forceinline__ void read_thread(const Shared& sh, int slot, int t, uint32_t (&w)[kThreadWords]) {
#pragma unroll
  for (int q = 0; q < kGranules; ++q) {
    const uint4 v = sh.data[slot][granule(t, q)];
    w[4 * q] = v.x;
    w[4 * q + 1] = v.y;
    w[4 * q + 2] = v.z;
    w[4 * q + 3] = v.w;
  }
}
// The thread's 128 bytes from its unaligned gather window (phase 1..15):
// nine 128-bit loads, then a word select (warp-uniform in practice: the
// windows of a segment share its alignment) and a byte funnel, in place.
#if MLCK_FNV_MMA
// ---- final pass on the tensor cores.  With d_p = (u_p ^ b_p) - u_p, where
// u_p is the low byte of the hash before byte p, the recurrence unrolls to
//   h_N = P^N h_0 + sum_p P^(N-p) d_p,   d_p = b_p - 2 (u_p & b_p),
// two dot products of byte vectors with powers of P.  Splitting each weight
// into eight 8-bit limbs turns them into u8 x u8 -> s32 MMAs.  Per warp
// (128 segments of 32 bytes, span end E_w) the MMA computes
//   C[j][n] = sum_seg x_{seg,j} limb_n(P^(E_w - end_seg))  (j = byte in segment)
// with A = the interleaved words as they sit in shared memory: word j of a
// thread holds byte j of its four segments, i.e. four consecutive k of one
// row of A.  Rows are permuted so a lane's a0/a1 of both row blocks are one
// 16-byte granule: row g <-> byte 4g + 2rb, row g + 8 <-> byte 4g + 2rb + 1.
// k-block kb takes a0 from thread 8kb + 2q and a2 from thread 8kb + 2q + 1
// (conflict-free with the 9-granule stride).  The automaton vector uses the
// limbs of -2 P^(...) into the same accumulators; the epilogue applies
// P^(32 - j) and the limb shifts.  Every accumulator entry stays below
// 2 * 128 * 255 * 255 < 2^25.
__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// segment (of the warp's 128) behind k of k-block kb
__host__ __device__ constexpr int mma_segment(int kb, int k) {
  return 32 * kb + 8 * ((k & 15) >> 2) + ((k >> 4) << 2) + (k & 3);
}
// One pass over the warp's 32 threads' words of a chunk's rows (after
// __syncwarp); wfrag = the B fragment tables.
__device__ __forceinline__ void mma_pass_rows(const uint4* rows, const uint2 (*wfrag)[4][32], int warp, int lane,
                                              int tab, int (&acc)[2][4]) {
  const int g = lane >> 2, q = lane & 3, t0 = 32 * warp + 2 * q;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    const uint4 lo = rows[granule(t0 + 8 * kb, g)];
    const uint4 hi = rows[granule(t0 + 8 * kb + 1, g)];
    const uint2 b = wfrag[tab][kb][lane];
    mma_u8(acc[0], lo.x, lo.y, hi.x, hi.y, b.x, b.y);
    mma_u8(acc[1], lo.z, lo.w, hi.z, hi.w, b.x, b.y);
  }
}
__device__ __forceinline__ void mma_pass(const Shared& sh, int slot, int warp, int lane, int tab,
                                         int (&acc)[2][4]) {
  mma_pass_rows(sh.data[slot], sh.wfrag, warp, lane, tab, acc);
}
// Tables (once per CTA): B fragments and epilogue weights.
template <typename S>
__device__ __forceinline__ void mma_tables(S& sh, int tid) {
  if (tid < 2 * 4 * 32) {
    const int tab = tid >> 7, kb = (tid >> 5) & 3, lane = tid & 31, n = lane >> 2, q = lane & 3;
    uint32_t b[2] = {0, 0};
    for (int h = 0; h < 2; ++h)
      for (int e = 0; e < 4; ++e) {
        const int seg = mma_segment(kb, 16 * h + 4 * q + e);
        uint64_t wgt = pow_u64(kPrime, 32ull * (127 - seg));
        if (tab) wgt *= ~1ull;  // -2 P^(...) mod 2^64
        b[h] |= static_cast<uint32_t>((wgt >> (8 * n)) & 0xffu) << (8 * e);
      }
    sh.wfrag[tab][kb][lane] = make_uint2(b[0], b[1]);
  } else if (tid < 2 * 4 * 32 + 32 * 4) {
    const int i = tid - 256, lane = i >> 2, m = i & 3, g = lane >> 2, q = lane & 3;
    sh.kpos[lane][m] = pow_u64(kPrime, 32 - (4 * g + m)) << (16 * q);
  }
}
// The warp's sum_p P^(E_w - p) d_p (this lane's share) from the accumulators.
template <typename S>
__device__ __forceinline__ uint64_t mma_epilogue(const S& sh, int lane, const int (&acc)[2][4]) {
  uint64_t t = 0;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb) {
    const uint64_t v0 = static_cast<uint64_t>(static_cast<uint32_t>(acc[rb][1])) * 256u +
                        static_cast<uint32_t>(acc[rb][0]);
    const uint64_t v1 = static_cast<uint64_t>(static_cast<uint32_t>(acc[rb][3])) * 256u +
                        static_cast<uint32_t>(acc[rb][2]);
    t += v0 * sh.kpos[lane][2 * rb] + v1 * sh.kpos[lane][2 * rb + 1];
  }
  return t;
}
// The automaton from the segment starts (st byte i = segment i), leaving
// u & b in place of the bytes: w[k] <- u_k & w[k] for all four segments.
__device__ __forceinline__ void automaton_and(uint32_t (&w)[kThreadWords], uint32_t st) {
  constexpr uint32_t M = 0x00ff00ffu;
  uint32_t ac = st & M, bd = st & ~M;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t y = w[k];
    w[k] = ((ac & M) | (bd & ~M)) & y;
    ac = ((ac ^ y) & M) * 0xb3u;
    bd = ((bd ^ y) & ~M) * 0xb3u;
  }
}
// automaton_and that also returns the state after each segment's last
// byte (byte lane i = segment i): the witness check of fnv_witness_kernel.
__device__ __forceinline__ uint32_t automaton_and_ends(uint32_t (&w)[kThreadWords], uint32_t st) {
  constexpr uint32_t M = 0x00ff00ffu;
  uint32_t ac = st & M, bd = st & ~M;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t y = w[k];
    w[k] = ((ac & M) | (bd & ~M)) & y;
    ac = ((ac ^ y) & M) * 0xb3u;
    bd = ((bd ^ y) & ~M) * 0xb3u;
  }
  return (ac & M) | (bd & ~M);
}

// ---- verification against a witness.  A record hashed by fnv_kernel can
// keep the low byte of the hash at the start of every 32-byte segment (the
// segment starts its look-back resolved; one u32 per 128-byte row, byte i =
// segment i).  Re-hashing the record then needs no rounds and no look-back:
// every row runs the automaton from its witnessed starts, the two dot
// products follow on the tensor cores, and each segment's end state is
// compared with the next segment's witnessed start.  If every comparison
// holds the witnessed starts are the true ones (induction from the seed's
// low byte), so the sum is exactly FNV-1a-64 of the bytes now in memory;
// if one fails (a stale witness, bytes changed) the caller hashes the
// record with fnv_kernel.  Either way the result is the exact hash.
// (fnv_witness_kernel in kernels.cu)
#endif

// Record row t of a window landed `delta` bytes into the slot (0 < delta <
// 128): linear granules 8t + delta/16 ... + 8 of the swizzled rows (rows t
// and t + 1; a quarter-warp's lanes still hit 8 bank groups), then a byte
// funnel by delta % 16 (uniform over the chunk).
__device__ __forceinline__ void read_thread_shifted(const Shared& sh, int slot, int t, uint32_t delta,
                                                   uint32_t (&w)[kThreadWords]) {
  const int a = static_cast<int>(delta >> 4);
  uint32_t x[kThreadWords + 4];
#pragma unroll
  for (int q = 0; q <= kGranules; ++q) {
    const int l = a + q, r = t + (l >> 3);
    const uint4 v = sh.data[slot][granule(r, l & 7)];
    x[4 * q] = v.x;
    x[4 * q + 1] = v.y;
    x[4 * q + 2] = v.z;
    x[4 * q + 3] = v.w;
  }
  const uint32_t ph = delta & 15u;
  const uint32_t sel = 0x3210u + 0x1111u * (ph & 3u);  // bytes (ph&3) .. (ph&3)+3 of a:b
  switch (ph >> 2) {
#define MLCK_REALIGN(W)                                                      \
  case W:                                                                    \
    _Pragma("unroll") for (int i = 0; i < kThreadWords; ++i) x[i] = __byte_perm(x[i + W], x[i + W + 1], sel); \
    break;
    MLCK_REALIGN(0)
    MLCK_REALIGN(1)
    MLCK_REALIGN(2)
    MLCK_REALIGN(3)
#undef MLCK_REALIGN
  }
#pragma unroll
  for (int i = 0; i < kThreadWords; ++i) w[i] = x[i];
}

}  // namespace fnv
}  // namespace mlck
