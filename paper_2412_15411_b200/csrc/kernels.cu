// kernels.cu -- sm_100a kernels of the checkpoint data path and their
// host-side launchers (declared in kernels.cuh).
#define MLCK_DEFINE_KERNELS 1
#include "adam.cuh"
#include "codec.cuh"
#include "fnv.cuh"
#include "kernels.cuh"
#include "pack.cuh"

#include <algorithm>
#include <mutex>
#include <cstring>
#include <string>

namespace mlck {

// ---------------------------------------------------------------- FNV (K2)
namespace {

using fnv::kSlots;
// Hand-offs: PUB(s) is a named barrier (compute warps arrive, the look-back
// warp of slot s waits for all of them); the result goes back through the
// mbarrier res[s] (one arrival per round), so compute warps never wait for
// each other -- a fast warp moves on to the next slot's turn.
__device__ __forceinline__ int bar_pub(int s) { return 1 + s; }
// Copies: STORE(s) -- the compute warps have the slot's record-aligned rows
// in shared memory (the look-back warp then issues the TMA stores; the
// compute warps wait on sres[s] before overwriting the rows in round 1).
__device__ __forceinline__ int bar_store(int s) { return 1 + fnv::kSlots + s; }

// Profile laps of one thread's clock (kProf only): consecutive buckets, so
// they add up to the loop time.
template <bool kProf, int N>
struct Laps {
  long long t[N] = {};
  long long last = 0;
  __device__ __forceinline__ void start() {
    if (kProf) last = clock64();
  }
  __device__ __forceinline__ void mark(int b) {
    if (kProf) {
      const long long now = clock64();
      t[b] += now - last;
      last = now;
    }
  }
};

// ---- tcgen05 helpers: the chunk-wide dot products of the witness verifier
// (fnv_witness_tc_kernel).  Per chunk, a 128 x 16 x 512 u8 MMA: A = the
// chunk's 512 rows in shared memory (M = the 128 byte positions of a row,
// K = the row: the TMA's 128-byte-swizzled rows are the canonical MN-major
// SWIZZLE_128B operand), B = the 8-bit limbs of P^-(128 k) (or of
// -2 P^-(128 k)) for row k, s32 accumulators (< 2^26) in TMEM.
constexpr int kTcN = 16;  // MMA N (limbs 0-7 used, 8-15 zero)
__device__ uint8_t g_tcw[2][fnv::kComputeThreads][kTcN];  // B tables (init_constants)

__device__ __forceinline__ bool mbar_try(unsigned long long* m, uint32_t parity) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok)
               : "r"(fnv::smem_addr(m)), "r"(parity)
               : "memory");
  return ok != 0;
}
// A bounded wait: a protocol error ends the kernel with the record marked
// unverified (the caller re-hashes it) instead of hanging the GPU.
__device__ __forceinline__ bool mbar_wait_tc(unsigned long long* m, uint32_t parity, volatile uint32_t* abort) {
  for (uint32_t n = 1;; ++n) {
    if (mbar_try(m, parity)) return true;
    if ((n & 255u) == 0 && (*abort || n > (1u << 24))) {
      *abort = 1;
      return false;
    }
  }
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// shared-memory matrix descriptors (sm_100 layout: start >> 4 @0, LBO >> 4
// @16, SBO >> 4 @32, version 1 @46, layout type @61)
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}
// kind::i8, u8 x u8 -> s32, A and B MN-major, N = 16, M = 128
constexpr uint32_t kTcIdesc = (2u << 4) | (1u << 15) | (1u << 16) | ((kTcN >> 3) << 17) | ((128 >> 4) << 24);
// D[tmem] (+)= A[128 x 512 rows at a] . B[512 x 16 at b]: 16 MMAs of K = 32
// (accumulate = 0: the first overwrites D)
__device__ __forceinline__ void tc_chunk_mma(uint32_t d_tmem, uint32_t a, uint32_t b, uint32_t accumulate = 0) {
#pragma unroll
  for (int k = 0; k < fnv::kComputeThreads / 32; ++k) {
    // A: SWIZZLE_128B MN-major, 8-row atoms 1 KiB apart, K-step = 32 rows (4 KiB)
    const uint64_t da = tc_desc(a + 4096u * k, 0, 1024, 2);
    // B: no swizzle, MN-major, core matrices of 8 rows x 16 B, 128 B apart along K
    const uint64_t db = tc_desc(b + 512u * k, 128, 0, 0);
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
        "l"(da), "l"(db), "r"(kTcIdesc), "r"(k | accumulate)
        : "memory");
  }
}
__device__ __forceinline__ void tc_commit(unsigned long long* m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(fnv::smem_addr(m))
               : "memory");
}
// 8 columns of this warp's 32 TMEM lanes
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}


// Compute warps: per slot turn, take the look-back result of the round
// published on the previous turn, then (after round 3) hash the slot's bytes
// and refill it, else compute and publish the next round.
template <bool kProf, bool kGather>
__device__ __forceinline__ uint64_t fnv_compute(fnv::Shared& sh, const uint8_t* data, uint64_t n,
                                                const fnv::Scratch& scr, int64_t n_chunks,
                                                const int64_t (&first)[kSlots], int64_t stride,
                                                const fnv::Copy& cp, bool tma) {
  using namespace fnv;
  // TMA mode: the slot's look-back warp loads whole chunks through the tensor
  // map; rows at or past the last full 128-byte row are written here
  const uint64_t rows_full = n / kThreadBytes;
  const int tid = static_cast<int>(threadIdx.x) - kComputeTidBase, warp = tid >> 5, lane = tid & 31;
#if MLCK_FNV_MMA
  // P^-(end of the warp's span in the chunk)
  const uint64_t pinv_t = pow_u64(kPrimeInv, static_cast<uint64_t>(kThreadBytes) * 32 * (warp + 1));
#else
  const uint64_t pinv_t = pow_u64(kPrimeInv, static_cast<uint64_t>(kThreadBytes) * (tid + 1));
#endif
  int64_t chunk[kSlots];
  int rnd[kSlots];
  bool pend[kSlots];
  uint32_t st[kSlots];    // segment start bits, byte i = segment i
  uint32_t keep[kSlots];  // pending round: lane exclusive map [0,3), segment maps 0..kSegs-2 above
  uint32_t par = 0;       // data mbarrier phase parity per slot
  uint32_t rpar = 0;      // result mbarrier phase parity per slot
  uint32_t spar = 0;      // copies: store mbarrier phase parity per slot
  uint32_t rdpar = 0;     // fused: neighbour-read mbarrier phase parity per slot
  const bool copy = cp.n_dst > 0;
  uint64_t acc = 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    chunk[s] = first[s];
    rnd[s] = 0;
    pend[s] = false;
    st[s] = 0;
    keep[s] = 0;
    if (chunk[s] >= 0 && !tma) load_thread(sh, s, tid, data, n, chunk[s]);
  }
  (void)warp;
  // [0] rounds, [1] waits for look-back results, [2] final passes, [3] other
  // [4] refill issue, [5] round-0 data wait, [6] mma + automaton part of the final pass
  Laps<kProf, 7> lap;
  lap.start();
  for (bool any = true; any;) {
    any = false;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      if (chunk[s] < 0) continue;
      any = true;
      if (pend[s]) {
        lap.mark(3);
        fnv::mbar_wait(&sh.res[s], (rpar >> s) & 1u);
        rpar ^= 1u << s;
        // lane start -> segment starts through the segment maps
#if MLCK_FNV_PACKED_MAPS
        const uint32_t add = starts_lanes(keep[s], map_apply(keep[s] & 7u, sh.wstart[s][warp]));
#else
        uint32_t ss = map_apply(keep[s] & 7u, sh.wstart[s][warp]);
        uint32_t add = ss;
#pragma unroll
        for (int i = 1; i < kSegs; ++i) {
          ss = map_apply((keep[s] >> (3 * i)) & 7u, ss);
          add |= ss << (8 * i);
        }
#endif
        st[s] |= add << (2 * rnd[s]);
        lap.mark(1);
        pend[s] = false;
        if (++rnd[s] == kRounds) {
#if MLCK_FNV_MMA
          // ---- final pass: sum_p P^(E_w - p) (b_p - 2 (u_p & b_p)) on the
          // tensor cores (bytes past n are zero and contribute nothing)
          {
            int mac[2][4] = {};
            mma_pass(sh, s, warp, lane, 0, mac);  // the data vector
            uint32_t w[kThreadWords];
            read_thread(sh, s, tid, w);
            automaton_and(w, st[s]);
            __syncwarp();  // every lane has read the data words
            write_thread(sh, s, tid, w);
            __syncwarp();
            mma_pass(sh, s, warp, lane, 1, mac);  // the u & b vector, weights -2 P^(...)
            acc += mma_epilogue(sh, lane, mac) * (pinv_t * chunk_weight(chunk[s]));
          }
          {  // the row's segment starts, for later verification (fnv_witness_kernel);
             // the pointer comes from shared memory, not a live register
            uint32_t* const wp = *reinterpret_cast<uint32_t* volatile*>(&sh.witness);
            const uint64_t row = static_cast<uint64_t>(chunk[s]) * kComputeThreads + tid;
            if (wp && row * kThreadBytes < n) wp[row] = st[s];
          }
          lap.mark(6);
#else
          // ---- final pass: the real recurrence from each segment's start
          uint32_t w[kThreadWords];
          read_thread(sh, s, tid, w);
          const uint64_t p0 = static_cast<uint64_t>(chunk[s]) * kChunk + static_cast<uint64_t>(tid) * kThreadBytes;
          if (p0 + kThreadBytes <= n) {
            uint32_t lo[kSegs], hi[kSegs];
#pragma unroll
            for (int i = 0; i < kSegs; ++i) {
              lo[i] = (st[s] >> (8 * i)) & 0xffu;
              hi[i] = 0;
            }
#pragma unroll
            for (int k = 0; k < 32; ++k)  // interleaved: byte i of word k = segment i, byte k
#pragma unroll
              for (int i = 0; i < kSegs; ++i) fnv_byte(lo[i], hi[i], (w[k] >> (8 * i)) & 0xffu);
            uint64_t g = 0;  // sum_i G_i P^(32 (kSegs-1-i))
#pragma unroll
            for (int i = 0; i < kSegs; ++i)
              g = g * kPow32 + ((static_cast<uint64_t>(hi[i]) << 32) | (lo[i] & ~0xffu));
            acc += g * (pinv_t * chunk_weight(chunk[s]));
            if (p0 + kThreadBytes == n) {
              *scr.ulast = lo[kSegs - 1] & 0xffu;
              __threadfence();
            }
          } else if (p0 < n) {  // holds the last byte: one chain to n
            // (bytes from shared memory: a run-time index into w[] would put
            // w in local memory on the hot path too)
            uint32_t lo = st[s] & 0xffu, hi = 0;
            for (int k = 0; k < kThreadBytes && p0 + k < n; ++k) {  // stream byte k: segment k/32
              const uint32_t* g = reinterpret_cast<const uint32_t*>(&sh.data[s][granule(tid, (k & 31) >> 2)]);
              fnv_byte(lo, hi, (g[k & 3] >> (8 * (k >> 5))) & 0xffu);
            }
            const uint64_t g = (static_cast<uint64_t>(hi) << 32) | (lo & ~0xffu);
            acc += g * pow_u64(kPrimeInv, n);
            *scr.ulast = lo & 0xffu;
            __threadfence();
          }
#endif
          if (kProf && scr.trace && tid == 0) scr.trace[chunk[s] * 12 + 9] = gtimer();
          lap.mark(2);
          // ---- refill (thread-private granules: no CTA barrier needed); the
          // bytes land while the other slots take their turns
          chunk[s] = sh.next[s];  // the ticket the look-back warp took in round 3
          rnd[s] = 0;
          st[s] = 0;
          par ^= 1u << s;
          if (tma) {
            bar_arrive(bar_pub(s), kBarThreads);  // done with the bytes: the look-back warp refills
          } else if (chunk[s] >= 0) {
            load_thread(sh, s, tid, data, n, chunk[s]);
          }
          lap.mark(4);
          continue;
        }
      }
      // ---- compute and publish round rnd[s]
      if (rnd[s] == 0) {
        lap.mark(0);
        fnv::mbar_wait(&sh.mbar[s][tma ? 0 : warp], (par >> s) & 1u);
        if (tma && !kGather) {
          const uint64_t row = static_cast<uint64_t>(chunk[s]) * kComputeThreads + tid;
          if (row >= rows_full) {  // the partial last row, or zeros past the record
            const uint64_t p = row * kThreadBytes;
            load_thread_bytes(sh, s, tid, [&](int i) -> uint32_t { return p + i < n ? data[p + i] : 0u; }, false);
          }
        }
        lap.mark(5);
        if (kProf && scr.trace && tid == 0) {
          scr.trace[chunk[s] * 12 + 0] = gtimer();
          scr.trace[chunk[s] * 12 + 10] = smid();
        }
      }
      uint32_t w[kThreadWords];
#ifdef MLCK_FUSED_NOSHIFT  // development A/B only (wrong bytes): the cost of the shifted read
      const uint32_t delta = 0u;
#else
      const uint32_t delta = kGather && rnd[s] == 0 ? sh.shift[s] : 0u;  // uniform over the chunk
#endif
      if (delta)
        read_thread_shifted(sh, s, tid, delta, w);
      else
        read_thread(sh, s, tid, w);
      const bool store = copy && rnd[s] == 0;
      if (rnd[s] == 0) {
        if (delta) {
          // every window is read before its rows are rewritten aligned: the
          // warp's lanes (syncwarp) and the previous warp's last lane, whose
          // window overhangs into this warp's first row (a handshake with
          // the neighbour, not a barrier over all compute warps)
          __syncwarp();
          if (lane == 0 && warp + 1 < kComputeWarps) mbar_arrive(&sh.rd[s][warp + 1]);
          if (warp > 0) fnv::mbar_wait(&sh.rd[s][warp], (rdpar >> s) & 1u);
          rdpar ^= 1u << s;
          write_thread(sh, s, tid, w);
        }
        if (store) {  // record-aligned rows in place: out to every destination
          fence_async_shared();
          bar_arrive(bar_store(s), kBarThreads);
          const uint64_t row = static_cast<uint64_t>(chunk[s]) * kComputeThreads + tid;
          if (row == rows_full && (n & (kThreadBytes - 1))) {  // the partial last row (TMA stores clip it)
            const uint8_t* rb = reinterpret_cast<const uint8_t*>(sh.data[s]);
            for (uint32_t k = 0; k < (n & (kThreadBytes - 1)); ++k) {
              const uint8_t b = rb[16 * granule(tid, k >> 4) + (k & 15)];
              for (int d = 0; d < cp.n_dst; ++d) cp.dst_ptr[d][rows_full * kThreadBytes + k] = b;
            }
          }
        }
        interleave(w);  // fresh bytes: interleave the segments once, in place
        if (!store) write_thread(sh, s, tid, w);
      } else if (copy && rnd[s] == 1) {
        // copies: the rows stayed record-aligned for the TMA stores through
        // round 0; interleaved in place now, once the stores have read them
        interleave(w);
        fnv::mbar_wait(&sh.sres[s], (spar >> s) & 1u);
        spar ^= 1u << s;
        write_thread(sh, s, tid, w);
      }
#if MLCK_FNV_PACKED_MAPS
      uint32_t e0, e1, kp;
      if (MLCK_FNV_ROUND0_LINEAR && rnd[s] == 0)
        round0_lanes(w, &e0, &e1);
      else if (rnd[s] < 2)
        round_lanes_low(w, st[s], rnd[s], &e0, &e1);
      else
        round_lanes_high(w, st[s], rnd[s], &e0, &e1);
      const uint32_t tm = compose_lanes(e0, e1, &kp);
#else
      uint32_t m[kSegs];
      if (MLCK_FNV_ROUND0_LINEAR && rnd[s] == 0)
        round0_maps(w, m);
      else if (rnd[s] < 2)
        round_maps_low(w, st[s], rnd[s], m);
      else
        round_maps_high(w, st[s], rnd[s], m);
      uint32_t tm = m[0], kp = 0;
#pragma unroll
      for (int i = 1; i < kSegs; ++i) {
        kp |= m[i - 1] << (3 * i);
        tm = map_compose(m[i], tm);
      }
#endif
      uint32_t wtot;
      keep[s] = map_scan_warp(tm, &wtot) | kp;
      if (lane == 0) sh.wmap[s][warp] = wtot;
      bar_arrive(bar_pub(s), kBarThreads);
      pend[s] = true;
      lap.mark(0);
    }
  }
  if (copy && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  if (kProf && tid == 0) {
    lap.mark(3);
    atomicAdd(scr.prof + 2, static_cast<unsigned long long>(lap.t[0]));
    atomicAdd(scr.prof + 3, static_cast<unsigned long long>(lap.t[1]));
    atomicAdd(scr.prof + 4, static_cast<unsigned long long>(lap.t[2]));
    atomicAdd(scr.prof + 6, static_cast<unsigned long long>(lap.t[3]));
    atomicAdd(scr.prof + 16, static_cast<unsigned long long>(lap.t[4]));
    atomicAdd(scr.prof + 17, static_cast<unsigned long long>(lap.t[5]));
    atomicAdd(scr.prof + 20, static_cast<unsigned long long>(lap.t[6]));
  }
  return acc;
}

#if MLCK_FNV_COMPUTE_ONE_COPY
// fnv_compute with one copy of the turn code for every slot (the slot a
// run-time value): the per-slot state lives in shared memory (chunk ids per
// warp, start bits and pending maps per thread) and in packed registers
// (round and pending flags), so the compute warps' hot code is a third of
// the unrolled form's and fits the instruction caches.
template <bool kProf, bool kGather>
__device__ __forceinline__ uint64_t fnv_compute1(fnv::Shared& sh, const uint8_t* data, uint64_t n,
                                                 const fnv::Scratch& scr, int64_t n_chunks,
                                                 const int64_t (&first)[kSlots], int64_t stride,
                                                 const fnv::Copy& cp, bool tma) {
  using namespace fnv;
  static_assert(MLCK_FNV_MMA, "the one-copy compute loop has the tensor-core final pass only");
  const uint64_t rows_full = n / kThreadBytes;
  const int tid = static_cast<int>(threadIdx.x) - kComputeTidBase, warp = tid >> 5, lane = tid & 31;
#if MLCK_FNV_MMA
  const uint64_t pinv_t = pow_u64(kPrimeInv, static_cast<uint64_t>(kThreadBytes) * 32 * (warp + 1));
#else
  const uint64_t pinv_t = pow_u64(kPrimeInv, static_cast<uint64_t>(kThreadBytes) * (tid + 1));
#endif
  uint32_t rndp = 0;   // round of slot s: bits 4s .. 4s+3
  uint32_t pendp = 0;  // bit s: a published round of slot s awaits its result
  uint32_t par = 0, rpar = 0, spar = 0, rdpar = 0;  // mbarrier phase parities per slot (as fnv_compute)
  const bool copy = cp.n_dst > 0;
  uint64_t acc = 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    sh.cw[s][warp] = first[s];
    sh.cst[s][tid] = 0;
    sh.ckeep[s][tid] = 0;
    if (first[s] >= 0 && !tma) load_thread(sh, s, tid, data, n, first[s]);
  }
  (void)stride;
  (void)n_chunks;
  Laps<kProf, 7> lap;
  lap.start();
  for (bool any = true; any;) {
    any = false;
#pragma unroll 1
    for (int s = 0; s < kSlots; ++s) {
      int64_t c = sh.cw[s][warp];
      if (c < 0) continue;
      any = true;
      uint32_t r = (rndp >> (4 * s)) & 15u;
      uint32_t stv = sh.cst[s][tid];
      if ((pendp >> s) & 1u) {
        lap.mark(3);
        fnv::mbar_wait(&sh.res[s], (rpar >> s) & 1u);
        rpar ^= 1u << s;
        const uint32_t kp = sh.ckeep[s][tid];
#if MLCK_FNV_PACKED_MAPS
        const uint32_t add = starts_lanes(kp, map_apply(kp & 7u, sh.wstart[s][warp]));
#else
        uint32_t ss = map_apply(kp & 7u, sh.wstart[s][warp]);
        uint32_t add = ss;
#pragma unroll
        for (int i = 1; i < kSegs; ++i) {
          ss = map_apply((kp >> (3 * i)) & 7u, ss);
          add |= ss << (8 * i);
        }
#endif
        stv |= add << (2 * r);
        lap.mark(1);
        pendp &= ~(1u << s);
        if (++r == kRounds) {
          {
            int mac[2][4] = {};
            mma_pass(sh, s, warp, lane, 0, mac);  // the data vector
            uint32_t w[kThreadWords];
            read_thread(sh, s, tid, w);
            automaton_and(w, stv);
            __syncwarp();
            write_thread(sh, s, tid, w);
            __syncwarp();
            mma_pass(sh, s, warp, lane, 1, mac);  // the u & b vector, weights -2 P^(...)
            acc += mma_epilogue(sh, lane, mac) * (pinv_t * chunk_weight(c));
          }
          {
            uint32_t* const wp = *reinterpret_cast<uint32_t* volatile*>(&sh.witness);
            const uint64_t row = static_cast<uint64_t>(c) * kComputeThreads + tid;
            if (wp && row * kThreadBytes < n) wp[row] = stv;
          }
          lap.mark(6);
          if (kProf && scr.trace && tid == 0) scr.trace[c * 12 + 9] = gtimer();
          lap.mark(2);
          c = sh.next[s];  // the ticket the look-back warp took in round 3
          sh.cw[s][warp] = c;
          rndp &= ~(15u << (4 * s));
          sh.cst[s][tid] = 0;
          par ^= 1u << s;
          if (tma) {
            bar_arrive(bar_pub(s), kBarThreads);
          } else if (c >= 0) {
            load_thread(sh, s, tid, data, n, c);
          }
          lap.mark(4);
          continue;
        }
      }
      // ---- compute and publish round r
      if (r == 0) {
        lap.mark(0);
        fnv::mbar_wait(&sh.mbar[s][tma ? 0 : warp], (par >> s) & 1u);
        if (tma && !kGather) {
          const uint64_t row = static_cast<uint64_t>(c) * kComputeThreads + tid;
          if (row >= rows_full) {
            const uint64_t p = row * kThreadBytes;
            load_thread_bytes(sh, s, tid, [&](int i) -> uint32_t { return p + i < n ? data[p + i] : 0u; }, false);
          }
        }
        lap.mark(5);
        if (kProf && scr.trace && tid == 0) {
          scr.trace[c * 12 + 0] = gtimer();
          scr.trace[c * 12 + 10] = smid();
        }
      }
      uint32_t w[kThreadWords];
      const uint32_t delta = kGather && r == 0 ? sh.shift[s] : 0u;
      if (delta)
        read_thread_shifted(sh, s, tid, delta, w);
      else
        read_thread(sh, s, tid, w);
      const bool store = copy && r == 0;
      if (r == 0) {
        if (delta) {
          __syncwarp();
          if (lane == 0 && warp + 1 < kComputeWarps) mbar_arrive(&sh.rd[s][warp + 1]);
          if (warp > 0) fnv::mbar_wait(&sh.rd[s][warp], (rdpar >> s) & 1u);
          rdpar ^= 1u << s;
          write_thread(sh, s, tid, w);
        }
        if (store) {
          fence_async_shared();
          bar_arrive(bar_store(s), kBarThreads);
          const uint64_t row = static_cast<uint64_t>(c) * kComputeThreads + tid;
          if (row == rows_full && (n & (kThreadBytes - 1))) {
            const uint8_t* rb = reinterpret_cast<const uint8_t*>(sh.data[s]);
            for (uint32_t k = 0; k < (n & (kThreadBytes - 1)); ++k) {
              const uint8_t b = rb[16 * granule(tid, k >> 4) + (k & 15)];
              for (int d = 0; d < cp.n_dst; ++d) cp.dst_ptr[d][rows_full * kThreadBytes + k] = b;
            }
          }
        }
        interleave(w);
        if (!store) write_thread(sh, s, tid, w);
      } else if (copy && r == 1) {
        interleave(w);
        fnv::mbar_wait(&sh.sres[s], (spar >> s) & 1u);
        spar ^= 1u << s;
        write_thread(sh, s, tid, w);
      }
#if MLCK_FNV_PACKED_MAPS
      uint32_t e0, e1, kp;
      if (MLCK_FNV_ROUND0_LINEAR && r == 0)
        round0_lanes(w, &e0, &e1);
      else if (r < 2)
        round_lanes_low(w, stv, r, &e0, &e1);
      else
        round_lanes_high(w, stv, r, &e0, &e1);
      const uint32_t tm = compose_lanes(e0, e1, &kp);
#else
      uint32_t m[kSegs];
      if (MLCK_FNV_ROUND0_LINEAR && r == 0)
        round0_maps(w, m);
      else if (r < 2)
        round_maps_low(w, stv, r, m);
      else
        round_maps_high(w, stv, r, m);
      uint32_t tm = m[0], kp = 0;
#pragma unroll
      for (int i = 1; i < kSegs; ++i) {
        kp |= m[i - 1] << (3 * i);
        tm = map_compose(m[i], tm);
      }
#endif
      uint32_t wtot;
      sh.ckeep[s][tid] = map_scan_warp(tm, &wtot) | kp;
      if (lane == 0) sh.wmap[s][warp] = wtot;
      bar_arrive(bar_pub(s), kBarThreads);
      pendp |= 1u << s;
      rndp = (rndp & ~(15u << (4 * s))) | (r << (4 * s));
      sh.cst[s][tid] = stv;
      lap.mark(0);
    }
  }
  if (copy && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (kProf && tid == 0) {
    lap.mark(3);
    atomicAdd(scr.prof + 2, static_cast<unsigned long long>(lap.t[0]));
    atomicAdd(scr.prof + 3, static_cast<unsigned long long>(lap.t[1]));
    atomicAdd(scr.prof + 4, static_cast<unsigned long long>(lap.t[2]));
    atomicAdd(scr.prof + 6, static_cast<unsigned long long>(lap.t[3]));
    atomicAdd(scr.prof + 16, static_cast<unsigned long long>(lap.t[4]));
    atomicAdd(scr.prof + 17, static_cast<unsigned long long>(lap.t[5]));
    atomicAdd(scr.prof + 20, static_cast<unsigned long long>(lap.t[6]));
  }
  return acc;
}
#endif

// Look-back warp of slot s: for every round the compute warps publish on
// the slot it folds their warp maps into the chunk's map, publishes it,
// looks back for the chunk's start bits and hands each warp its start.  Only
// this slot's turns involve it, so the slots' look-backs run concurrently.
template <bool kProf, bool kGather>
__device__ __forceinline__ void fnv_lookback(fnv::Shared& sh, int s, uint64_t seed, const fnv::Scratch& scr,
                                             int64_t chunk, int64_t n_chunks, int64_t stride,
                                             const CUtensorMap* tmap, uint64_t n, const fnv::Copy& cp) {
  using namespace fnv;
  const int lane = threadIdx.x & 31;
  const unsigned long long tag = static_cast<unsigned long long>(scr.epoch) << 32;
  // [1] idle at PUB, [2] probe loads, [3] spins, [4] compose, [5] publish + hand-off
  long long lb[6] = {0, 0, 0, 0, 0, 0};
  long long* lp = kProf ? lb : nullptr;
  const long long t_begin = kProf ? clock64() : 0;
  lb[0] = t_begin;
  auto mark = [&](int b) {
    if (kProf) {
      const long long now = clock64();
      lb[b] += now - lb[0];
      lb[0] = now;
    }
  };
  const uint64_t rows_full = n / kThreadBytes;
  const bool copy = cp.n_dst > 0;
  if (kGather && chunk >= 0) {
    const Run run = find_run(cp, chunk);
    if (lane == 0) tma_load_src(sh, s, cp, run, chunk);
  } else if (tmap && lane == 0 && chunk >= 0) {
    tma_load_chunk(sh, s, tmap, chunk, rows_full);
  }
  while (chunk >= 0) {
    uint32_t word = 0;  // the chunk's status bits as published
    int64_t next = -1;
    Run nrun{};  // kGather: the run of the next chunk, looked up beside the last round
    if (copy) {  // the compute warps have the rows aligned: out to every destination
      bar_sync(bar_store(s), kBarThreads);
      if (lane == 0) tma_store_chunk(sh, s, cp, chunk, rows_full);
      __syncwarp();
    }
    for (int r = 0; r < kRounds; ++r) {
      if (copy && r == 1 && lane == 0) {  // round 1 rewrites the rows: once the stores have read them
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(&sh.sres[s]);
      }
      mark(5);
      bar_sync(bar_pub(s), kBarThreads);
      if (r == kRounds - 1) {
        // the slot's next chunk: a ticket taken now, in the order the slots
        // reach their last round, so a CTA's chunks rise in its turn order and
        // every chunk's predecessors are already held by running CTAs (no
        // co-residency needed); handed to the compute warps with this round's
        // result
        if (lane == 0) {
          const unsigned long long t = atomicAdd(scr.ticket, 1ull);
          sh.next[s] = t < static_cast<unsigned long long>(n_chunks) ? static_cast<int64_t>(t) : -1;
        }
        __syncwarp();
        next = sh.next[s];
        if (kGather && next >= 0) nrun = find_run(cp, next);
      }
      const uint32_t wm = lane < kComputeWarps ? sh.wmap[s][lane] : 0u;
      mark(1);
      uint32_t ctot;
      const uint32_t wex = map_scan_warp(wm, &ctot);
      if (lane == 0) {
        word = (word & ~(7u << 20)) | (ctot << (3 * r)) | (static_cast<uint32_t>(r + 1) << 20);
        st_relaxed_gpu_u64(scr.status + chunk * kStatusStride, tag | word);
        if (kProf && scr.trace) scr.trace[chunk * 12 + 1 + 2 * r] = gtimer();
      }
      mark(5);
      const uint32_t start = look_back2_warp(scr, chunk, r, static_cast<uint32_t>(seed >> (2 * r)) & 3u, lp);
      if (lane == 0) {
        word = (word & ~(7u << 24)) | (map_apply(ctot, start) << (12 + 2 * r)) |
               (static_cast<uint32_t>(r + 1) << 24);
        st_relaxed_gpu_u64(scr.status + chunk * kStatusStride, tag | word);
        if (kProf && scr.trace) scr.trace[chunk * 12 + 2 + 2 * r] = gtimer();
      }
      if (lane < kComputeWarps) sh.wstart[s][lane] = map_apply(wex, start);
      if (kProf && r == kRounds - 1 && lane == 0) atomicAdd(scr.prof + 5, 1ull);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.res[s]);  // release: wstart is visible to the waiters
    }
    if (kGather || tmap) {  // the compute warps are done with the bytes: load the slot's next chunk
      bar_sync(bar_pub(s), kBarThreads);
      if (lane == 0 && next >= 0) {
        if (kGather)
          tma_load_src(sh, s, cp, nrun, next);
        else
          tma_load_chunk(sh, s, tmap, next, rows_full);
      }
    }
    chunk = next;
  }
  if (copy && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  mark(5);
  if (kProf && lane == 0) {
    for (int b = 1; b <= 5; ++b) atomicAdd(scr.prof + 7 + b, static_cast<unsigned long long>(lb[b]));
    atomicAdd(scr.prof + 13, static_cast<unsigned long long>(clock64() - t_begin));
  }
}

// Persistent CTAs (one per SM, kSlots chunks in flight each).  The CTA that
// finishes last combines the terms and writes the trailer (serialize_record
// appends the checksum, snapshot.hpp:142).
#ifdef MLCK_FNV_MAXREG
#define MLCK_FNV_BOUNDS __maxnreg__(MLCK_FNV_MAXREG)
#else
#define MLCK_FNV_BOUNDS __launch_bounds__(fnv::kThreads, 1)
#endif
template <bool kProf, bool kGather>
__global__ void MLCK_FNV_BOUNDS
    fnv_kernel(const uint8_t* data, uint64_t n, uint64_t seed, fnv::Scratch scr, int64_t n_chunks,
               TrailerDsts trailer, const __grid_constant__ fnv::Copy cp, const __grid_constant__ CUtensorMap tmap,
               int use_tma) {
  using namespace fnv;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KiB-aligned rows whatever the base of the dynamic window
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0)
    for (int s = 0; s < kSlots; ++s) {
      for (int w = 0; w < kComputeWarps; ++w) mbar_init(&sh.mbar[s][w], kGather || use_tma ? 1 : 32);
      mbar_init(&sh.res[s], 1);
      mbar_init(&sh.sres[s], 1);
      for (int w = 0; w < kComputeWarps; ++w) mbar_init(&sh.rd[s][w], 1);
    }
#if MLCK_FNV_MMA
  mma_tables(sh, tid);
#endif
  __syncthreads();
  // Chunks are handed out by a ticket counter: a CTA takes its first kSlots
  // chunks at once when it starts, then one per slot as the slot reaches its
  // last round (fnv_lookback).  Tickets rise in the CTA's turn order and only
  // running CTAs hold them, so every chunk's look-back waits on chunks that
  // are already being hashed: any grid size, any co-scheduled work.
  if (tid == 0) {
    sh.witness = scr.witness;
    const unsigned long long t0 = atomicAdd(scr.ticket, static_cast<unsigned long long>(kSlots));
#pragma unroll
    for (int s = 0; s < kSlots; ++s)
      sh.next[s] = t0 + s < static_cast<unsigned long long>(n_chunks) ? static_cast<int64_t>(t0 + s) : -1;
  }
  __syncthreads();
  const int64_t stride = 0;
  int64_t first[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) first[s] = sh.next[s];
  __syncthreads();  // sh.next is rewritten by the look-back warps from here on
  uint64_t acc = 0;
  const bool tma = kGather || use_tma;  // chunks land by TMA (from the sources under kGather)
  if (compute_warp(warp) >= 0) {
#if MLCK_FNV_COMPUTE_ONE_COPY
    acc = fnv_compute1<kProf, kGather>(sh, data, n, scr, n_chunks, first, stride, cp, tma);
#else
    acc = fnv_compute<kProf, kGather>(sh, data, n, scr, n_chunks, first, stride, cp, tma);
#endif
  } else {
#if MLCK_FNV_LB_ONE_COPY
    // one copy of the look-back code for every slot's warp (the slot is a
    // run-time value): the kernel's hot code fits the instruction caches
    const int s = MLCK_FNV_LB_FIRST ? warp : warp - kComputeWarps;
    int64_t f = first[0];
#pragma unroll
    for (int q = 1; q < kSlots; ++q)
      if (s == q) f = first[q];
    fnv_lookback<kProf, kGather>(sh, s, seed, scr, f, n_chunks, stride, !kGather && use_tma ? &tmap : nullptr, n,
                                 cp);
#else
#pragma unroll
    for (int s = 0; s < kSlots; ++s)
      if (warp == lookback_warp(s))
        fnv_lookback<kProf, kGather>(sh, s, seed, scr, first[s], n_chunks, stride,
                                     !kGather && use_tma ? &tmap : nullptr, n, cp);
#endif
  }
  // CTA sum -> global accumulator; the last CTA finishes the hash
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) sh.red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    uint64_t sum = 0;
    for (int q = 0; q < kWarps; ++q) sum += sh.red[q];
    atomicAdd(scr.accum, static_cast<unsigned long long>(sum));
    __threadfence();
    const uint32_t done = atomicAdd(scr.finished, 1u) + 1;
    if (done == gridDim.x) {
      __threadfence();
      const uint64_t total = atomicAdd(scr.accum, 0ull);
      const uint32_t u = atomicAdd(scr.ulast, 0u);
#if MLCK_FNV_MMA
      (void)u;
      const uint64_t h = pow_p(n) * (total + seed);
#else
      const uint64_t h = pow_p(n) * (total + (seed & ~0xffull)) + u;
#endif
      const uint32_t err = atomicAdd(scr.error, 0u);
      if (err) atomicOr(scr.sticky, 1u);  // reported by the host at its next synchronization
      *scr.result = err ? 0ull : h;
      // a hash the watchdog cut short is not the record's: poison the trailer
      // so every copy fails parse_record's checksum instead of carrying it
      const uint64_t tr = err ? ~h : h;
      for (int r = 0; r < trailer.n; ++r)
        for (int b = 0; b < 8; ++b) trailer.p[r][b] = static_cast<uint8_t>(tr >> (8 * b));
    }
  }
}

// The thread's own row from global bytes, zeros past n (the record's last,
// partial row and rows past the end -- the tensor map covers full rows only).
__device__ __forceinline__ void witness_row_bytes(uint4* rows, int tid, const uint8_t* data, uint64_t n, uint64_t p) {
  using namespace fnv;
  for (int q = 0; q < kGranules; ++q) {
    uint32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x = 0;
      for (int b = 0; b < 4; ++b) {
        const uint64_t o = p + 16 * q + 4 * i + b;
        x |= (o < n ? static_cast<uint32_t>(data[o]) : 0u) << (8 * b);
      }
      v[i] = x;
    }
    rows[granule(tid, q)] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

constexpr int kWitnessBufs = 3;  // chunks in flight per SM
// the chunk's witness words and the next chunk's first (a 16-byte multiple)
constexpr int kWitnessWords = fnv::kComputeThreads + 4;
struct WitnessSmem {
  uint4 data[kWitnessBufs][fnv::kComputeThreads * fnv::kGranules];  // 1 KiB-aligned rows (TMA swizzle)
  uint32_t wit[kWitnessBufs][kWitnessWords];                         // the rows' witnessed starts
  uint2 wfrag[2][4][32];
  unsigned long long kpos[32][4];
  unsigned long long red[fnv::kComputeWarps];
  unsigned long long full[kWitnessBufs];   // the chunk's rows and witness words landed
  unsigned long long empty[kWitnessBufs];  // every compute warp is done with the buffer
};
constexpr size_t kWitnessSmem = sizeof(WitnessSmem) + 1024;
constexpr int kWitnessThreads = fnv::kComputeThreads + 32;  // + the producer warp

// Re-hash of a record against its witness (fnv.cuh, automaton_and_ends).
// Persistent and warp-specialized: one CTA per SM walks chunks blockIdx.x,
// +gridDim.x, ...; its producer warp keeps kWitnessBufs chunks in flight --
// the rows by tensor-map loads, the witness words by a bulk copy, one
// mbarrier per buffer -- and refills a buffer once all compute warps have
// released it, so compute warps never wait on each other or on a global
// load.  *bad <- 1 when a witnessed start disagrees with the automaton (the
// caller then runs fnv_kernel).  The witness array holds >= kWitnessWords
// words past the record's last chunk start (mlck_blob::reserve_witness).
__device__ uint2 g_wfrag[2][4][32];             // mma_pass B fragments (init_constants)
__device__ unsigned long long g_kpos[32][4];    // mma_epilogue weights
__constant__ unsigned long long c_pinv_warp[fnv::kComputeWarps];  // P^-(4096 (w + 1))

__global__ void __launch_bounds__(kWitnessThreads, 1)
    fnv_witness_kernel(const uint8_t* data, uint64_t n, uint64_t seed, const uint32_t* witness, fnv::Scratch scr,
                       unsigned long long* bad, int64_t n_chunks, const __grid_constant__ CUtensorMap tmap,
                       uint64_t rows_full) {
  using namespace fnv;
  extern __shared__ __align__(1024) unsigned char smem_w[];
  WitnessSmem& sh = *reinterpret_cast<WitnessSmem*>(smem_w + ((1024u - (smem_addr(smem_w) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n_seg = (n + 31) / 32;
  const int64_t G = gridDim.x;
  if (tid < 2 * 4 * 32) (&sh.wfrag[0][0][0])[tid] = (&g_wfrag[0][0][0])[tid];
  if (tid < 32 * 4) (&sh.kpos[0][0])[tid] = (&g_kpos[0][0])[tid];
  if (tid == 0)
    for (int b = 0; b < kWitnessBufs; ++b) {
      mbar_init(&sh.full[b], 1);
      mbar_init(&sh.empty[b], kComputeWarps);
    }
  __syncthreads();  // tables, barriers
  uint64_t acc = 0;
  bool ok = true;
  if (warp == kComputeWarps) {  // ---- producer
    if (lane == 0)
      for (int64_t i = 0, chunk = blockIdx.x; chunk < n_chunks; ++i, chunk += G) {
        const int b = static_cast<int>(i % kWitnessBufs);
        if (i >= kWitnessBufs) mbar_wait(&sh.empty[b], static_cast<uint32_t>(i / kWitnessBufs - 1) & 1u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint64_t row0 = static_cast<uint64_t>(chunk) * kComputeThreads;
        int boxes = 0;
#pragma unroll
        for (int x = 0; x < kComputeThreads / kTmaBoxRows; ++x) boxes += row0 + kTmaBoxRows * x < rows_full;
        mbar_arrive_expect_tx(&sh.full[b], boxes * kTmaBoxRows * kThreadBytes + 4 * kWitnessWords);
        for (int x = 0; x < boxes; ++x)
          tma_load_rows(&sh.data[b][kGranules * kTmaBoxRows * x], &tmap, static_cast<int32_t>(row0 + kTmaBoxRows * x),
                        &sh.full[b]);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(&sh.wit[b][0])),
            "l"(witness + row0), "r"(4 * kWitnessWords), "r"(smem_addr(&sh.full[b]))
            : "memory");
      }
  } else {  // ---- compute warps
    const uint64_t pinv_w = c_pinv_warp[warp];
    for (int64_t i = 0, chunk = blockIdx.x; chunk < n_chunks; ++i, chunk += G) {
      const int b = static_cast<int>(i % kWitnessBufs);
      uint4* rows = sh.data[b];
      mbar_wait(&sh.full[b], static_cast<uint32_t>(i / kWitnessBufs) & 1u);
      const uint64_t row = static_cast<uint64_t>(chunk) * kComputeThreads + tid;
      uint32_t st = 0, expect = 0, check = 0;
      if (row * kThreadBytes < n) {
        st = sh.wit[b][tid];
        const uint64_t seg0 = 4 * row;
        const uint32_t next = seg0 + 4 < n_seg ? (sh.wit[b][tid + 1] & 0xffu) : 0u;
        expect = (st >> 8) | (next << 24);  // segment i ends where segment i+1 starts
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (seg0 + q + 1 < n_seg) check |= 0xffu << (8 * q);
        if (row == 0 && (st & 0xffu) != (seed & 0xffu)) ok = false;
      }
      if (row >= rows_full) witness_row_bytes(rows, tid, data, n, row * kThreadBytes);
      uint32_t w[kThreadWords];
      read_thread_rows(rows, tid, w);
      interleave(w);
      write_thread_rows(rows, tid, w);
      __syncwarp();
      int mac[2][4] = {};
      mma_pass_rows(rows, sh.wfrag, warp, lane, 0, mac);  // the data vector
      const uint32_t ends = automaton_and_ends(w, st);
      if ((ends ^ expect) & check) ok = false;
      __syncwarp();  // every lane has read the data words
      write_thread_rows(rows, tid, w);
      __syncwarp();
      mma_pass_rows(rows, sh.wfrag, warp, lane, 1, mac);  // the u & b vector, weights -2 P^(...)
      acc += mma_epilogue(sh, lane, mac) * (pinv_w * chunk_weight(chunk));
      __syncwarp();  // the warp's reads of the buffer are done
      if (lane == 0) mbar_arrive(&sh.empty[b]);
    }
  }
  if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicExch(bad, 1ull);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && warp < kComputeWarps) sh.red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    uint64_t sum = 0;
    for (int q = 0; q < kComputeWarps; ++q) sum += sh.red[q];
    atomicAdd(scr.accum, static_cast<unsigned long long>(sum));
    __threadfence();
    if (atomicAdd(scr.finished, 1u) + 1 == gridDim.x) {
      __threadfence();
      const uint64_t total = atomicAdd(scr.accum, 0ull);
      *scr.result = pow_p(n) * (total + seed);
    }
  }
}


// ---- the verifier on the 5th-generation tensor cores (tcgen05 + TMEM).
// Per chunk, two 128 x 16 x 512 u8 MMAs do every dot product of the chunk:
// A = the chunk's 512 rows as they sit in shared memory (M = the 128 byte
// positions of a row, K = the row: the TMA's 128-byte-swizzled rows ARE the
// canonical MN-major SWIZZLE_128B operand layout), B = the 8-bit limbs of
// P^-(128 k) (and of -2 P^-(128 k)) for row k.  MMA 1 reads the bytes as
// landed (natural order), MMA 2 the rows the compute warps overwrite with
// u & b (interleaved order: byte 4j + s of a row = segment s, byte j).  The
// accumulators (s32, < 2^26) go to TMEM; four warps fold a chunk's 128 x 8
// limb sums with P^-(byte position) two chunks later.  Compute threads keep
// only the automaton: no fragment loads, no mma.sync, one row write.
#ifndef MLCK_WITNESS_TC
#define MLCK_WITNESS_TC 1
#endif
constexpr int kTcThreads = fnv::kComputeThreads + 96;  // + the producer warp + one warp per MMA
constexpr uint32_t kTcCols = 128;                     // TMEM columns: [buffer][2 accumulators][16]
struct WitnessTcSmem {
  uint4 data[kWitnessBufs][fnv::kComputeThreads * fnv::kGranules];  // 1 KiB-aligned rows (TMA swizzle)
  uint8_t wb[2][fnv::kComputeThreads][kTcN];                         // B: [data | -2][row k][limb n], 16 KiB
  uint32_t wit[kWitnessBufs][kWitnessWords];
  unsigned long long full[kWitnessBufs], empty[kWitnessBufs];        // producer <-> MMA / compute warps
  unsigned long long mma1[kWitnessBufs], mma2[kWitnessBufs];         // MMA 1 / 2 complete
  unsigned long long uab[kWitnessBufs], tfree[kWitnessBufs];         // u & b rows written / accumulators read
  unsigned long long tail;                                           // the last chunk's partial rows written
  unsigned long long red[32];
  uint32_t tmem;
  uint32_t abort;
};
constexpr size_t kWitnessTcSmem = sizeof(WitnessTcSmem) + 1024;
__global__ void __launch_bounds__(kTcThreads, 1)
    fnv_witness_tc_kernel(const uint8_t* data, uint64_t n, uint64_t seed, const uint32_t* witness, fnv::Scratch scr,
                          unsigned long long* bad, int64_t n_chunks, const __grid_constant__ CUtensorMap tmap,
                          uint64_t rows_full) {
  using namespace fnv;
  extern __shared__ __align__(1024) unsigned char smem_t[];
  WitnessTcSmem& sh = *reinterpret_cast<WitnessTcSmem*>(smem_t + ((1024u - (smem_addr(smem_t) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n_seg = (n + 31) / 32;
  const int64_t G = gridDim.x;
  constexpr int kProducer = kComputeWarps, kMma = kComputeWarps + 1, kMma2 = kComputeWarps + 2;
  {  // B tables
    const uint4* src = reinterpret_cast<const uint4*>(&g_tcw[0][0][0]);
    uint4* dst = reinterpret_cast<uint4*>(&sh.wb[0][0][0]);
    for (int i = tid; i < static_cast<int>(sizeof(sh.wb) / 16); i += kTcThreads) dst[i] = src[i];
  }
  if (tid == 0) {
    for (int b = 0; b < kWitnessBufs; ++b) {
      mbar_init(&sh.full[b], 1);
      mbar_init(&sh.empty[b], 1);
      mbar_init(&sh.mma1[b], 1);
      mbar_init(&sh.mma2[b], 1);
      mbar_init(&sh.uab[b], kComputeWarps);
      mbar_init(&sh.tfree[b], 4);
    }
    mbar_init(&sh.tail, kComputeWarps);
    sh.abort = 0;
  }
  if (warp == kMma) {  // TMEM for 3 x 2 accumulators (one warp allocates and frees)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&sh.tmem)),
                 "r"(kTcCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_shared();  // the B tables, for the tensor cores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem;
  volatile uint32_t* abort = &sh.abort;
  // (32-bit chunk counters: buffer index and phase by multiply, not a 64-bit division)
  const uint32_t my_chunks = blockIdx.x < n_chunks ? static_cast<uint32_t>((n_chunks - 1 - blockIdx.x) / G + 1) : 0;
  uint64_t acc = 0;
  bool ok = true;
  if (warp == kProducer) {  // ---- rows + witness words of every chunk, kWitnessBufs ahead
    if (lane == 0)
      for (uint32_t i = 0; i < my_chunks; ++i) {
        const int b = static_cast<int>(i % kWitnessBufs);
        if (i >= kWitnessBufs && !mbar_wait_tc(&sh.empty[b], static_cast<uint32_t>(i / kWitnessBufs - 1) & 1u, abort))
          break;
        const uint64_t row0 = (blockIdx.x + static_cast<uint64_t>(i) * G) * kComputeThreads;
        int boxes = 0;
#pragma unroll
        for (int x = 0; x < kComputeThreads / kTmaBoxRows; ++x) boxes += row0 + kTmaBoxRows * x < rows_full;
        mbar_arrive_expect_tx(&sh.full[b], boxes * kTmaBoxRows * kThreadBytes + 4 * kWitnessWords);
        for (int x = 0; x < boxes; ++x)
          tma_load_rows(&sh.data[b][kGranules * kTmaBoxRows * x], &tmap, static_cast<int32_t>(row0 + kTmaBoxRows * x),
                        &sh.full[b]);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(&sh.wit[b][0])),
            "l"(witness + row0), "r"(4 * kWitnessWords), "r"(smem_addr(&sh.full[b]))
            : "memory");
      }
  } else if (warp == kMma) {  // ---- MMA 1 of every chunk, as soon as its bytes land
    if (lane == 0)
      for (uint32_t i = 0; i < my_chunks; ++i) {
        const int b = static_cast<int>(i % kWitnessBufs);
        const uint32_t ph = static_cast<uint32_t>(i / kWitnessBufs) & 1u;
        if (!mbar_wait_tc(&sh.full[b], ph, abort)) break;
        if (i >= kWitnessBufs && !mbar_wait_tc(&sh.tfree[b], ph ^ 1u, abort)) break;  // chunk i-3 folded
        const bool last = ((blockIdx.x + static_cast<uint64_t>(i) * G) + 1) * kComputeThreads > rows_full;
        if (last && !mbar_wait_tc(&sh.tail, 0, abort)) break;  // the partial rows, written by their threads
        tc_fence_after();
        tc_chunk_mma(tmem + 2 * kTcN * b, smem_addr(&sh.data[b][0]), smem_addr(&sh.wb[0][0][0]));  // bytes as landed
        tc_commit(&sh.mma1[b]);
      }
  } else if (warp == kMma2) {  // ---- MMA 2 of every chunk, once its u & b rows are written
    if (lane == 0)
      for (uint32_t i = 0; i < my_chunks; ++i) {
        const int b = static_cast<int>(i % kWitnessBufs);
        const uint32_t ph = static_cast<uint32_t>(i / kWitnessBufs) & 1u;
        // (uab follows mma1 of the same chunk, which followed the fold of chunk i-3)
        if (!mbar_wait_tc(&sh.uab[b], ph, abort)) break;
        tc_fence_after();
        tc_chunk_mma(tmem + 2 * kTcN * b + kTcN, smem_addr(&sh.data[b][0]), smem_addr(&sh.wb[1][0][0]));
        tc_commit(&sh.mma2[b]);
        tc_commit(&sh.empty[b]);  // the rows are free for the producer
      }
  } else {  // ---- compute warps: the automaton; warps 0-3 fold the accumulators
    const int m = 32 * (warp & 3) + lane;                                      // this lane's TMEM lane
    const uint64_t w_nat = pow_u64(kPrimeInv, static_cast<uint64_t>(m));       // MMA 1: natural byte m
    const uint64_t w_il = pow_u64(kPrimeInv, static_cast<uint64_t>(32 * (m & 3) + (m >> 2)));  // MMA 2: 4j+s
    auto fold = [&](uint32_t j) {
      const int b = static_cast<int>(j % kWitnessBufs);
      if (!mbar_wait_tc(&sh.mma2[b], static_cast<uint32_t>(j / kWitnessBufs) & 1u, abort)) return;
      tc_fence_after();
      uint32_t r0[8], r1[8];
      const uint32_t t = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + 2 * kTcN * b;
      tc_ld8(t, r0);
      tc_ld8(t + kTcN, r1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      uint64_t s0 = 0, s1 = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s0 += static_cast<uint64_t>(r0[q]) << (8 * q);
        s1 += static_cast<uint64_t>(r1[q]) << (8 * q);
      }
      acc += (s0 * w_nat + s1 * w_il) * chunk_weight(static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(j) * G);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.tfree[b]);
    };
    for (uint32_t i = 0; i < my_chunks; ++i) {  // (a timed-out wait breaks the loop)
      const int b = static_cast<int>(i % kWitnessBufs);
      const uint32_t ph = static_cast<uint32_t>(i / kWitnessBufs) & 1u;
      if (warp < 4 && i > 1) fold(i - 2);  // the sums of two chunks back, long done
      if (!mbar_wait_tc(&sh.full[b], ph, abort)) break;
      const int64_t chunk = blockIdx.x + static_cast<int64_t>(i) * G;
      uint4* rows = sh.data[b];
      const uint64_t row = static_cast<uint64_t>(chunk) * kComputeThreads + tid;
      uint32_t st = 0, expect = 0, check = 0;
      const bool tail_chunk = (static_cast<uint64_t>(chunk) + 1) * kComputeThreads > rows_full;
      if (!tail_chunk && (static_cast<uint64_t>(chunk) + 1) * kComputeThreads < rows_full) {
        // interior chunk: every row full and followed by another (the next
        // chunk's first witness word rides along)
        st = sh.wit[b][tid];
        expect = (st >> 8) | ((sh.wit[b][tid + 1] & 0xffu) << 24);
        check = ~0u;
        if (chunk == 0 && tid == 0 && (st & 0xffu) != (seed & 0xffu)) ok = false;
      } else if (row * kThreadBytes < n) {
        st = sh.wit[b][tid];
        const uint64_t seg0 = 4 * row;
        const uint32_t next = seg0 + 4 < n_seg ? (sh.wit[b][tid + 1] & 0xffu) : 0u;
        expect = (st >> 8) | (next << 24);  // segment i ends where segment i+1 starts
        if (seg0 + 4 < n_seg) {
          check = ~0u;
        } else {  // the record's last row: no successor past the last segment
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (seg0 + q + 1 < n_seg) check |= 0xffu << (8 * q);
        }
        if (row == 0 && (st & 0xffu) != (seed & 0xffu)) ok = false;
      }
      if (tail_chunk) {  // the partial rows: before MMA 1
        if (row >= rows_full) witness_row_bytes(rows, tid, data, n, row * kThreadBytes);
        fence_async_shared();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.tail);
      }
      uint32_t w[kThreadWords];
      read_thread_rows(rows, tid, w);
      interleave(w);
      const uint32_t ends = automaton_and_ends(w, st);
      if ((ends ^ expect) & check) ok = false;
      if (!mbar_wait_tc(&sh.mma1[b], ph, abort)) break;  // MMA 1 has read the bytes
      write_thread_rows(rows, tid, w);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.uab[b]);
    }
    for (uint32_t j = my_chunks > 2 ? my_chunks - 2 : 0; warp < 4 && j < my_chunks && !*abort; ++j) fold(j);
  }
  if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicExch(bad, 1ull);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) sh.red[warp] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*abort && tid == 0) atomicExch(bad, 1ull);  // a wait timed out: the sum is not the record's
  if (warp == kMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcCols) : "memory");
  if (tid == 0) {
    uint64_t sum = 0;
    for (int q = 0; q < 4; ++q) sum += sh.red[q];
    atomicAdd(scr.accum, static_cast<unsigned long long>(sum));
    __threadfence();
    if (atomicAdd(scr.finished, 1u) + 1 == gridDim.x) {
      __threadfence();
      const uint64_t total = atomicAdd(scr.accum, 0ull);
      *scr.result = pow_p(n) * (total + seed);
    }
  }
}

}  // namespace

void init_constants() {
  // P^-(c * kChunk) = T0[c & 1023] * T1[(c >> 10) & 1023] * T2[c >> 20]
  static unsigned long long t[3][1024];
  for (int l = 0; l < 3; ++l) {
    const uint64_t step = fnv::pow_u64(fnv::kPrimeInv, static_cast<uint64_t>(fnv::kChunk) << (10 * l));
    uint64_t x = 1;
    for (int i = 0; i < 1024; ++i) {
      t[l][i] = x;
      x *= step;
    }
  }
  MLCK_CUDA(cudaMemcpyToSymbol(fnv::c_wchunk, t, sizeof(t)));
  // the witness kernel's tensor-core tables (fnv.cuh mma_tables, once)
  static uint2 wf[2][4][32];
  static unsigned long long kp[32][4], pw[fnv::kComputeWarps];
  for (int tab = 0; tab < 2; ++tab)
    for (int kb = 0; kb < 4; ++kb)
      for (int lane = 0; lane < 32; ++lane) {
        const int nn = lane >> 2, q = lane & 3;
        uint32_t b[2] = {0, 0};
        for (int h = 0; h < 2; ++h)
          for (int e = 0; e < 4; ++e) {
            const int seg = fnv::mma_segment(kb, 16 * h + 4 * q + e);
            uint64_t wgt = fnv::pow_u64(fnv::kPrime, 32ull * (127 - seg));
            if (tab) wgt *= ~1ull;
            b[h] |= static_cast<uint32_t>((wgt >> (8 * nn)) & 0xffu) << (8 * e);
          }
        wf[tab][kb][lane] = make_uint2(b[0], b[1]);
      }
  for (int lane = 0; lane < 32; ++lane)
    for (int m = 0; m < 4; ++m) {
      const int g = lane >> 2, q = lane & 3;
      kp[lane][m] = fnv::pow_u64(fnv::kPrime, 32 - (4 * g + m)) << (16 * q);
    }
  for (int w = 0; w < fnv::kComputeWarps; ++w)
    pw[w] = fnv::pow_u64(fnv::kPrimeInv, static_cast<uint64_t>(fnv::kThreadBytes) * 32 * (w + 1));
  // tcgen05 verifier B tables: limb n of P^-(128 k) and of -2 P^-(128 k)
  static uint8_t tw[2][fnv::kComputeThreads][kTcN];
  std::memset(tw, 0, sizeof(tw));
  for (int k = 0; k < fnv::kComputeThreads; ++k) {
    const uint64_t pk = fnv::pow_u64(fnv::kPrimeInv, 128ull * k);
    for (int nn = 0; nn < 8; ++nn) {
      tw[0][k][nn] = static_cast<uint8_t>(pk >> (8 * nn));
      tw[1][k][nn] = static_cast<uint8_t>((pk * ~1ull) >> (8 * nn));
    }
  }
  MLCK_CUDA(cudaMemcpyToSymbol(g_tcw, tw, sizeof(tw)));
  MLCK_CUDA(cudaMemcpyToSymbol(g_wfrag, wf, sizeof(wf)));
  MLCK_CUDA(cudaMemcpyToSymbol(g_kpos, kp, sizeof(kp)));
  MLCK_CUDA(cudaMemcpyToSymbol(c_pinv_warp, pw, sizeof(pw)));
}

uint64_t fnv_chunks(uint64_t n) { return div_up(n, fnv::kChunk); }
// [256 B header: chunk ticket u64 @0, finished u32 @8, accum u64 @16, ulast u32 @24, error u32
//  @28, sticky watchdog u32 @32 (not cleared per launch)] [status: n_chunks
//  words of 8 B at a kStatusStride * 8 B (128 B) stride]
size_t fnv_scratch_words(uint64_t n) { return (256 + fnv_chunks(n) * fnv::kStatusStride * 8) / 4; }

uint64_t fnv_chunk_bytes() { return fnv::kChunk; }
uint32_t fnv_sticky_word() { return 8; }

// The bytes [data, data + n) as a [n / 128 rows x 128 bytes] tensor map (the
// full rows only), 256-row boxes landing in the 128-byte swizzle the FNV
// kernels' shared-memory rows use.  False when the TMA cannot serve it.
// `rows` x 128-byte rows at data as a tensor map with `box_rows`-row boxes in
// the 128-byte swizzle of the FNV kernels' shared-memory rows.
#ifndef MLCK_TMA_L2_PROMOTION
#define MLCK_TMA_L2_PROMOTION 3  // CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
void encode_rows(const uint8_t* data, uint64_t rows, uint32_t box_rows, CUtensorMap* tmap) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    MLCK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                      &q));
    if (q != cudaDriverEntryPointSuccess || !encode) throw Error(kCuda, "cuTensorMapEncodeTiled unavailable");
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(fnv::kThreadBytes), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(fnv::kThreadBytes)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(fnv::kThreadBytes), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(data), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            static_cast<CUtensorMapL2promotion>(MLCK_TMA_L2_PROMOTION), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}
bool make_row_tmap(const uint8_t* data, uint64_t n, CUtensorMap* tmap) {
  std::memset(tmap, 0, sizeof(*tmap));
  const uint64_t rows = n / fnv::kThreadBytes;
  if (rows == 0 || (reinterpret_cast<uintptr_t>(data) & 15u) != 0 || rows >= (1ull << 31)) return false;
  encode_rows(data, rows, fnv::kTmaBoxRows, tmap);
  return true;
}

void launch_fnv(const uint8_t* data, uint64_t n, uint64_t seed, uint32_t* scratch, uint32_t epoch,
                unsigned long long* result, const TrailerDsts& trailer, cudaStream_t stream,
                unsigned long long* prof, unsigned long long* trace, const FnvFused* fused,
                int reserve_sms, const pack::Dsts* copies, uint32_t* witness) {
  const uint64_t n_chunks = fnv_chunks(n);
  fnv::Scratch scr{};
  scr.witness = witness;
  scr.ticket = reinterpret_cast<unsigned long long*>(scratch);
  scr.finished = scratch + 2;
  scr.accum = reinterpret_cast<unsigned long long*>(scratch + 4);
  scr.ulast = scratch + 6;
  scr.error = scratch + 7;
  scr.sticky = scratch + fnv_sticky_word();
  scr.result = result;
  scr.status = reinterpret_cast<unsigned long long*>(scratch + 64);
  scr.epoch = epoch;
  scr.prof = prof;
  scr.trace = trace;
  MLCK_CUDA(cudaMemsetAsync(scratch, 0, 32, stream));  // words 0-7: status is epoch-tagged, word 8 sticky
  if (n_chunks == 0) {
    // empty input: h = seed
    launch_fnv_empty(seed, result, trailer, stream);
    return;
  }
  // one CTA per SM (its shared memory holds kSlots chunks); tickets make any
  // grid size correct, reserve_sms leaves SMs to co-scheduled work
  static int sms_of[64] = {0};
  int dev = 0;
  MLCK_CUDA(cudaGetDevice(&dev));
  int& sms = sms_of[dev & 63];
  if (sms == 0) {
    for (auto* k : {fnv_kernel<false, false>, fnv_kernel<true, false>, fnv_kernel<false, true>,
                    fnv_kernel<true, true>})
      MLCK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(fnv::kSmemBytes)));
    int per_sm = 0;
    MLCK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fnv_kernel<false, false>, fnv::kThreads,
                                                             fnv::kSmemBytes));
    if (per_sm < 1) throw Error(kCuda, "fnv_kernel does not fit on an SM");
    MLCK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const uint64_t grid = std::min<uint64_t>(div_up(n_chunks, fnv::kSlots), static_cast<uint64_t>(std::max(1, sms - reserve_sms)));
  // copies: TMA stores of every hashed chunk; fused: chunks from the sources
  static_assert(sizeof(FnvRun) == sizeof(fnv::Run) && kFnvMaxSrc == fnv::kMaxSrc, "FnvRun mirrors fnv::Run");
  fnv::Copy cp;
  std::memset(&cp, 0, sizeof(cp));
  if (copies && copies->n > 0) {
    if (n < fnv::kThreadBytes || (reinterpret_cast<uintptr_t>(data) & 15u))
      throw_invalid("hash copies need a 16-byte aligned record of at least one row");
    cp.n_dst = copies->n;
    for (int d = 0; d < copies->n; ++d) {
      if (reinterpret_cast<uintptr_t>(copies->p[d]) & 15u) throw_invalid("copy destinations must be 16-byte aligned");
      encode_rows(copies->p[d], n / fnv::kThreadBytes, fnv::kTmaBoxRows, &cp.dst[d]);
      cp.dst_ptr[d] = copies->p[d];
    }
  }
  if (fused) {
    if (!cp.n_dst) throw_invalid("a fused snapshot stores to at least the record");
    if (fused->n_src < 1 || fused->n_src > fnv::kMaxSrc) throw_invalid("fused snapshot: 1-6 source maps");
    for (int m = 0; m < fused->n_src; ++m) {
      const uint64_t rows = fused->src_bytes[m] / fnv::kThreadBytes;
      if ((reinterpret_cast<uintptr_t>(fused->src[m]) & 15u) || rows == 0 || rows >= (1ull << 31))
        throw_invalid("fused snapshot: a source map must be 16-byte aligned, 128 B .. 256 GiB");
      encode_rows(fused->src[m], rows, fnv::kTmaBoxRows, &cp.src[m][0]);
      encode_rows(fused->src[m], rows, 8, &cp.src[m][1]);
    }
    cp.runs = reinterpret_cast<const fnv::Run*>(fused->runs);
    cp.n_runs = fused->n_runs;
#ifdef MLCK_FUSED_NOSTORE  // development A/B only (no record written): the cost of the TMA stores
    cp.n_dst = 0;
#endif
  }
  // the record as a [n / 128 rows x 128 bytes] tensor, loaded in 256-row
  // boxes in the 128-byte swizzle the shared-memory rows use
  CUtensorMap tmap;
  const int use_tma = !fused && make_row_tmap(data, n, &tmap) ? 1 : 0;
  if (cp.n_dst && !fused && !use_tma) throw_invalid("hash copies need the record's tensor map");
  const bool pf = prof || trace;
  auto k = fused ? (pf ? fnv_kernel<true, true> : fnv_kernel<false, true>)
                 : (pf ? fnv_kernel<true, false> : fnv_kernel<false, false>);
  k<<<static_cast<unsigned>(grid), fnv::kThreads, fnv::kSmemBytes, stream>>>(
      data, n, seed, scr, static_cast<int64_t>(n_chunks), trailer, cp, tmap, use_tma);
  MLCK_CUDA(cudaGetLastError());
}

namespace {
// The straddling chunks of a fused snapshot: block (x, j) gathers 4 KiB of
// chunk chunks[j], 16 bytes per thread (zeros past the record end).
__global__ void patch_chunks_kernel(const pack::Segment* __restrict__ segs, int n_segs,
                                    const int64_t* __restrict__ chunks, uint64_t n, uint8_t* __restrict__ out) {
  const uint64_t off = 4096ull * blockIdx.x + 16ull * threadIdx.x;
  const uint64_t pos = static_cast<uint64_t>(chunks[blockIdx.y]) * fnv::kChunk + off;
  uint32_t v[4] = {0, 0, 0, 0};
  if (pos < n) {
    int s = pack::find_segment(segs, n_segs, pos);
    for (int k = 0; k < 16 && pos + k < n; ++k) {
      while (segs[s].dst + segs[s].len <= pos + k) ++s;
      v[k >> 2] |= static_cast<uint32_t>(segs[s].src[pos + k - segs[s].dst]) << (8 * (k & 3));
    }
  }
  *reinterpret_cast<uint4*>(out + static_cast<uint64_t>(blockIdx.y) * fnv::kChunk + off) =
      make_uint4(v[0], v[1], v[2], v[3]);
}
}  // namespace

void launch_patch_chunks(const pack::Segment* segs, int n_segs, const int64_t* chunks, uint64_t n_patch, uint64_t n,
                         uint8_t* out, cudaStream_t stream) {
  if (!n_patch) return;
  static_assert(fnv::kChunk % 4096 == 0, "4 KiB blocks");
  patch_chunks_kernel<<<dim3(fnv::kChunk / 4096, static_cast<unsigned>(n_patch)), 256, 0, stream>>>(
      segs, n_segs, chunks, n, out);
  MLCK_CUDA(cudaGetLastError());
}

namespace {
__global__ void fnv_empty_kernel(uint64_t seed, unsigned long long* result, TrailerDsts trailer) {
  *result = seed;
  for (int r = 0; r < trailer.n; ++r)
    for (int b = 0; b < 8; ++b) trailer.p[r][b] = static_cast<uint8_t>(seed >> (8 * b));
}
}  // namespace

void launch_fnv_empty(uint64_t seed, unsigned long long* result, const TrailerDsts& trailer,
                      cudaStream_t stream) {
  fnv_empty_kernel<<<1, 1, 0, stream>>>(seed, result, trailer);
  MLCK_CUDA(cudaGetLastError());
}

void launch_fnv_witness(const uint8_t* data, uint64_t n, uint64_t seed, const uint32_t* witness, uint32_t* scratch,
                        unsigned long long* result, unsigned long long* bad, cudaStream_t stream, int ctas) {
  MLCK_CUDA(cudaMemsetAsync(scratch, 0, 32, stream));
  MLCK_CUDA(cudaMemsetAsync(bad, 0, 8, stream));
  if (n == 0) {
    launch_fnv_empty(seed, result, TrailerDsts{}, stream);
    return;
  }
  static int sms_of[64] = {0};
  int dev = 0;
  MLCK_CUDA(cudaGetDevice(&dev));
  int& sms = sms_of[dev & 63];
  if (!sms) {
    MLCK_CUDA(cudaFuncSetAttribute(fnv_witness_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kWitnessSmem)));
    MLCK_CUDA(cudaFuncSetAttribute(fnv_witness_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kWitnessTcSmem)));
    MLCK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  CUtensorMap tmap;
  const uint64_t rows_full = make_row_tmap(data, n, &tmap) ? n / fnv::kThreadBytes : 0;
  fnv::Scratch scr{};
  scr.finished = scratch + 2;
  scr.accum = reinterpret_cast<unsigned long long*>(scratch + 4);
  scr.result = result;
  const int64_t n_chunks = static_cast<int64_t>(fnv_chunks(n));
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n_chunks, ctas > 0 ? std::min(ctas, sms) : sms));
  if (MLCK_WITNESS_TC && rows_full > 0)  // the dot products on tcgen05 (the record's rows load by TMA)
    fnv_witness_tc_kernel<<<grid, kTcThreads, kWitnessTcSmem, stream>>>(data, n, seed, witness, scr, bad, n_chunks,
                                                                        tmap, rows_full);
  else
    fnv_witness_kernel<<<grid, kWitnessThreads, kWitnessSmem, stream>>>(data, n, seed, witness, scr, bad, n_chunks,
                                                                        tmap, rows_full);
  MLCK_CUDA(cudaGetLastError());
}


// ---------------------------------------------------------------- pack (K1)
void launch_pack(const pack::Segment* segs, int n_segs, uint64_t total, const pack::Dsts& d,
                 cudaStream_t stream, uint64_t lo) {
  if (total <= lo) return;
  if (lo % pack::kTile) throw_invalid("pack piece start must be tile aligned");
  const uint64_t first = lo / pack::kTile, tiles = div_up(total, pack::kTile) - first;
  pack::pack_kernel<<<static_cast<unsigned>(tiles), pack::kThreads, 0, stream>>>(segs, n_segs, total, d, first);
  MLCK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- record walk
namespace {
__device__ __forceinline__ uint64_t rd(const uint8_t* p, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

// parse_record's header/entry walk (snapshot.hpp:166-196) after the
// checksum passed.  One thread per blob: entry k's offset depends on the
// parameter count of entry k-1.
__global__ void walk_kernel(const WalkJob* jobs, int n_jobs) {
  const int j = blockIdx.x;
  if (j >= n_jobs || threadIdx.x != 0) return;
  const WalkJob job = jobs[j];
  WalkResult* res = job.result;
  const uint8_t* b = job.blob;
  const uint64_t end = job.n >= 8 ? job.n - 8 : 0;
  uint64_t pos = 0;
  res->status = kWalkOk;
  res->n_entries = 0;
#define NEED(k)                          \
  if (pos + (k) > end) {                 \
    res->status = kWalkTruncated;        \
    return;                              \
  }
  NEED(4);
  if (rd(b + pos, 4) != 0x4b434c4du) {
    res->status = kWalkMagic;
    return;
  }
  pos += 4;
  NEED(4);
  res->version = static_cast<uint32_t>(rd(b + pos, 4));
  pos += 4;
  if (res->version != 1u) {
    res->status = kWalkVersion;
    return;
  }
  NEED(1); res->kind = b[pos]; pos += 1;
  NEED(8); res->iteration = rd(b + pos, 8); pos += 8;
  NEED(8); res->window_start = rd(b + pos, 8); pos += 8;
  NEED(4); res->wsparse = static_cast<uint32_t>(rd(b + pos, 4)); pos += 4;
  NEED(4); res->slot = static_cast<uint32_t>(rd(b + pos, 4)); pos += 4;
  NEED(8); res->data_seed = rd(b + pos, 8); pos += 8;
  NEED(4); res->op_count = static_cast<uint32_t>(rd(b + pos, 4)); pos += 4;
  for (uint32_t i = 0; i < res->op_count; ++i) {
    WalkEntry e;
    NEED(4); e.id = static_cast<uint32_t>(rd(b + pos, 4)); pos += 4;
    NEED(1); e.mode = b[pos]; pos += 1;
    NEED(8); e.param_count = rd(b + pos, 8); pos += 8;
    e.step = 0;
    if (e.mode == 0) {
      NEED(8); e.step = rd(b + pos, 8); pos += 8;
      e.payload_offset = pos;
      if (e.param_count > end || 12 * e.param_count > end - pos) {
        res->status = kWalkTruncated;
        return;
      }
      pos += 12 * e.param_count;
    } else {
      if (job.compute_bytes != 1 && job.compute_bytes != 2 && job.compute_bytes != 4) {
        res->status = kWalkWidth;
        return;
      }
      e.payload_offset = pos;
      const uint64_t need = static_cast<uint64_t>(job.compute_bytes) * e.param_count;
      if (e.param_count > end || need > end - pos) {
        res->status = kWalkTruncated;
        return;
      }
      pos += need;
    }
    if (i < job.cap) job.entries[i] = e;
    res->n_entries = i + 1;
  }
#undef NEED
}
}  // namespace

void launch_walk(const WalkJob* jobs, int n_jobs, cudaStream_t stream) {
  if (n_jobs == 0) return;
  walk_kernel<<<n_jobs, 32, 0, stream>>>(jobs, n_jobs);
  MLCK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- replay (K3)
void launch_replay(const adam::ConvOp* ops, int n_ops, const float* const* gptr, const float2* bc, uint32_t n_bc,
                   adam::StepConst* steps, const adam::Opt& o, int cb, uint64_t total_units, cudaStream_t stream) {
  if (total_units == 0) return;
  if (n_bc) {
    adam::replay_steps_kernel<<<(n_bc + 127) / 128, 128, 0, stream>>>(bc, steps, n_bc);
    MLCK_CUDA(cudaGetLastError());
  }
  const uint64_t blocks = total_units;  // total_units counts CTAs (run_replay)
  adam::replay_kernel<<<static_cast<unsigned>(blocks), adam::kReplayThreads, 0, stream>>>(ops, n_ops, gptr, bc,
                                                                                        steps, o, cb, total_units);
  MLCK_CUDA(cudaGetLastError());
}

int replay_cta_threads() { return adam::kReplayThreads; }
int replay_unit_elems() { return adam::kReplayVec; }

void launch_fastmath_check(uint64_t n, uint64_t seed, unsigned long long* counts, cudaStream_t stream) {
  adam::fastmath_check_kernel<<<148 * 8, 256, 0, stream>>>(n, seed, counts);
  MLCK_CUDA(cudaGetLastError());
}

namespace {
__global__ void adam_arrays_kernel(float* w, float* m, float* v, const float* g, uint64_t n,
                                   adam::Opt o, float bc1, float bc2) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float ww = w[i], mm = m[i], vv = v[i];
    adam::adam_elem(ww, mm, vv, g[i], o, bc1, bc2);
    w[i] = ww;
    m[i] = mm;
    v[i] = vv;
  }
}
}  // namespace

void launch_adam_arrays(float* w, float* m, float* v, const float* g, uint64_t n,
                        const adam::Opt& o, float bc1, float bc2, cudaStream_t stream) {
  if (n == 0) return;
  const unsigned blocks = static_cast<unsigned>(div_up(n, 256) < 148ull * 16 ? div_up(n, 256) : 148ull * 16);
  adam_arrays_kernel<<<blocks, 256, 0, stream>>>(w, m, v, g, n, o, bc1, bc2);
  MLCK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- codecs
namespace {
__global__ void quantize_kernel(const float* in, float* out, uint64_t n, int cb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    // bit moves only: round_to_format returns NaN untouched, payload and
    // signalling bit included (tensor.hpp:39), so no FP op may touch it
    const uint32_t b = reinterpret_cast<const uint32_t*>(in)[i];
    uint32_t o = b;
    if ((b & 0x7fffffffu) <= 0x7f800000u) {
      const float x = __uint_as_float(b);
      if (cb == 2) o = __float_as_uint(codec::decode_half(codec::encode_half(x)));
      else if (cb == 1) o = __float_as_uint(codec::decode_e4m3(codec::encode_e4m3(x)));
    }
    reinterpret_cast<uint32_t*>(out)[i] = o;
  }
}
__global__ void encode_kernel(const float* in, void* codes, uint64_t n, int cb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    codec::store_code(codes, i, in[i], cb);
}
__global__ void decode_kernel(const void* codes, float* out, uint64_t n, int cb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = codec::load_code(codes, i, cb);
}
unsigned grid_for(uint64_t n) {
  const uint64_t b = div_up(n, 256);
  return static_cast<unsigned>(b < 148ull * 32 ? (b ? b : 1) : 148ull * 32);
}
__global__ void pack_generic_kernel(const float* in, uint16_t* out, uint64_t n, int eb, int mb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = codec::pack_generic(in[i], eb, mb);
}
__global__ void unpack_generic_kernel(const uint16_t* in, float* out, uint64_t n, int eb, int mb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = codec::unpack_generic(in[i], eb, mb);
}
}  // namespace

void launch_pack_reduced(const float* in, uint16_t* codes, uint64_t n, int eb, int mb, cudaStream_t stream) {
  if (!n) return;
  pack_generic_kernel<<<grid_for(n), 256, 0, stream>>>(in, codes, n, eb, mb);
  MLCK_CUDA(cudaGetLastError());
}
void launch_unpack_reduced(const uint16_t* codes, float* out, uint64_t n, int eb, int mb, cudaStream_t stream) {
  if (!n) return;
  unpack_generic_kernel<<<grid_for(n), 256, 0, stream>>>(codes, out, n, eb, mb);
  MLCK_CUDA(cudaGetLastError());
}

void launch_quantize(const float* in, float* out, uint64_t n, int cb, cudaStream_t stream) {
  if (!n) return;
  quantize_kernel<<<grid_for(n), 256, 0, stream>>>(in, out, n, cb);
  MLCK_CUDA(cudaGetLastError());
}
void launch_encode(const float* in, void* codes, uint64_t n, int cb, cudaStream_t stream) {
  if (!n) return;
  encode_kernel<<<grid_for(n), 256, 0, stream>>>(in, codes, n, cb);
  MLCK_CUDA(cudaGetLastError());
}
void launch_decode(const void* codes, float* out, uint64_t n, int cb, cudaStream_t stream) {
  if (!n) return;
  decode_kernel<<<grid_for(n), 256, 0, stream>>>(codes, out, n, cb);
  MLCK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- synthetic
namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// == mlo_synth_value (oracle/moelab_oracle.c)
__device__ __forceinline__ float synth(uint64_t key, uint64_t index, float lo, float span) {
  const uint64_t x = mix64(key ^ index);
  const float u = static_cast<float>(x >> 40) * 0x1.0p-24f;
  return __fadd_rn(lo, __fmul_rn(span, u));
}
__global__ void synth_kernel(float* out, uint64_t n, uint64_t key, float lo, float span) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = synth(key, i, lo, span);
}
}  // namespace

uint64_t synth_key(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x632be59bd9b4e019ull * (stream + 1);
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void launch_synth(float* out, uint64_t n, uint64_t seed, uint64_t stream_id, float lo, float hi,
                  cudaStream_t stream) {
  if (!n) return;
  const float span = hi - lo;
  synth_kernel<<<grid_for(n), 256, 0, stream>>>(out, n, synth_key(seed, stream_id), lo, span);
  MLCK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- copies
namespace {
// SM-driven copy (peer HBM log ring: remote stores over NVLink)
__global__ void copy_kernel(uint4* dst, const uint4* src, uint64_t n_vec) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_vec;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

namespace {
// Replica push on a fixed set of SMs: one CTA per SM (the dynamic shared
// memory request keeps any other CTA off it), 128-bit loads from the local
// record and stores to every replica (peer pointers: NVLink stores).
__global__ void __launch_bounds__(1024, 1)
    push_kernel(const uint4* __restrict__ src, uint64_t n_vec, pack::Dsts d) {
  for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < n_vec; i += gridDim.x * 1024ull) {
    const uint4 v = ld_stream(src + i);
#pragma unroll
    for (int r = 0; r < pack::kMaxDst; ++r)
      if (r < d.n) st_v4(d.p[r] + 16 * i, v);
  }
}
}  // namespace

void launch_push(const uint8_t* src, uint64_t bytes, const pack::Dsts& d, int ctas, cudaStream_t stream) {
  static size_t smem = 0;
  if (smem == 0) {
    smem = 120 * 1024;  // > half an SM's shared memory: one CTA per SM
    MLCK_CUDA(cudaFuncSetAttribute(push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  }
  const uint64_t n_vec = bytes / 16;
  if (n_vec)
    push_kernel<<<ctas, 1024, smem, stream>>>(reinterpret_cast<const uint4*>(src), n_vec, d);
  MLCK_CUDA(cudaGetLastError());
  for (int r = 0; r < d.n; ++r)
    if (bytes > n_vec * 16)
      MLCK_CUDA(cudaMemcpyAsync(d.p[r] + n_vec * 16, src + n_vec * 16, bytes - n_vec * 16, cudaMemcpyDefault,
                                stream));
}

void launch_copy16(void* dst, const void* src, uint64_t bytes, cudaStream_t stream) {
  const uint64_t n_vec = bytes / 16;
  if (n_vec) {
    copy_kernel<<<grid_for(n_vec), 256, 0, stream>>>(static_cast<uint4*>(dst),
                                                     static_cast<const uint4*>(src), n_vec);
    MLCK_CUDA(cudaGetLastError());
  }
  const uint64_t rem = bytes - n_vec * 16;
  if (rem)
    MLCK_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + n_vec * 16,
                              static_cast<const uint8_t*>(src) + n_vec * 16, rem,
                              cudaMemcpyDeviceToDevice, stream));
}

}  // namespace mlck
