// pack.cuh -- K1: gather byte segments into one contiguous, byte-packed
// container at arbitrary alignment (the MLCK record of snapshot.hpp:61-144,
// the MLST image of engine.hpp:246-261, the dense MLCK of snapshot.hpp:251).
//
// The reference builds the record with std::vector appends
// (ByteWriter::raw, digest.hpp:67-69) and per-element codec calls
// (write_compute, snapshot.hpp:77-93).  Here the device arena already holds
// every payload in its wire encoding (master|m|v contiguous per operator,
// compute codes per operator), so a record is a list of (dst offset, length,
// src pointer) segments: 45-byte header + 13/21-byte entry headers from a
// small metadata buffer, and payload spans straight from the arena.
//
// Output-driven: each CTA owns one 16 KiB output tile; a tile lying inside
// one segment (the common case -- payloads are MBs) is copied with aligned
// 128-bit loads, a per-tile byte funnel shift (payload offsets are arbitrary
// mod 16: 45 + 13k + 8f + ... bytes) and aligned 128-bit stores to the local
// buffer and to every replica (peer-mapped pointers go out over NVLink).
// Tiles that straddle segment boundaries (one per boundary) take a byte path.
#pragma once

#include "mlck_common.cuh"

namespace mlck {
namespace pack {

#ifndef MLCK_PACK_THREADS
#define MLCK_PACK_THREADS 256
#endif
#ifndef MLCK_PACK_VEC
#define MLCK_PACK_VEC 2
#endif
constexpr int kThreads = MLCK_PACK_THREADS;
constexpr int kVecPerThread = MLCK_PACK_VEC;
constexpr int kTile = kThreads * kVecPerThread * 16;  // 8 KiB (swept: 4-16 KiB, 128-512 threads)
constexpr int kMaxDst = 4;                            // local + up to 3 replicas

struct Segment {
  uint64_t dst;  // byte offset in the output
  uint64_t len;
  const uint8_t* src;
};

struct Dsts {
  uint8_t* p[kMaxDst];
  int n;
};

__device__ __forceinline__ int find_segment(const Segment* segs, int n_segs, uint64_t pos) {
  int lo = 0, hi = n_segs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].dst <= pos) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// out = bytes [sh, sh+16) of the 32-byte concatenation a|b (little endian)
__device__ __forceinline__ uint4 funnel16(const uint4& a, const uint4& b, uint32_t sh) {
  const uint32_t r = (sh & 3u) * 8u;
  uint4 o;
  switch (sh >> 2) {
    case 0:
      o.x = __funnelshift_r(a.x, a.y, r); o.y = __funnelshift_r(a.y, a.z, r);
      o.z = __funnelshift_r(a.z, a.w, r); o.w = __funnelshift_r(a.w, b.x, r);
      break;
    case 1:
      o.x = __funnelshift_r(a.y, a.z, r); o.y = __funnelshift_r(a.z, a.w, r);
      o.z = __funnelshift_r(a.w, b.x, r); o.w = __funnelshift_r(b.x, b.y, r);
      break;
    case 2:
      o.x = __funnelshift_r(a.z, a.w, r); o.y = __funnelshift_r(a.w, b.x, r);
      o.z = __funnelshift_r(b.x, b.y, r); o.w = __funnelshift_r(b.y, b.z, r);
      break;
    default:
      o.x = __funnelshift_r(a.w, b.x, r); o.y = __funnelshift_r(b.x, b.y, r);
      o.z = __funnelshift_r(b.y, b.z, r); o.w = __funnelshift_r(b.z, b.w, r);
      break;
  }
  return o;
}

__device__ __forceinline__ uint4 shfl_down_v4(const uint4& v) {
  uint4 r;
  r.x = __shfl_down_sync(0xffffffffu, v.x, 1);
  r.y = __shfl_down_sync(0xffffffffu, v.y, 1);
  r.z = __shfl_down_sync(0xffffffffu, v.z, 1);
  r.w = __shfl_down_sync(0xffffffffu, v.w, 1);
  return r;
}

// Copies tile bytes [t0, t1) byte by byte (tiles straddling segments, tail).
__device__ inline void copy_tile_bytes(const Segment* segs, int n_segs, uint64_t t0, uint64_t t1,
                                       const Dsts& d) {
  int s = find_segment(segs, n_segs, t0 + threadIdx.x < t1 ? t0 + threadIdx.x : t0);
  for (uint64_t pos = t0 + threadIdx.x; pos < t1; pos += kThreads) {
    while (s + 1 < n_segs && segs[s + 1].dst <= pos) ++s;
    const uint8_t b = segs[s].src[pos - segs[s].dst];
#pragma unroll
    for (int r = 0; r < kMaxDst; ++r)
      if (r < d.n) d.p[r][pos] = b;
  }
}

#ifdef MLCK_DEFINE_KERNELS
// Tiles [first_tile, ...) of the record up to byte `total` (a piece of it
// when the record is packed in pieces).
__global__ void __launch_bounds__(kThreads) pack_kernel(const Segment* __restrict__ segs, int n_segs,
                                                        uint64_t total, Dsts d, uint64_t first_tile) {
  const uint64_t t0 = (first_tile + blockIdx.x) * kTile;
  if (t0 >= total) return;
  const uint64_t t1 = t0 + kTile < total ? t0 + kTile : total;
  const int s = find_segment(segs, n_segs, t0);
  const Segment seg = segs[s];
  if (t1 - t0 != kTile || seg.dst + seg.len < t1) {
    copy_tile_bytes(segs, n_segs, t0, t1, d);
    return;
  }
  const uint8_t* src = seg.src + (t0 - seg.dst);
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src) & 15u);
  const uint8_t* base = src - sh;
  const int lane = threadIdx.x & 31;
  uint4 a[kVecPerThread];
#pragma unroll
  for (int q = 0; q < kVecPerThread; ++q)
    a[q] = ld_stream(base + 16 * (q * kThreads + threadIdx.x));
  if (sh == 0) {
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q) {
      const uint64_t off = t0 + 16 * (q * kThreads + threadIdx.x);
#pragma unroll
      for (int r = 0; r < kMaxDst; ++r)
        if (r < d.n) st_v4(d.p[r] + off, a[q]);
    }
    return;
  }
  uint4 tail[kVecPerThread];
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < kVecPerThread; ++q)
      tail[q] = ld_stream(base + 16 * (q * kThreads + threadIdx.x + 1));
  }
#pragma unroll
  for (int q = 0; q < kVecPerThread; ++q) {
    uint4 b = shfl_down_v4(a[q]);
    if (lane == 31) b = tail[q];
    const uint4 o = funnel16(a[q], b, sh);
    const uint64_t off = t0 + 16 * (q * kThreads + threadIdx.x);
#pragma unroll
    for (int r = 0; r < kMaxDst; ++r)
      if (r < d.n) st_v4(d.p[r] + off, o);
  }
}
#endif  // MLCK_DEFINE_KERNELS

}  // namespace pack
}  // namespace mlck
