// kernels.cu -- sm_100a kernels of the checkpoint data path and their
// host-side launchers (declared in kernels.cuh).
#define MLCK_DEFINE_KERNELS 1
#include "adam.cuh"
#include "codec.cuh"
#include "fnv.cuh"
#include "kernels.cuh"
#include "pack.cuh"

#include <algorithm>

namespace mlck {

// ---------------------------------------------------------------- FNV (K2)
namespace {

// K1 fused into K2: the thread's 64 output bytes gathered from the record's
// segment table (header bytes + arena spans at arbitrary alignment) with
// aligned 128-bit loads and a funnel shift, written to the local record and
// every replica (peer pointers: NVLink stores), then hashed from registers'
// worth of data the thread just wrote.
__device__ __forceinline__ void gather_write64(const pack::Segment* __restrict__ segs, int n_segs,
                                               uint64_t pos0, uint64_t n, const pack::Dsts& d) {
  if (pos0 >= n) return;
  const int s = pack::find_segment(segs, n_segs, pos0);
  const pack::Segment seg = segs[s];
  if (pos0 + 64 <= n && seg.dst + seg.len >= pos0 + 64) {
    const uint8_t* src = seg.src + (pos0 - seg.dst);
    const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src) & 15u);
    const uint8_t* base = src - sh;
    uint4 a[5];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = ld_stream(base + 16 * i);
    a[4] = sh ? ld_stream(base + 64) : a[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 o = sh ? pack::funnel16(a[i], a[i + 1], sh) : a[i];
#pragma unroll
      for (int r = 0; r < pack::kMaxDst; ++r)
        if (r < d.n) st_v4(d.p[r] + pos0 + 16 * i, o);
    }
    return;
  }
  int k = s;  // straddles segments (headers) or the record end: byte path
  const uint64_t end = pos0 + 64 < n ? pos0 + 64 : n;
  for (uint64_t p = pos0; p < end; ++p) {
    while (k + 1 < n_segs && segs[k + 1].dst <= p) ++k;
    const uint8_t b = segs[k].src[p - segs[k].dst];
#pragma unroll
    for (int r = 0; r < pack::kMaxDst; ++r)
      if (r < d.n) d.p[r][p] = b;
  }
}

// `data` is not __restrict__: in the fused mode it is the local record the
// same kernel just wrote (no read-only / non-coherent cache path allowed).
__global__ void __launch_bounds__(fnv::kThreads, 65536 / (64 * fnv::kThreads)) fnv_kernel(const uint8_t* data,
                                                             uint64_t n, uint64_t seed,
                                                             fnv::Scratch scr, uint64_t n_chunks,
                                                             TrailerDsts trailer,
                                                             const pack::Segment* __restrict__ segs,
                                                             int n_segs, pack::Dsts dsts) {
  __shared__ fnv::SharedState sh;
  __shared__ int64_t s_chunk;
  // Persistent CTAs take chunks in ticket order, so every predecessor of a
  // chunk is resident or finished when its look-back spins on it.
  while (true) {
    if (threadIdx.x == 0) s_chunk = atomicAdd(scr.ticket, 1u);
    __syncthreads();
    const int64_t chunk = s_chunk;
    if (chunk >= static_cast<int64_t>(n_chunks)) return;
    if (n_segs > 0)  // fused pack: write this thread's bytes, then hash them
      gather_write64(segs, n_segs,
                     static_cast<uint64_t>(chunk) * fnv::kChunk + threadIdx.x * 64ull, n, dsts);
    const bool last = fnv::chunk_contribution(data, chunk, n, seed, scr, n_chunks, sh);
    // the block that finished last also writes the trailer bytes
    // (serialize_record appends the checksum, snapshot.hpp:142)
    if (last) {
      const unsigned long long h = sh.pc;
      for (int r = 0; r < trailer.n; ++r)
        for (int b = 0; b < 8; ++b) trailer.p[r][b] = static_cast<uint8_t>(h >> (8 * b));
    }
    __syncthreads();  // s_chunk is rewritten next iteration
  }
}

}  // namespace

void init_constants() {
  unsigned long long t[fnv::kThreads];
  const uint64_t p64 = fnv::pow_p(64);
  uint64_t x = 1;
  for (int k = 0; k < fnv::kThreads; ++k) {
    t[k] = x;
    x *= p64;
  }
  MLCK_CUDA(cudaMemcpyToSymbol(fnv::c_pow64, t, sizeof(t)));
  uint32_t qlo[fnv::kBytesPerThread], qhi[fnv::kBytesPerThread];
  unsigned long long qsum = 0;
  for (int k = 0; k < fnv::kBytesPerThread; ++k) {
    const uint64_t q = fnv::pow_p(static_cast<uint64_t>(fnv::kBytesPerThread - k));
    qlo[k] = static_cast<uint32_t>(q);
    qhi[k] = static_cast<uint32_t>(q >> 32);
    qsum += q;
  }
  const unsigned long long qbias = 512ull * qsum;
  MLCK_CUDA(cudaMemcpyToSymbol(fnv::c_qlo, qlo, sizeof(qlo)));
  MLCK_CUDA(cudaMemcpyToSymbol(fnv::c_qhi, qhi, sizeof(qhi)));
  MLCK_CUDA(cudaMemcpyToSymbol(fnv::c_qbias, &qbias, sizeof(qbias)));
}

uint64_t fnv_chunks(uint64_t n) { return div_up(n, fnv::kChunk); }
// [256 B header: ticket u32 @0, finished u32 @8, accum u64 @16]
// [status: n_chunks words of 8 B at a 256 B stride]
size_t fnv_scratch_words(uint64_t n) { return (256 + fnv_chunks(n) * fnv::kStatusStride * 8) / 4; }

void launch_fnv(const uint8_t* data, uint64_t n, uint64_t seed, uint32_t* scratch, uint32_t epoch,
                unsigned long long* result, const TrailerDsts& trailer, cudaStream_t stream,
                unsigned long long* prof, unsigned long long* trace, const pack::Segment* segs,
                int n_segs, const pack::Dsts* dsts) {
  const uint64_t n_chunks = fnv_chunks(n);
  fnv::Scratch scr;
  scr.ticket = scratch;
  scr.finished = scratch + 2;
  scr.accum = reinterpret_cast<unsigned long long*>(scratch + 4);
  scr.result = result;
  scr.status = reinterpret_cast<unsigned long long*>(scratch + 64);
  scr.epoch = epoch;
  scr.prof = prof;
  scr.trace = trace;
  MLCK_CUDA(cudaMemsetAsync(scratch, 0, 256, stream));  // header only: status is epoch-tagged
  if (n_chunks == 0) {
    // empty input: h = seed
    launch_fnv_empty(seed, result, trailer, stream);
    return;
  }
  static int resident = 0;  // CTAs per SM at full occupancy
  if (resident == 0) {
    MLCK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, fnv_kernel, fnv::kThreads, 0));
    if (resident < 1) resident = 1;
  }
  int sms = kSmCount;
  {
    int dev = 0;
    MLCK_CUDA(cudaGetDevice(&dev));
    MLCK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const uint64_t grid = std::min<uint64_t>(n_chunks, static_cast<uint64_t>(resident) * sms);
  pack::Dsts d{};
  if (dsts) d = *dsts;
  fnv_kernel<<<static_cast<unsigned>(grid), fnv::kThreads, 0, stream>>>(
      data, n, seed, scr, n_chunks, trailer, segs, segs ? n_segs : 0, d);
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

// ---------------------------------------------------------------- pack (K1)
void launch_pack(const pack::Segment* segs, int n_segs, uint64_t total, const pack::Dsts& d,
                 cudaStream_t stream) {
  if (total == 0) return;
  const uint64_t tiles = div_up(total, pack::kTile);
  pack::pack_kernel<<<static_cast<unsigned>(tiles), pack::kThreads, 0, stream>>>(segs, n_segs,
                                                                                 total, d);
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
void launch_replay(const adam::ConvOp* ops, int n_ops, const float* const* gptr, const float2* bc,
                   const adam::Opt& o, int cb, uint64_t total_units, cudaStream_t stream) {
  if (total_units == 0) return;
  const uint64_t blocks = div_up(total_units, 256);
  adam::replay_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(ops, n_ops, gptr, bc, o,
                                                                         cb, total_units);
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
}  // namespace

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
