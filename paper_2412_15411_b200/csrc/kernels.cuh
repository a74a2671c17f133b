// kernels.cuh -- host launchers for the kernels in kernels.cu.
#pragma once

#include "adam.cuh"
#include "mlck_common.cuh"
#include "pack.cuh"

namespace mlck {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;  // digest.hpp:18

struct TrailerDsts {
  uint8_t* p[pack::kMaxDst];
  int n;
};

// ---- record walk (parse_record after the checksum)
enum WalkStatus : uint32_t { kWalkOk = 0, kWalkTruncated = 1, kWalkMagic = 3, kWalkVersion = 4, kWalkWidth = 5 };
struct WalkEntry {
  uint32_t id;
  uint8_t mode;
  uint64_t param_count;
  uint64_t step;
  uint64_t payload_offset;
};
struct WalkResult {
  uint32_t status, version, op_count, n_entries;
  uint8_t kind;
  uint64_t iteration, window_start, data_seed;
  uint32_t wsparse, slot;
};
struct WalkJob {
  const uint8_t* blob;
  uint64_t n;
  int compute_bytes;
  uint32_t cap;
  WalkEntry* entries;
  WalkResult* result;
};

// Fused snapshot: the FNV kernel loads the record's chunks from its sources
// by TMA (runs: chunks [c0, c1) are rows row0 + 512 (c - c0) ... of source
// `map`, shifted by `delta` bytes; map n_src = the patch buffer of the chunks
// that straddle segments), hashes them and stores them to every copies dst.
struct FnvRun {
  int64_t c0, c1, row0;
  int32_t map, delta;
};
constexpr int kFnvMaxSrc = 6;  // source maps per launch, the patch buffer included
struct FnvFused {
  const FnvRun* runs;  // device, sorted by c0, covering every chunk
  int n_runs;
  const uint8_t* src[kFnvMaxSrc];  // source allocations (16-byte aligned), the patch buffer last
  uint64_t src_bytes[kFnvMaxSrc];
  int n_src;
};
// The straddling chunks of a fused snapshot: chunk chunks[j] of the record
// (bytes from `segs`, zeros past n) to out + j * fnv_chunk_bytes().
void launch_patch_chunks(const pack::Segment* segs, int n_segs, const int64_t* chunks, uint64_t n_patch, uint64_t n,
                         uint8_t* out, cudaStream_t stream);

void init_constants();
uint64_t fnv_chunk_bytes();
uint32_t fnv_sticky_word();  // scratch word of the sticky watchdog flag
uint64_t fnv_chunks(uint64_t n);
size_t fnv_scratch_words(uint64_t n);
void launch_fnv(const uint8_t* data, uint64_t n, uint64_t seed, uint32_t* scratch, uint32_t epoch,
                unsigned long long* result, const TrailerDsts& trailer, cudaStream_t stream,
                unsigned long long* prof = nullptr, unsigned long long* trace = nullptr,
                const FnvFused* fused = nullptr, int reserve_sms = 0,
                const pack::Dsts* copies = nullptr,  // also store the hashed bytes to these (TMA)
                uint32_t* witness = nullptr);        // non-null: the rows' segment starts (fnv.cuh)
// Exact re-hash of n bytes against the witness fnv_kernel left (one u32 per
// 128-byte row); *bad = 1 when the witness does not match the bytes (the
// caller then hashes with launch_fnv).  scratch as launch_fnv's.
void launch_fnv_witness(const uint8_t* data, uint64_t n, uint64_t seed, const uint32_t* witness, uint32_t* scratch,
                        unsigned long long* result, unsigned long long* bad, cudaStream_t stream, int ctas = 0);
inline uint64_t fnv_witness_words(uint64_t n) { return (n + 127) / 128; }
// Copy `bytes` from src to every dst with `ctas` CTAs of one SM each.
void launch_push(const uint8_t* src, uint64_t bytes, const pack::Dsts& d, int ctas, cudaStream_t stream);
void launch_fnv_empty(uint64_t seed, unsigned long long* result, const TrailerDsts& trailer,
                      cudaStream_t stream);
// Packs record bytes [lo, total) (lo a multiple of pack::kTile).
void launch_pack(const pack::Segment* segs, int n_segs, uint64_t total, const pack::Dsts& d,
                 cudaStream_t stream, uint64_t lo = 0);
void launch_walk(const WalkJob* jobs, int n_jobs, cudaStream_t stream);
// (bc: the host's bias corrections per (operator, step); steps: device
// scratch of n_bc StepConst the launch fills first)
void launch_replay(const adam::ConvOp* ops, int n_ops, const float* const* gptr, const float2* bc, uint32_t n_bc,
                   adam::StepConst* steps, const adam::Opt& o, int cb, uint64_t total_units, cudaStream_t stream);
// Threads per replay CTA (launch_replay's total_units counts CTAs: each
// operator's 4-element units round up to whole CTAs).
int replay_unit_elems();  // consecutive elements per replay thread
int replay_cta_threads();
// Self-check of the replay kernel's spelled-out IEEE fast paths (adam.cuh).
void launch_fastmath_check(uint64_t n, uint64_t seed, unsigned long long* counts, cudaStream_t stream);
void launch_adam_arrays(float* w, float* m, float* v, const float* g, uint64_t n,
                        const adam::Opt& o, float bc1, float bc2, cudaStream_t stream);
void launch_quantize(const float* in, float* out, uint64_t n, int cb, cudaStream_t stream);
void launch_encode(const float* in, void* codes, uint64_t n, int cb, cudaStream_t stream);
void launch_decode(const void* codes, float* out, uint64_t n, int cb, cudaStream_t stream);
void launch_pack_reduced(const float* in, uint16_t* codes, uint64_t n, int eb, int mb, cudaStream_t stream);
void launch_unpack_reduced(const uint16_t* codes, float* out, uint64_t n, int eb, int mb, cudaStream_t stream);
uint64_t synth_key(uint64_t seed, uint64_t stream);
void launch_synth(float* out, uint64_t n, uint64_t seed, uint64_t stream_id, float lo, float hi,
                  cudaStream_t stream);
void launch_copy16(void* dst, const void* src, uint64_t bytes, cudaStream_t stream);

}  // namespace mlck
