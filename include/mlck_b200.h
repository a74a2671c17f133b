/*
 * mlck_b200.h -- C ABI of the B200-native MoEtion checkpoint data path.
 *
 * The reference (/root/reference/proj/include/moelab) is a header-only C++20
 * API.  This ABI is what a drop-in replacement of its checkpoint path binds:
 * plain pointers and sizes, opaque handles, int status + thread-local message.
 * include/moelab_b200/checkpoint.hpp wraps it back into the reference's C++ signatures
 * (same names, same exception types and texts); INTEGRATION.md shows the
 * binding.  Every entry below cites the reference function it replaces.
 *
 * Status codes: 0 ok; 1 = the reference would throw std::invalid_argument;
 * 2 = std::runtime_error (integrity / state errors); 3 = CUDA failure.
 * mlck_last_error() returns the message of the last failing call on this
 * thread, with the reference's exception text where one exists.
 *
 * Threading: one host thread per mlck_ctx; calls on one ctx are ordered on
 * its stream.  Contexts on different devices are independent.
 */
#ifndef MLCK_B200_H
#define MLCK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLCK_OK 0
#define MLCK_EINVAL 1
#define MLCK_ERUNTIME 2
#define MLCK_ECUDA 3

typedef struct mlck_ctx mlck_ctx;
typedef struct mlck_state mlck_state;
typedef struct mlck_blob mlck_blob;
typedef struct mlck_gradlog mlck_gradlog;
typedef struct mlck_log mlck_log;

/* OptimizerConfig (engine.hpp:21-28). kind 0 = Adam, 1 = SGD. */
typedef struct {
  int32_t kind;
  float lr, beta1, beta2, eps;
} mlck_optimizer;

/* Header fields of an MLCK record (snapshot.hpp:61-70). */
typedef struct {
  uint8_t kind;
  uint64_t iteration;
  uint64_t window_start;
  uint32_t wsparse;
  uint32_t slot;
  uint64_t data_seed;
  uint32_t op_count;
} mlck_record_info;

/* One decoded entry (ParsedRecord entries, snapshot.hpp:182-195); payloads
 * stay on the device at payload_offset inside the blob. */
typedef struct {
  uint32_t id;
  uint8_t mode; /* 0 Full, 1 ComputeOnly */
  uint64_t param_count;
  uint64_t step;
  uint64_t payload_offset;
} mlck_entry_info;

/* ---- errors / context -------------------------------------------------- */
const char* mlck_last_error(void);
int mlck_ctx_create(int device, mlck_ctx** out);
/* Destroy a context's blobs, states, gradient logs and upstream logs first:
 * their handles refer to it. */
int mlck_ctx_destroy(mlck_ctx* ctx);
/* Launch all work of this ctx on `stream` (a cudaStream_t; NULL = the
 * context's own non-blocking stream). */
int mlck_ctx_set_stream(mlck_ctx* ctx, void* stream);
int mlck_ctx_synchronize(mlck_ctx* ctx);
/* Number of kernels this ctx launched so far (bench gpu_launches). */
uint64_t mlck_ctx_kernel_launches(mlck_ctx* ctx);
/* Per-kernel timing with CUDA events on the launch stream (pack, fnv,
 * fnv_verify, walk, replay).  mlck_ctx_timings synchronizes, returns the
 * labels as CSV and the durations (ms) recorded since the last read. */
int mlck_ctx_set_timing(mlck_ctx* ctx, int on);
/* Snapshot transport.  -1 (default) auto: 2 when every replica is in this
 * GPU's HBM, else 1.  2: one fused kernel -- the FNV kernel loads the
 * record's chunks straight from their sources (the state arena, the codes;
 * TMA, shifted windows), hashes them and stores them to the blob and every
 * replica by TMA (chunks that straddle segments are pre-gathered; a record
 * whose payload spans more than 5 allocations, or is mostly straddling
 * chunks, takes transport 0).  1: pack kernel, then copy engines push the
 * record while the FNV kernel hashes it.  5: pack kernel, then the FNV
 * kernel stores the replicas from the bytes it stages (no second read).
 * 3: pack kernel, then a push kernel on reserved SMs stores the record to
 * the replicas while the FNV kernel hashes it on the other SMs.  0: the pack
 * kernel stores the replicas, then the FNV kernel.  4: copy engines after
 * the hash (no overlap). */
int mlck_ctx_set_replica_mode(mlck_ctx* ctx, int mode);
/* SMs the hash kernel leaves to co-scheduled work (training kernels beside
 * a snapshot); 0 = all SMs.  The kernel hands chunks out by ticket, so any
 * grid is correct -- this only trades hash throughput for room. */
int mlck_ctx_set_hash_reserve(mlck_ctx* ctx, int sms);
/* Asynchronous trailer hash (default off): with replicas in this GPU's HBM
 * (transport 0) the FNV kernel of a record runs on a side stream after its
 * pack, so the next snapshot's pack (another blob) starts without waiting
 * for it -- the hash leaves the snapshot's critical path.
 * Every reader of a record (parse, conversion, to_host, save, replication,
 * the next snapshot into the same blob) waits for its hash; synchronize,
 * event_record and the memcpy / memset helpers join all pending hashes. */
int mlck_ctx_set_hash_async(mlck_ctx* ctx, int on);
/* Conversion / localized recovery of witnessed records: verify them on
 * `witness_sms` SMs while the replay runs on the rest (0 = verify first,
 * then replay; the default).  Errors keep the reference's order either way;
 * on an error `out`'s operator arrays are unspecified. */
int mlck_ctx_set_convert_overlap(mlck_ctx* ctx, int witness_sms);
/* Witnessed verification (default on).  A record the hash kernel writes
 * keeps, beside its blob, the low byte of the FNV state at every 32-byte
 * segment start (3 % of the record).  parse_record / check_coverage /
 * conversion re-hash such a record without the look-back rounds: each row
 * runs the automaton from its witnessed starts and each segment's end state
 * must equal the next witnessed start -- if all do, the starts are the true
 * ones and the sum is exactly FNV-1a-64 of the bytes in memory; if one does
 * not (stale witness, changed bytes) the record is re-hashed from scratch.
 * The result is the exact checksum either way, and the witness is not part
 * of the record (the MLCK wire format is unchanged).  Records from files,
 * host bytes or peers have no witness.  used / fallbacks count witnessed verifications
 * and those that fell back. */
int mlck_ctx_set_witness(mlck_ctx* ctx, int on);
int mlck_ctx_witness_stats(mlck_ctx* ctx, uint64_t* used, uint64_t* fallbacks);
int mlck_ctx_timings(mlck_ctx* ctx, char* labels_csv, uint64_t labels_cap, float* ms,
                     uint32_t cap, uint32_t* n);

/* ---- device state arena: TrainState / OperatorState (engine.hpp:33-51) -- */
/* Each operator's master|m|v is one contiguous 12P-byte span (the Full
 * payload body); compute weights are kept in their wire encoding (fp16 bits,
 * 1-byte E4M3-240 codes or fp32) -- OperatorState::compute is the decoded
 * image of exactly these codes. */
int mlck_state_create(mlck_ctx* ctx, uint32_t n_ops, const uint64_t* param_counts,
                      int compute_bytes, mlck_state** out);
int mlck_state_destroy(mlck_state* st);
int mlck_state_set_meta(mlck_state* st, uint64_t iteration, uint64_t data_seed);
int mlck_state_get_meta(mlck_state* st, uint64_t* iteration, uint64_t* data_seed);
/* Host arrays in; compute = quantize(master) on the device
 * (OperatorState::refresh_compute, engine.hpp:41-44). */
int mlck_state_upload_op(mlck_state* st, uint32_t id, const float* master, const float* m,
                         const float* v, uint64_t step, int has_full_state);
/* Host arrays out (any pointer may be NULL); compute decoded to float. */
int mlck_state_download_op(mlck_state* st, uint32_t id, float* master, float* m, float* v,
                           uint64_t* step, float* compute, int* has_full_state);
int mlck_state_set_step(mlck_state* st, uint32_t id, uint64_t step, int has_full_state);
/* Device pointers of an operator (compute: its code array). */
int mlck_state_op_ptrs(mlck_state* st, uint32_t id, float** master, float** m, float** v,
                       void** compute);
/* Counter-based synthetic state (benchmark inputs; oracle mlo_synth_value):
 * master U(-.25,.25), m U(-1e-3,1e-3), v U(0,1e-6), step = `step`. */
int mlck_state_fill_synthetic(mlck_state* st, uint64_t seed, uint64_t step);
/* Engine::serialize_state "MLST" (engine.hpp:246-261): size query with
 * host_out = NULL; else packs on the device and copies to host_out. */
int mlck_state_serialize(mlck_state* st, uint8_t* host_out, uint64_t cap, uint64_t* size);
/* Same bytes into a device blob. */
int mlck_state_serialize_blob(mlck_state* st, mlck_blob* out);

/* ---- device blobs (SparseCheckpoint::blobs element, snapshot.hpp:304) --- */
int mlck_blob_create(mlck_ctx* ctx, uint64_t capacity, mlck_blob** out);
int mlck_blob_destroy(mlck_blob* b);
int mlck_blob_from_host(mlck_ctx* ctx, const uint8_t* bytes, uint64_t n, mlck_blob** out);
uint64_t mlck_blob_size(const mlck_blob* b);
void* mlck_blob_device_ptr(const mlck_blob* b);
/* Device pointer of the blob's witness (u32 per 128-byte row of the body),
 * NULL when it has none for its current record. */
void* mlck_blob_witness_ptr(const mlck_blob* b);
int mlck_blob_to_host(const mlck_blob* b, uint8_t* host, uint64_t cap);
/* Replica targets written by the same pack kernel as the local copy: a
 * device pointer of >= capacity bytes (local HBM, or a peer buffer opened
 * with mlck_ipc_open / peer access).  Up to 3 replicas. */
int mlck_blob_add_replica(mlck_blob* b, void* device_ptr, uint64_t capacity);
int mlck_blob_clear_replicas(mlck_blob* b);
/* A witness buffer beside a replica (same device as the replica, e.g. the
 * peer's HBM through CUDA IPC): after each record's hash its witness (one u32
 * per 128-byte row, ~3.1 % of the record) is copied there, behind the record
 * (it is part of mlck_blob_replication's completion).  `capacity` must be at
 * least mlck_witness_bytes(record size); cleared by mlck_blob_clear_replicas.
 * A node recovering from that replica wraps the record and the witness
 * (mlck_blob_wrap), so parse / conversion / localized recovery verify it on
 * the witnessed path instead of re-hashing from scratch -- still exact: a
 * witness that does not match the bytes only costs the from-scratch hash. */
int mlck_blob_add_replica_witness(mlck_blob* b, void* device_ptr, uint64_t capacity);
/* Bytes a witness buffer needs for a record of `record_bytes` (the witness
 * plus the verifier's bulk over-read). */
uint64_t mlck_witness_bytes(uint64_t record_bytes);
/* A read-only blob over `n` record bytes the caller owns in device memory (a
 * replica buffer), with the record's witness if `witness` is not null; no
 * copy.  Parse, coverage, conversion and localized recovery read it in place;
 * snapshots into it are refused.  Destroying it frees nothing of the caller's.
 * The witness buffer must span mlck_witness_bytes(n) bytes; a record or
 * witness running past the allocation it points into is refused. */
int mlck_blob_wrap(mlck_ctx* ctx, void* record, uint64_t n, const void* witness, mlck_blob** out);

/* ---- window lifecycle and durability (SparseCheckpoint::replication /
 * persisted(), snapshot.hpp:300-320; "one persisted + one
 * in-flight") -------------------------------------------------------------
 * Replication of the blob's last record without blocking: *done = the
 * number of replicas holding the complete record (trailer included), 0 while
 * its push is in flight or before any record was written. */
int mlck_blob_replication(mlck_blob* b, uint32_t* done);
/* Persist the record bytes -- the MLCK v1 wire format, i.e. the reference's
 * SparseCheckpoint::blobs element -- to a file (D2H in pinned 64 MiB pieces
 * overlapped with the writes, then fsync).  Errors: "persist: ..." (2). */
int mlck_blob_save(mlck_blob* b, const char* path, uint64_t* written);
/* Read a record file into a new device blob (unparsed: parse_record and the
 * conversion verify it). */
int mlck_blob_load(mlck_ctx* ctx, const char* path, mlck_blob** out);

/* ---- K1+K2: snapshot pack ----------------------------------------------
 * serialize_record(take_sparse_snapshot(engine, slot, slot_index), plan,
 * kind, window_start, wsparse)  (snapshot.hpp:204-241 + 115-144):
 * validates the slot ("snapshot slot references unknown operator N",
 * "snapshot: operator N in active set has no full state"), orders entries by
 * id, packs the byte-exact MLCK record (+ FNV-1a-64 trailer) into `out` and
 * every replica of `out`. */
int mlck_snapshot_record(mlck_state* st, const uint32_t* active, uint32_t n_active,
                         const uint32_t* compute_only, uint32_t n_compute_only,
                         uint32_t slot_index, uint8_t kind, uint64_t window_start,
                         uint32_t wsparse, mlck_blob* out);
/* The same call with the record delivered to host memory (the reference's
 * std::vector<uint8_t> return): device pack + one D2H copy. */
int mlck_snapshot_record_host(mlck_state* st, const uint32_t* active, uint32_t n_active,
                              const uint32_t* compute_only, uint32_t n_compute_only,
                              uint32_t slot_index, uint8_t kind, uint64_t window_start,
                              uint32_t wsparse, mlck_blob* scratch, uint8_t* host_out,
                              uint64_t cap, uint64_t* size);
/* take_dense_checkpoint(engine).serialize(plan) (snapshot.hpp:245-295):
 * "dense checkpoint: operator N is frozen" when an op lacks full state. */
int mlck_dense_checkpoint(mlck_state* st, mlck_blob* out);

/* Self-check of the conversion replay's exact-IEEE fast paths: n_div random
 * divisions inside their range and every float32 inside the sqrt range,
 * each against __fdiv_rn / __fsqrt_rn.  mismatches[0] = division,
 * mismatches[1] = square root (both must be 0). */
int mlck_fastmath_check(mlck_ctx* ctx, uint64_t n_div, uint64_t seed, uint64_t* mismatches);
/* fnv1a64 (digest.hpp:18-25) over n device bytes. */
int mlck_fnv1a64(mlck_ctx* ctx, const void* device_ptr, uint64_t n, uint64_t seed, uint64_t* out);

/* ---- parse / coverage ----------------------------------------------------
 * parse_record (snapshot.hpp:153-197): verifies the trailer on the device
 * ("container checksum mismatch"), then magic/version ("container: bad
 * magic", "container: unsupported version N"), walks the entry table
 * ("container truncated").  Entry metadata out; payloads stay on device. */
int mlck_parse_record(mlck_blob* b, int compute_bytes, mlck_record_info* info,
                      mlck_entry_info* entries, uint32_t cap, uint32_t* n_entries);
/* Decode one entry's payload to host floats (read_compute, snapshot.hpp:95-111). */
int mlck_read_entry(mlck_blob* b, const mlck_entry_info* e, int compute_bytes, float* master,
                    float* m, float* v, float* compute);
/* SparseCheckpoint::check_coverage (snapshot.hpp:322-334). */
int mlck_check_coverage(mlck_blob* const* blobs, uint32_t n_blobs, uint64_t op_count,
                        int compute_bytes);
/* conversion_plan (recovery.hpp:123-137): parse_record of every record (raw
 * parse errors, as the reference: no slot wrapping) and, per record k, the
 * ids of its Full entries in entry order -- step k's `activating`
 * (record_index = k, replay_iteration = window_start + k + 1 follow from k).
 * counts[k] = number of ids of record k; ids concatenated in record order
 * into `activating` (cap entries; *total = the number needed). */
int mlck_conversion_plan(mlck_blob* const* blobs, uint32_t n_blobs, int compute_bytes,
                         uint32_t* activating, uint64_t cap, uint64_t* counts, uint64_t* total);

/* ---- gradient log (inputs of Adam replay) --------------------------------
 * Per-iteration, per-operator fp32 gradients, device resident.  The reference
 * re-derives them by re-running the toy model (engine.hpp:214-222); the GPU
 * path logs them once and replays Adam from the log (bit-identical, SURVEY.md
 * 8(c)).  Iterations are absolute; capacity counts iterations kept. */
int mlck_gradlog_create(mlck_ctx* ctx, uint32_t n_ops, const uint64_t* param_counts,
                        uint32_t capacity_iterations, mlck_gradlog** out);
int mlck_gradlog_destroy(mlck_gradlog* g);
/* Host floats in (P of the op). */
int mlck_gradlog_put(mlck_gradlog* g, uint64_t iteration, uint32_t op_id, const float* host);
/* Device pointer of the slot for (iteration, op) -- allocates the slot. */
int mlck_gradlog_slot(mlck_gradlog* g, uint64_t iteration, uint32_t op_id, float** device_ptr);
int mlck_gradlog_fill_synthetic(mlck_gradlog* g, uint64_t first_iteration, uint32_t n_iterations,
                                uint64_t seed);
/* Capture of a trainer-owned device gradient into the log: a copy on the
 * ctx stream, ordered after the trainer's work queued there (the zero-copy
 * alternative: the trainer's backward writes into mlck_gradlog_slot). */
int mlck_gradlog_capture(mlck_gradlog* g, uint64_t iteration, uint32_t op_id, const float* device_src);
/* Device bytes the log holds (capacity_iterations x sum of the ops' slots). */
uint64_t mlck_gradlog_bytes(const mlck_gradlog* g);

/* ---- Adam ----------------------------------------------------------------
 * optimizer_step_adam (engine.hpp:738-753) on device arrays; *step is the
 * host-side counter (incremented before the bias corrections, as the
 * reference does). */
int mlck_optimizer_step_adam(mlck_ctx* ctx, float* master, float* m, float* v, uint64_t* step,
                             const float* grad, uint64_t n, const mlck_optimizer* opt);
/* Engine::apply_updates (engine.hpp:699-728) for the listed operators with
 * the gradients of `iteration` from `g`: Adam or SGD, then refresh_compute. */
int mlck_state_apply_updates(mlck_state* st, const uint32_t* ids, uint32_t n_ids,
                             mlck_gradlog* g, uint64_t iteration, const mlck_optimizer* opt);

/* ---- K3: sparse-to-dense conversion --------------------------------------
 * sparse_to_dense_convert (recovery.hpp:180-227) with Adam replay from the
 * gradient log: verifies every record (FNV trailer), takes each operator's
 * unique Full payload (slot k) and applies W-k optimizer steps from the
 * gradients of iterations window_start+k+1 .. window_start+W in one fused
 * pass, writing master/m/v + compute codes into `out` (sized like the model)
 * and setting its iteration (window_start+W; the record's for W == 1) and
 * data_seed.  Errors: "sparse checkpoint incomplete: n of W records",
 * "sparse checkpoint record (slot k): <parse error>",
 * "conversion finished with frozen operator N". */
int mlck_sparse_to_dense_convert(mlck_state* out, mlck_blob* const* blobs, uint32_t n_blobs,
                                 uint64_t window_start, uint32_t wsparse, uint64_t data_seed,
                                 mlck_gradlog* g, const mlck_optimizer* opt);

/* localized_recover(engine, RecoverySegment, ckpt, logs, target)
 * (recovery.hpp:240-244) with the scope given as the reference does: the
 * segment's stage range [stage_lo, stage_hi] and Engine::stage_of_op for
 * every operator (stage_of_op[id], n_ops entries).  Before replaying it
 * checks, like run_scoped (engine.hpp:361-366, 393-400), that `log` holds
 * every boundary tensor the segment consumes for iterations a+1 .. target:
 * (it, gmb, stage_lo-1, fwd) when stage_lo > 0 and (it, gmb, stage_hi, bwd)
 * when stage_hi < n_stages-1, gmb < n_global_microbatches (dp x M) --
 * "upstream log missing entry: ..." otherwise (log may be NULL only when
 * the segment spans every stage).  Then as mlck_localized_recover. */
int mlck_localized_recover_segment(mlck_state* out, int32_t stage_lo, int32_t stage_hi,
                                   const int32_t* stage_of_op, int32_t n_stages,
                                   mlck_blob* const* blobs, uint32_t n_blobs, uint64_t window_start,
                                   uint32_t wsparse, uint64_t data_seed, mlck_log* log,
                                   uint32_t n_global_microbatches, mlck_gradlog* g,
                                   uint64_t target_iteration, const mlck_optimizer* opt);

/* localized_recover (recovery.hpp:240-289): conversion restricted to the
 * operators `scope_ids` (the failed stages' operators, Engine::stage_of_op),
 * then the lost iterations after the window up to target_iteration; every
 * in-scope operator replays iterations a+k+1 .. max(a+W, target) from the
 * gradient log.  Only in-scope operators of `out` are written.  Errors as
 * the reference: "sparse checkpoint incomplete", "sparse checkpoint record
 * (slot k): ...", "localized recovery left operator N frozen". */
int mlck_localized_recover(mlck_state* out, const uint32_t* scope_ids, uint32_t n_scope,
                           mlck_blob* const* blobs, uint32_t n_blobs, uint64_t window_start,
                           uint32_t wsparse, uint64_t data_seed, mlck_gradlog* g,
                           uint64_t target_iteration, const mlck_optimizer* opt);

/* ---- the miniature MoE trainer on the GPU (moelab::Engine, engine.hpp:
 * 150-730): the recompute half of conversion / recovery and
 * a GPU producer of the boundary log and of the weight-gradient log. ------
 * EngineConfig's model / parallel / optimizer / precision fields
 * (engine.hpp:96-124, core.hpp:66-191); params < 0 = derived from the toy
 * dimensions.  Operator ids as ModelSpec::operators (layer-major, E experts,
 * NE, gate).  A state (mlck_state) of the engine's param_counts holds the
 * operators; its data_seed is the data stream's seed. */
typedef struct mlck_engine mlck_engine;
typedef struct {
  int32_t layers, experts_per_layer, top_k, shared_experts;
  int32_t token_dim, expert_hidden, nonexpert_hidden, residual;
  int64_t expert_params, nonexpert_params, gate_params;
  int32_t pp_stages, dp_degree, microbatches, compute_bytes;
  int64_t microbatch_size;
  mlck_optimizer optimizer;
} mlck_engine_config;
int mlck_engine_create(mlck_ctx* ctx, const mlck_engine_config* cfg, mlck_engine** out);
int mlck_engine_destroy(mlck_engine* e);
uint32_t mlck_engine_op_count(const mlck_engine* e);
int mlck_engine_param_counts(const mlck_engine* e, uint64_t* out);
int32_t mlck_engine_stage_of_op(const mlck_engine* e, uint32_t id);
/* Engine::run_iteration(modes, log) (engine.hpp:189-207) on `st`:
 * forward + backward of every micro-batch, Adam / SGD on the active
 * operators, st's iteration + 1.  frozen: n_ops flags (NULL = all active).
 * log_out (may be NULL): the sender-side boundary copies of the iteration.
 * grads_out (may be NULL): the active operators' weight gradients land in
 * its slots of the new iteration -- the zero-copy capture the logged-
 * gradient conversion replays. */
int mlck_engine_run_iteration(mlck_engine* e, mlck_state* st, const uint8_t* frozen, mlck_log* log_out,
                              mlck_gradlog* grads_out);
/* Engine::replay_scoped_iteration (engine.hpp:214-222): stages
 * [stage_lo, stage_hi] of `ops` at `iteration`, boundary inputs from log_in
 * ("upstream log missing entry: ..."), updates of the active in-scope ops. */
int mlck_engine_replay_scoped_iteration(mlck_engine* e, mlck_state* ops, uint64_t iteration, int32_t stage_lo,
                                        int32_t stage_hi, const uint8_t* frozen, mlck_log* log_in);
/* sparse_to_dense_convert (recovery.hpp:180-227) with the reference's own
 * replay: each window iteration re-run forward + backward, frozen operators
 * without weight gradients.  Errors as mlck_sparse_to_dense_convert. */
int mlck_sparse_to_dense_convert_recompute(mlck_engine* e, mlck_state* out, mlck_blob* const* blobs,
                                           uint32_t n_blobs, uint64_t window_start, uint32_t wsparse,
                                           uint64_t data_seed);
/* localized_recover(engine, RecoverySegment{stage_lo, stage_hi}, ckpt,
 * logs, target) (recovery.hpp:240-289) by recompute: only the segment's
 * stages run, boundary tensors from `logs`; in-scope operators of `out`. */
int mlck_localized_recover_recompute(mlck_engine* e, mlck_state* out, int32_t stage_lo, int32_t stage_hi,
                                     mlck_blob* const* blobs, uint32_t n_blobs, uint64_t window_start,
                                     uint32_t wsparse, uint64_t data_seed, mlck_log* logs,
                                     uint64_t target_iteration);

/* ---- K4: upstream boundary log (LogKey/UpstreamLog, engine.hpp:55-94) ----
 * kind 0: pinned host ring (copy engine, side stream); kind 1: device ring
 * on `device` (peer HBM over NVLink when device != ctx device). */
int mlck_log_create(mlck_ctx* ctx, int kind, int device, uint64_t capacity_bytes,
                    mlck_log** out);
/* kind 2: a ring on caller-owned device memory (e.g. a peer GPU's buffer
 * opened with mlck_ipc_open: the pipeline successor's HBM); not freed by
 * mlck_log_destroy. */
int mlck_log_create_external(mlck_ctx* ctx, void* device_base, uint64_t capacity_bytes,
                             mlck_log** out);
int mlck_log_destroy(mlck_log* l);
/* Records the sender-side copy of a boundary tensor (engine.hpp:383-385,
 * 407-409); src is device memory produced on the ctx stream. Overwrites an
 * existing key like the reference's map assignment.
 * Source lifetime: the copy runs on the log's low-priority side stream once
 * the ctx stream's work so far is done.  In the default ORDERED mode the ctx
 * stream then waits for the copy, so any later work on the ctx stream may
 * overwrite src -- the reference's synchronous copy, seen from the stream.
 * In ASYNC mode (mlck_log_set_async(l, 1)) nothing waits: src must stay
 * unmodified until mlck_log_fence() has ordered the writer's stream after
 * the copies (or mlck_log_sync() returned). */
int mlck_log_put(mlck_log* l, uint64_t iteration, uint32_t micro_batch, uint32_t boundary,
                 uint8_t direction, const float* device_src, uint64_t n_floats);
int mlck_log_set_async(mlck_log* l, int async);
/* Makes `stream` (a cudaStream_t; NULL = the ctx stream) wait for every
 * copy put() issued so far, without blocking the host. */
int mlck_log_fence(mlck_log* l, void* stream);
/* UpstreamLog::at (engine.hpp:71-79): "upstream log missing entry: ..." */
int mlck_log_get(mlck_log* l, uint64_t iteration, uint32_t micro_batch, uint32_t boundary,
                 uint8_t direction, float* host_out, uint64_t cap_floats, uint64_t* n_floats);
/* Device-side copy of an entry into dst (replay input), ordered on the ctx
 * stream after the work queued there (no host synchronization). */
int mlck_log_get_device(mlck_log* l, uint64_t iteration, uint32_t micro_batch, uint32_t boundary,
                        uint8_t direction, float* device_dst, uint64_t cap_floats,
                        uint64_t* n_floats);
uint64_t mlck_log_count(mlck_log* l);
uint64_t mlck_log_bytes(mlck_log* l);
/* i-th entry in LogKey order (std::map order of the reference). */
int mlck_log_entry(mlck_log* l, uint64_t index, uint64_t* iteration, uint32_t* micro_batch,
                   uint32_t* boundary, uint8_t* direction, float* host_out, uint64_t cap_floats,
                   uint64_t* n_floats);
/* gc_logs (engine.hpp:90-94): drop iteration < persisted_window_start. */
int mlck_gc_logs(mlck_log* l, uint64_t persisted_window_start);
/* upstream_log_bytes(model, plan, wsparse) (recovery.hpp:296-304): the
 * retained worst case, 2 windows x W x 2(S-1)M dp entries of mb x d floats. */
int64_t mlck_upstream_log_bytes(int32_t token_dim, int32_t pp_stages, int32_t microbatches,
                                int64_t microbatch_size, int32_t dp_degree, int64_t wsparse);
/* check_log_budget(model, plan, wsparse, cluster) (recovery.hpp:308-317):
 * MLCK_EINVAL with "upstream log budget exceeded: need N bytes of host
 * memory, budget B" when cpu_mem_per_node * nodes cannot hold it (a budget
 * <= 0 is unchecked). */
int mlck_check_log_budget(int32_t token_dim, int32_t pp_stages, int32_t microbatches,
                          int64_t microbatch_size, int32_t dp_degree, int64_t wsparse,
                          double cpu_mem_per_node, int32_t nodes);
/* Wait until every put() has landed. */
int mlck_log_sync(mlck_log* l);

/* ---- codecs (tensor.hpp:99-183), on device --------------------------------
 * Generic reduced formats: pack_reduced(x, ebits, mbits) / unpack_reduced
 * (tensor.hpp:127-183) over n device values (codes are uint16), 2 <= ebits <= 8,
 * 1 <= mbits, ebits + mbits <= 15. */
int mlck_pack_reduced(mlck_ctx* ctx, const float* device_in, uint16_t* device_codes, uint64_t n,
                      int ebits, int mbits);
int mlck_unpack_reduced(mlck_ctx* ctx, const uint16_t* device_codes, float* device_out, uint64_t n,
                        int ebits, int mbits);
/* The reference's scalar forms quantize_value (tensor.hpp:99-111),
 * pack_reduced, unpack_reduced: n host values through the device kernels
 * (the scalar API of the shim is n = 1). */
int mlck_quantize_values(mlck_ctx* ctx, const float* host_in, float* host_out, uint64_t n,
                         int compute_bytes);
int mlck_pack_reduced_values(mlck_ctx* ctx, const float* host_in, uint16_t* host_codes, uint64_t n,
                             int ebits, int mbits);
int mlck_unpack_reduced_values(mlck_ctx* ctx, const uint16_t* host_codes, float* host_out, uint64_t n,
                               int ebits, int mbits);
int mlck_quantize(mlck_ctx* ctx, const float* device_in, float* device_out, uint64_t n,
                  int compute_bytes);
int mlck_encode_compute(mlck_ctx* ctx, const float* device_in, void* device_codes, uint64_t n,
                        int compute_bytes);
int mlck_decode_compute(mlck_ctx* ctx, const void* device_codes, float* device_out, uint64_t n,
                        int compute_bytes);

/* ---- multi-GPU replica placement (CUDA IPC over NVLink) ------------------ */
int mlck_ipc_export(mlck_ctx* ctx, void* device_ptr, uint8_t handle[64]);
int mlck_ipc_open(mlck_ctx* ctx, const uint8_t handle[64], void** device_ptr);
/* Closes a mapping mlck_ipc_open returned; pending snapshots finish first,
 * and every blob of the ctx drops the replicas registered inside it. */
int mlck_ipc_close(mlck_ctx* ctx, void* device_ptr);
int mlck_enable_peer_access(mlck_ctx* ctx, int peer_device);

/* ---- timing helpers for the benchmark (events on the ctx stream) --------- */
int mlck_event_record(mlck_ctx* ctx, int slot);
int mlck_event_elapsed_ms(mlck_ctx* ctx, int slot_a, int slot_b, float* ms);
/* Raw device allocation helpers (L2 flush buffer, synthetic inputs). */
int mlck_device_alloc(mlck_ctx* ctx, uint64_t bytes, void** ptr);
int mlck_device_free(mlck_ctx* ctx, void* ptr);
int mlck_device_memset(mlck_ctx* ctx, void* ptr, int value, uint64_t bytes);
int mlck_host_alloc_pinned(mlck_ctx* ctx, uint64_t bytes, void** ptr);
int mlck_host_free_pinned(mlck_ctx* ctx, void* ptr);
int mlck_memcpy_h2d(mlck_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int mlck_memcpy_d2h(mlck_ctx* ctx, void* dst, const void* src, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
