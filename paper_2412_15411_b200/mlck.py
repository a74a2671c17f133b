"""Python binding of the C ABI (include/mlck_b200.h) -- the host-side mirror
of the reference's moelab checkpoint API used by the tests and bench.py.

The reference is C++ (proj/include/moelab); its drop-in is the C++ shim in
include/moelab_b200/.  This module binds the same ABI with ctypes so pytest
and the benchmark can drive the sm_100a kernels.  It loads ONLY the in-tree
libmlck_b200.so and raises if it is missing: there is no CPU fallback.

Error mapping mirrors the reference: status 1 -> ValueError
(std::invalid_argument), 2/3 -> RuntimeError (std::runtime_error), with the
reference's message text.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MLCK_B200_LIB: a development build variant (scripts/build_variant.sh)
LIB_PATH = os.environ.get("MLCK_B200_LIB") or os.path.join(HERE, "_build", "libmlck_b200.so")

u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u16p = C.POINTER(C.c_uint16)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p


class MlckInvalid(ValueError):
    """std::invalid_argument in the reference."""


class MlckRuntime(RuntimeError):
    """std::runtime_error in the reference (integrity / state errors)."""


class Optimizer(C.Structure):
    """OptimizerConfig (engine.hpp:21-28)."""
    _fields_ = [("kind", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float)]

    @classmethod
    def adam(cls, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        return cls(0, lr, beta1, beta2, eps)

    @classmethod
    def sgd(cls, lr=1e-3):
        return cls(1, lr, 0.9, 0.999, 1e-8)


class EngineConfig(C.Structure):
    """EngineConfig (engine.hpp:96-124; core.hpp:66-191): params < 0 = derived."""
    _fields_ = [("layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("shared_experts", C.c_int32), ("token_dim", C.c_int32), ("expert_hidden", C.c_int32),
                ("nonexpert_hidden", C.c_int32), ("residual", C.c_int32), ("expert_params", C.c_int64),
                ("nonexpert_params", C.c_int64), ("gate_params", C.c_int64), ("pp_stages", C.c_int32),
                ("dp_degree", C.c_int32), ("microbatches", C.c_int32), ("compute_bytes", C.c_int32),
                ("microbatch_size", C.c_int64), ("optimizer", Optimizer)]

    @classmethod
    def from_dict(cls, c: dict) -> "EngineConfig":
        opt = Optimizer(int(c.get("optimizer_kind", 0)), c.get("lr", 1e-3), c.get("beta1", 0.9),
                        c.get("beta2", 0.999), c.get("eps", 1e-8))
        return cls(c["layers"], c["experts_per_layer"], c["top_k"], c.get("shared_experts", 0), c["token_dim"],
                   c["expert_hidden"], c["nonexpert_hidden"], int(c.get("residual", 1)),
                   int(c.get("expert_params", -1)), int(c.get("nonexpert_params", -1)),
                   int(c.get("gate_params", -1)), c["pp_stages"], c["dp_degree"], c["microbatches"],
                   int(c["compute_bytes"]), c["microbatch_size"], opt)


class RecordInfo(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("iteration", C.c_uint64), ("window_start", C.c_uint64),
                ("wsparse", C.c_uint32), ("slot", C.c_uint32), ("data_seed", C.c_uint64),
                ("op_count", C.c_uint32)]


class EntryInfo(C.Structure):
    _fields_ = [("id", C.c_uint32), ("mode", C.c_uint8), ("param_count", C.c_uint64),
                ("step", C.c_uint64), ("payload_offset", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make -C paper_2412_15411_b200` "
                              "(the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        sig = {
            "mlck_last_error": (C.c_char_p, []),
            "mlck_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "mlck_ctx_destroy": (C.c_int, [vp]),
            "mlck_ctx_set_stream": (C.c_int, [vp, vp]),
            "mlck_ctx_synchronize": (C.c_int, [vp]),
            "mlck_ctx_kernel_launches": (C.c_uint64, [vp]),
            "mlck_ctx_set_timing": (C.c_int, [vp, C.c_int]),
            "mlck_log_create_external": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp)]),
            "mlck_ctx_set_replica_mode": (C.c_int, [vp, C.c_int]),
            "mlck_ctx_timings": (C.c_int, [vp, C.c_char_p, C.c_uint64, f32p, C.c_uint32, u32p]),
            "mlck_state_create": (C.c_int, [vp, C.c_uint32, u64p, C.c_int, C.POINTER(vp)]),
            "mlck_state_destroy": (C.c_int, [vp]),
            "mlck_state_set_meta": (C.c_int, [vp, C.c_uint64, C.c_uint64]),
            "mlck_state_get_meta": (C.c_int, [vp, u64p, u64p]),
            "mlck_state_upload_op": (C.c_int, [vp, C.c_uint32, f32p, f32p, f32p, C.c_uint64, C.c_int]),
            "mlck_state_download_op": (C.c_int, [vp, C.c_uint32, f32p, f32p, f32p, u64p, f32p,
                                                 C.POINTER(C.c_int)]),
            "mlck_state_set_step": (C.c_int, [vp, C.c_uint32, C.c_uint64, C.c_int]),
            "mlck_state_op_ptrs": (C.c_int, [vp, C.c_uint32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                             C.POINTER(vp)]),
            "mlck_state_fill_synthetic": (C.c_int, [vp, C.c_uint64, C.c_uint64]),
            "mlck_state_serialize": (C.c_int, [vp, u8p, C.c_uint64, u64p]),
            "mlck_state_serialize_blob": (C.c_int, [vp, vp]),
            "mlck_blob_create": (C.c_int, [vp, C.c_uint64, C.POINTER(vp)]),
            "mlck_blob_destroy": (C.c_int, [vp]),
            "mlck_blob_from_host": (C.c_int, [vp, u8p, C.c_uint64, C.POINTER(vp)]),
            "mlck_blob_size": (C.c_uint64, [vp]),
            "mlck_blob_device_ptr": (vp, [vp]),
            "mlck_blob_to_host": (C.c_int, [vp, u8p, C.c_uint64]),
            "mlck_blob_add_replica": (C.c_int, [vp, vp, C.c_uint64]),
            "mlck_blob_clear_replicas": (C.c_int, [vp]),
            "mlck_blob_add_replica_witness": (C.c_int, [vp, vp, C.c_uint64]),
            "mlck_witness_bytes": (C.c_uint64, [C.c_uint64]),
            "mlck_blob_wrap": (C.c_int, [vp, vp, C.c_uint64, vp, C.POINTER(vp)]),
            "mlck_blob_replication": (C.c_int, [vp, C.POINTER(C.c_uint32)]),
            "mlck_fastmath_check": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]),
            "mlck_blob_save": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_uint64)]),
            "mlck_blob_load": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
            "mlck_snapshot_record": (C.c_int, [vp, u32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint8,
                                               C.c_uint64, C.c_uint32, vp]),
            "mlck_snapshot_record_host": (C.c_int, [vp, u32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                                    C.c_uint8, C.c_uint64, C.c_uint32, vp, vp, C.c_uint64,
                                                    u64p]),
            "mlck_dense_checkpoint": (C.c_int, [vp, vp]),
            "mlck_fnv1a64": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, u64p]),
            "mlck_fnv1a64_profile": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, u64p, u64p, vp]),
            "mlck_parse_record": (C.c_int, [vp, C.c_int, C.POINTER(RecordInfo), C.POINTER(EntryInfo),
                                            C.c_uint32, u32p]),
            "mlck_read_entry": (C.c_int, [vp, C.POINTER(EntryInfo), C.c_int, f32p, f32p, f32p, f32p]),
            "mlck_check_coverage": (C.c_int, [C.POINTER(vp), C.c_uint32, C.c_uint64, C.c_int]),
            "mlck_gradlog_create": (C.c_int, [vp, C.c_uint32, u64p, C.c_uint32, C.POINTER(vp)]),
            "mlck_gradlog_destroy": (C.c_int, [vp]),
            "mlck_gradlog_put": (C.c_int, [vp, C.c_uint64, C.c_uint32, f32p]),
            "mlck_gradlog_slot": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.POINTER(vp)]),
            "mlck_gradlog_fill_synthetic": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint64]),
            "mlck_optimizer_step_adam": (C.c_int, [vp, vp, vp, vp, u64p, vp, C.c_uint64,
                                                   C.POINTER(Optimizer)]),
            "mlck_state_apply_updates": (C.c_int, [vp, u32p, C.c_uint32, vp, C.c_uint64,
                                                   C.POINTER(Optimizer)]),
            "mlck_localized_recover": (C.c_int, [vp, u32p, C.c_uint32, C.POINTER(vp), C.c_uint32, C.c_uint64,
                                                 C.c_uint32, C.c_uint64, vp, C.c_uint64, C.POINTER(Optimizer)]),
            "mlck_sparse_to_dense_convert": (C.c_int, [vp, C.POINTER(vp), C.c_uint32, C.c_uint64, C.c_uint32,
                                                       C.c_uint64, vp, C.POINTER(Optimizer)]),
            "mlck_log_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, C.POINTER(vp)]),
            "mlck_log_destroy": (C.c_int, [vp]),
            "mlck_log_put": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint8, vp, C.c_uint64]),
            "mlck_log_get": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint8, f32p, C.c_uint64,
                                       u64p]),
            "mlck_log_get_device": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint8, vp,
                                              C.c_uint64, u64p]),
            "mlck_log_count": (C.c_uint64, [vp]),
            "mlck_log_bytes": (C.c_uint64, [vp]),
            "mlck_log_entry": (C.c_int, [vp, C.c_uint64, u64p, u32p, u32p, u8p, f32p, C.c_uint64, u64p]),
            "mlck_gc_logs": (C.c_int, [vp, C.c_uint64]),
            "mlck_log_sync": (C.c_int, [vp]),
            "mlck_quantize": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_int]),
            "mlck_encode_compute": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_int]),
            "mlck_decode_compute": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_int]),
            "mlck_ipc_export": (C.c_int, [vp, vp, u8p]),
            "mlck_ipc_open": (C.c_int, [vp, u8p, C.POINTER(vp)]),
            "mlck_ipc_close": (C.c_int, [vp, vp]),
            "mlck_enable_peer_access": (C.c_int, [vp, C.c_int]),
            "mlck_event_record": (C.c_int, [vp, C.c_int]),
            "mlck_event_elapsed_ms": (C.c_int, [vp, C.c_int, C.c_int, f32p]),
            "mlck_device_alloc": (C.c_int, [vp, C.c_uint64, C.POINTER(vp)]),
            "mlck_device_free": (C.c_int, [vp, vp]),
            "mlck_device_memset": (C.c_int, [vp, vp, C.c_int, C.c_uint64]),
            "mlck_host_alloc_pinned": (C.c_int, [vp, C.c_uint64, C.POINTER(vp)]),
            "mlck_host_free_pinned": (C.c_int, [vp, vp]),
            "mlck_memcpy_h2d": (C.c_int, [vp, vp, vp, C.c_uint64]),
            "mlck_memcpy_d2h": (C.c_int, [vp, vp, vp, C.c_uint64]),
            "mlck_ctx_set_hash_reserve": (C.c_int, [vp, C.c_int]),
            "mlck_gradlog_capture": (C.c_int, [vp, C.c_uint64, C.c_uint32, vp]),
            "mlck_ctx_set_witness": (C.c_int, [vp, C.c_int]),
            "mlck_ctx_set_hash_async": (C.c_int, [vp, C.c_int]),
            "mlck_ctx_set_convert_overlap": (C.c_int, [vp, C.c_int]),
            "mlck_engine_create": (C.c_int, [vp, C.POINTER(EngineConfig), C.POINTER(vp)]),
            "mlck_engine_destroy": (C.c_int, [vp]),
            "mlck_engine_op_count": (C.c_uint32, [vp]),
            "mlck_engine_param_counts": (C.c_int, [vp, u64p]),
            "mlck_engine_stage_of_op": (C.c_int32, [vp, C.c_uint32]),
            "mlck_engine_run_iteration": (C.c_int, [vp, vp, u8p, vp, vp]),
            "mlck_engine_replay_scoped_iteration": (C.c_int, [vp, vp, C.c_uint64, C.c_int32, C.c_int32, u8p, vp]),
            "mlck_sparse_to_dense_convert_recompute": (C.c_int, [vp, vp, C.POINTER(vp), C.c_uint32, C.c_uint64,
                                                                 C.c_uint32, C.c_uint64]),
            "mlck_localized_recover_recompute": (C.c_int, [vp, vp, C.c_int32, C.c_int32, C.POINTER(vp), C.c_uint32,
                                                           C.c_uint64, C.c_uint32, C.c_uint64, vp, C.c_uint64]),
            "mlck_ctx_witness_stats": (C.c_int, [vp, u64p, u64p]),
            "mlck_blob_witness_ptr": (vp, [vp]),
            "mlck_gradlog_bytes": (C.c_uint64, [vp]),
            "mlck_conversion_plan": (C.c_int, [C.POINTER(vp), C.c_uint32, C.c_int, u32p, C.c_uint64, u64p, u64p]),
            "mlck_localized_recover_segment": (C.c_int, [vp, C.c_int32, C.c_int32, i32p, C.c_int32, C.POINTER(vp),
                                                         C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, vp,
                                                         C.c_uint32, vp, C.c_uint64, C.POINTER(Optimizer)]),
            "mlck_log_set_async": (C.c_int, [vp, C.c_int]),
            "mlck_log_fence": (C.c_int, [vp, vp]),
            "mlck_upstream_log_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                                    C.c_int64]),
            "mlck_check_log_budget": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int64,
                                                C.c_double, C.c_int32]),
            "mlck_pack_reduced": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_int, C.c_int]),
            "mlck_unpack_reduced": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_int, C.c_int]),
            "mlck_quantize_values": (C.c_int, [vp, f32p, f32p, C.c_uint64, C.c_int]),
            "mlck_pack_reduced_values": (C.c_int, [vp, f32p, u16p, C.c_uint64, C.c_int, C.c_int]),
            "mlck_unpack_reduced_values": (C.c_int, [vp, u16p, f32p, C.c_uint64, C.c_int, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def check(rc: int):
    if rc == 0:
        return
    msg = lib().mlck_last_error().decode()
    if rc == 1:
        raise MlckInvalid(msg)
    raise MlckRuntime(msg)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _u32(ids):
    return np.ascontiguousarray(np.asarray(list(ids), dtype=np.uint32))


# --------------------------------------------------------------------------
class Context:
    """One device context (stream, staging, scratch)."""

    def __init__(self, device: int = 0):
        self.h = vp()
        check(lib().mlck_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            lib().mlck_ctx_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        check(lib().mlck_ctx_set_stream(self.h, stream_handle or None))

    def synchronize(self):
        check(lib().mlck_ctx_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(lib().mlck_ctx_kernel_launches(self.h))

    def set_replica_mode(self, mode: int):
        """-1 (default): auto (2 for replicas in local HBM, else 1); 1: pack,
        then copy engines overlapped with the hash; 5: pack, then the hash
        kernel stores the replicas; 3: pack, then a push kernel on reserved
        SMs overlapped with the hash; 2: fused gather+store+hash kernel; 0:
        pack-kernel stores, then hash; 4: copy engines after the hash."""
        check(lib().mlck_ctx_set_replica_mode(self.h, mode))

    def set_witness(self, on: bool):
        """Witnessed re-verification of records this context hashed (default on)."""
        check(lib().mlck_ctx_set_witness(self.h, 1 if on else 0))

    def witness_stats(self) -> tuple[int, int]:
        """(witnessed verifications, of which fell back to a full hash)."""
        u, f = C.c_uint64(), C.c_uint64()
        check(lib().mlck_ctx_witness_stats(self.h, C.byref(u), C.byref(f)))
        return u.value, f.value

    def set_convert_overlap(self, witness_sms: int):
        """Witnessed verification on `witness_sms` SMs beside the conversion replay (0 = sequential)."""
        check(lib().mlck_ctx_set_convert_overlap(self.h, witness_sms))

    def set_hash_async(self, on: bool):
        """Trailer hash on a side stream after the pack (default off)."""
        check(lib().mlck_ctx_set_hash_async(self.h, 1 if on else 0))

    def set_hash_reserve(self, sms: int):
        """SMs the hash kernel leaves to co-scheduled work (0 = all SMs)."""
        check(lib().mlck_ctx_set_hash_reserve(self.h, sms))

    # ---- codecs: the reference's scalar forms (tensor.hpp:99-183) on device
    def quantize_values(self, x, compute_bytes: int) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float32)
        out = np.empty_like(x)
        check(lib().mlck_quantize_values(self.h, _ptr(x, f32p), _ptr(out, f32p), x.size, compute_bytes))
        return out

    def pack_reduced_values(self, x, ebits: int, mbits: int) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float32)
        out = np.empty(x.size, dtype=np.uint16)
        check(lib().mlck_pack_reduced_values(self.h, _ptr(x, f32p), _ptr(out, u16p), x.size, ebits, mbits))
        return out

    def unpack_reduced_values(self, codes, ebits: int, mbits: int) -> np.ndarray:
        c = np.ascontiguousarray(np.atleast_1d(codes), dtype=np.uint16)
        out = np.empty(c.size, dtype=np.float32)
        check(lib().mlck_unpack_reduced_values(self.h, _ptr(c, u16p), _ptr(out, f32p), c.size, ebits, mbits))
        return out

    def fastmath_check(self, n_div: int, seed: int = 1) -> tuple[int, int]:
        """(division, sqrt) mismatches of the replay's spelled-out fast paths."""
        out = (C.c_uint64 * 2)()
        check(lib().mlck_fastmath_check(self.h, n_div, seed, out))
        return int(out[0]), int(out[1])

    def set_timing(self, on: bool):
        check(lib().mlck_ctx_set_timing(self.h, int(on)))

    def timings(self):
        """[(label, ms)] of the kernels launched since the last call."""
        labels = C.create_string_buffer(1 << 16)
        cap = 4096
        ms = (C.c_float * cap)()
        n = C.c_uint32()
        check(lib().mlck_ctx_timings(self.h, labels, 1 << 16, ms, cap, C.byref(n)))
        names = labels.value.decode().split(",") if n.value else []
        return [(names[i], float(ms[i])) for i in range(min(n.value, cap))]

    # raw memory helpers
    def alloc(self, nbytes: int) -> int:
        p = vp()
        check(lib().mlck_device_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def free(self, ptr: int):
        check(lib().mlck_device_free(self.h, ptr))

    def memset(self, ptr: int, value: int, nbytes: int):
        check(lib().mlck_device_memset(self.h, ptr, value, nbytes))

    def alloc_pinned(self, nbytes: int) -> int:
        p = vp()
        check(lib().mlck_host_alloc_pinned(self.h, nbytes, C.byref(p)))
        return p.value

    def free_pinned(self, ptr: int):
        check(lib().mlck_host_free_pinned(self.h, ptr))

    def h2d(self, dst: int, src: int, nbytes: int):
        check(lib().mlck_memcpy_h2d(self.h, dst, src, nbytes))

    def d2h(self, dst: int, src: int, nbytes: int):
        check(lib().mlck_memcpy_d2h(self.h, dst, src, nbytes))

    def upload(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        p = self.alloc(arr.nbytes)
        self.h2d(p, arr.ctypes.data, arr.nbytes)
        self.synchronize()
        return p

    def download(self, ptr: int, nbytes: int) -> bytes:
        out = np.empty(nbytes, dtype=np.uint8)
        self.d2h(out.ctypes.data, ptr, nbytes)
        self.synchronize()
        return out.tobytes()

    def event_record(self, slot: int):
        check(lib().mlck_event_record(self.h, slot))

    def event_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(lib().mlck_event_elapsed_ms(self.h, a, b, C.byref(ms)))
        return ms.value

    def fnv1a64(self, device_ptr: int, n: int, seed: int = 0xcbf29ce484222325) -> int:
        """fnv1a64 (digest.hpp:18-25) over device bytes."""
        out = C.c_uint64()
        check(lib().mlck_fnv1a64(self.h, device_ptr, n, seed, C.byref(out)))
        return out.value

    def fnv1a64_profile(self, device_ptr: int, n: int, seed: int = 0xcbf29ce484222325, trace=None):
        out = C.c_uint64()
        cnt = (C.c_uint64 * 24)()
        check(lib().mlck_fnv1a64_profile(self.h, device_ptr, n, seed, C.byref(out), cnt,
                                         trace.ctypes.data if trace is not None else None))
        keys = ["lookback_probes", "spin_rereads", "cycles_rounds", "cycles_wait", "cycles_final", "chunks",
                "cycles_other", "cycles_refill",
                "lb_idle", "lb_probe", "lb_spin", "lb_compose", "lb_publish", "lb_total", "lb_handoff", "lb_arrive",
                "cyc_refill", "cyc_data_wait", "cyc_round_core", "cyc_scan_pub", "cyc_final_hash", "x21", "x22", "x23"]
        return out.value, dict(zip(keys, [int(x) for x in cnt]))

    def enable_peer_access(self, peer: int):
        check(lib().mlck_enable_peer_access(self.h, peer))

    def ipc_export(self, ptr: int) -> bytes:
        h = (C.c_uint8 * 64)()
        check(lib().mlck_ipc_export(self.h, ptr, h))
        return bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        p = vp()
        check(lib().mlck_ipc_open(self.h, h, C.byref(p)))
        return p.value

    def ipc_close(self, ptr: int):
        check(lib().mlck_ipc_close(self.h, ptr))

    # codecs
    def quantize(self, dev_in: int, dev_out: int, n: int, cb: int):
        check(lib().mlck_quantize(self.h, dev_in, dev_out, n, cb))

    def encode_compute(self, dev_in: int, dev_codes: int, n: int, cb: int):
        check(lib().mlck_encode_compute(self.h, dev_in, dev_codes, n, cb))

    def decode_compute(self, dev_codes: int, dev_out: int, n: int, cb: int):
        check(lib().mlck_decode_compute(self.h, dev_codes, dev_out, n, cb))


@dataclass
class OpHost:
    master: np.ndarray
    m: np.ndarray
    v: np.ndarray
    step: int
    compute: np.ndarray
    has_full_state: bool


class DeviceState:
    """Device-resident TrainState (engine.hpp:47-51)."""

    def __init__(self, ctx: Context, param_counts, compute_bytes: int = 2):
        self.ctx = ctx
        self.param_counts = [int(p) for p in param_counts]
        self.compute_bytes = compute_bytes
        pc = np.ascontiguousarray(self.param_counts, dtype=np.uint64)
        self.h = vp()
        check(lib().mlck_state_create(ctx.h, len(pc), _ptr(pc, u64p), compute_bytes, C.byref(self.h)))

    def close(self):
        if self.h:
            if self.ctx.h:  # not after its context: the handle refers to it (memory returns at exit)
                lib().mlck_state_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_ops(self):
        return len(self.param_counts)

    def set_meta(self, iteration: int, data_seed: int):
        check(lib().mlck_state_set_meta(self.h, iteration, data_seed))

    def meta(self):
        it, seed = C.c_uint64(), C.c_uint64()
        check(lib().mlck_state_get_meta(self.h, C.byref(it), C.byref(seed)))
        return it.value, seed.value

    def upload_op(self, i, master, m, v, step, has_full_state=True):
        master, m, v = _f32(master), _f32(m), _f32(v)
        assert master.size == self.param_counts[i]
        check(lib().mlck_state_upload_op(self.h, i, _ptr(master, f32p), _ptr(m, f32p), _ptr(v, f32p), step,
                                         int(has_full_state)))

    def download_op(self, i) -> OpHost:
        n = self.param_counts[i]
        a = [np.empty(n, dtype=np.float32) for _ in range(4)]
        st, hf = C.c_uint64(), C.c_int()
        check(lib().mlck_state_download_op(self.h, i, *(_ptr(x, f32p) for x in a[:3]), C.byref(st),
                                           _ptr(a[3], f32p), C.byref(hf)))
        return OpHost(a[0], a[1], a[2], st.value, a[3], bool(hf.value))

    def set_step(self, i, step, has_full_state=True):
        check(lib().mlck_state_set_step(self.h, i, step, int(has_full_state)))

    def op_ptrs(self, i):
        ps = [vp() for _ in range(4)]
        check(lib().mlck_state_op_ptrs(self.h, i, *(C.byref(p) for p in ps)))
        return tuple(p.value for p in ps)

    def fill_synthetic(self, seed: int, step: int = 10):
        check(lib().mlck_state_fill_synthetic(self.h, seed, step))

    def serialize_state(self) -> bytes:
        """Engine::serialize_state (engine.hpp:246-261)."""
        n = C.c_uint64()
        check(lib().mlck_state_serialize(self.h, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.uint8)
        check(lib().mlck_state_serialize(self.h, _ptr(out, u8p), n.value, C.byref(n)))
        return out.tobytes()

    def serialize_state_blob(self, out: "Blob"):
        check(lib().mlck_state_serialize_blob(self.h, out.h))

    def apply_updates(self, ids, gradlog: "GradLog", iteration: int, opt: Optimizer | None = None):
        """Engine::apply_updates (engine.hpp:699-728) for the listed ops."""
        ids = _u32(ids)
        opt = opt or Optimizer.adam()
        check(lib().mlck_state_apply_updates(self.h, _ptr(ids, u32p), ids.size, gradlog.h, iteration,
                                             C.byref(opt)))


def witness_bytes(record_bytes: int) -> int:
    """Capacity a replica witness buffer needs for a record of record_bytes."""
    return int(lib().mlck_witness_bytes(record_bytes))


class Blob:
    """A serialized record in device memory (+ replicas)."""

    def __init__(self, ctx: Context, capacity: int = 256, _h=None):
        self.ctx = ctx
        self.h = vp()
        if _h is not None:
            self.h = _h
        else:
            check(lib().mlck_blob_create(ctx.h, capacity, C.byref(self.h)))

    @classmethod
    def from_host(cls, ctx: Context, data: bytes) -> "Blob":
        a = np.frombuffer(bytes(data), dtype=np.uint8)
        h = vp()
        check(lib().mlck_blob_from_host(ctx.h, _ptr(a, u8p) if a.size else None, a.size, C.byref(h)))
        return cls(ctx, _h=h)

    @classmethod
    def wrap(cls, ctx: Context, record_ptr: int, n: int, witness_ptr: int | None = None) -> "Blob":
        """A read-only blob over n record bytes in device memory the caller owns
        (a replica buffer), with its witness when given (mlck_blob_wrap)."""
        h = vp()
        check(lib().mlck_blob_wrap(ctx.h, record_ptr, n, witness_ptr, C.byref(h)))
        return cls(ctx, _h=h)

    def add_replica_witness(self, device_ptr: int, capacity: int):
        """Each record's witness also goes to this buffer beside a replica."""
        check(lib().mlck_blob_add_replica_witness(self.h, device_ptr, capacity))

    def close(self):
        if self.h:
            if self.ctx.h:  # not after its context: the handle refers to it (memory returns at exit)
                lib().mlck_blob_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def size(self) -> int:
        return int(lib().mlck_blob_size(self.h))

    @property
    def device_ptr(self) -> int:
        return int(lib().mlck_blob_device_ptr(self.h) or 0)

    @property
    def witness_ptr(self) -> int:
        """Device pointer of the record's witness (0 when it has none)."""
        return int(lib().mlck_blob_witness_ptr(self.h) or 0)

    def to_host(self) -> bytes:
        out = np.empty(self.size, dtype=np.uint8)
        check(lib().mlck_blob_to_host(self.h, _ptr(out, u8p), out.size))
        return out.tobytes()

    def add_replica(self, device_ptr: int, capacity: int):
        check(lib().mlck_blob_add_replica(self.h, device_ptr, capacity))

    def clear_replicas(self):
        check(lib().mlck_blob_clear_replicas(self.h))

    def replication(self) -> int:
        """Replicas holding the complete last record (0 while in flight)."""
        n = C.c_uint32()
        check(lib().mlck_blob_replication(self.h, C.byref(n)))
        return int(n.value)

    def save(self, path: str) -> int:
        """Persist the record bytes (MLCK v1 wire format) to `path`."""
        n = C.c_uint64()
        check(lib().mlck_blob_save(self.h, os.fsencode(path), C.byref(n)))
        return int(n.value)

    @classmethod
    def load(cls, ctx: Context, path: str) -> "Blob":
        h = vp()
        check(lib().mlck_blob_load(ctx.h, os.fsencode(path), C.byref(h)))
        return cls(ctx, _h=h)


def snapshot_record(state: DeviceState, active, compute_only, slot_index: int, kind: int = 1,
                    window_start: int = 0, wsparse: int = 1, out: Blob | None = None) -> Blob:
    """serialize_record(take_sparse_snapshot(engine, slot, slot_index), plan,
    kind, window_start, wsparse) (snapshot.hpp:204-241, 115-144)."""
    a, c = _u32(active), _u32(compute_only)
    out = out or Blob(state.ctx)
    check(lib().mlck_snapshot_record(state.h, _ptr(a, u32p), a.size, _ptr(c, u32p), c.size, slot_index, kind,
                                     window_start, wsparse, out.h))
    return out


def snapshot_record_host(state: DeviceState, active, compute_only, slot_index: int, kind=1, window_start=0,
                         wsparse=1, scratch: Blob | None = None, host_buf: int | None = None,
                         cap: int = 0) -> int | bytes:
    """Same record delivered to host memory (pinned host_buf when given)."""
    a, c = _u32(active), _u32(compute_only)
    scratch = scratch or Blob(state.ctx)
    n = C.c_uint64()
    args = (state.h, _ptr(a, u32p), a.size, _ptr(c, u32p), c.size, slot_index, kind, window_start, wsparse,
            scratch.h)
    if host_buf is not None:
        check(lib().mlck_snapshot_record_host(*args, host_buf, cap, C.byref(n)))
        return n.value
    check(lib().mlck_snapshot_record_host(*args, None, 0, C.byref(n)))
    out = np.empty(n.value, dtype=np.uint8)
    check(lib().mlck_snapshot_record_host(*args, out.ctypes.data, out.size, C.byref(n)))
    return out.tobytes()


def dense_checkpoint(state: DeviceState, out: Blob | None = None) -> Blob:
    """take_dense_checkpoint(engine).serialize(plan) (snapshot.hpp:245-295)."""
    out = out or Blob(state.ctx)
    check(lib().mlck_dense_checkpoint(state.h, out.h))
    return out


def parse_record(blob: Blob, compute_bytes: int):
    """parse_record (snapshot.hpp:153-197): (header dict, entry dicts)."""
    info = RecordInfo()
    n = C.c_uint32()
    check(lib().mlck_parse_record(blob.h, compute_bytes, C.byref(info), None, 0, C.byref(n)))
    cap = max(1, n.value)
    ents = (EntryInfo * cap)()
    check(lib().mlck_parse_record(blob.h, compute_bytes, C.byref(info), ents, cap, C.byref(n)))
    header = dict(kind=info.kind, iteration=info.iteration, window_start=info.window_start,
                  wsparse=info.wsparse, slot=info.slot, data_seed=info.data_seed)
    entries = [dict(id=ents[i].id, mode=ents[i].mode, param_count=ents[i].param_count, step=ents[i].step,
                    payload_offset=ents[i].payload_offset) for i in range(n.value)]
    return header, entries


def read_entry(blob: Blob, entry: dict, compute_bytes: int) -> dict:
    e = EntryInfo(entry["id"], entry["mode"], entry["param_count"], entry["step"], entry["payload_offset"])
    P = entry["param_count"]
    if entry["mode"] == 0:
        a = [np.empty(P, dtype=np.float32) for _ in range(3)]
        check(lib().mlck_read_entry(blob.h, C.byref(e), compute_bytes, *(_ptr(x, f32p) for x in a), None))
        return dict(master=a[0], m=a[1], v=a[2], step=entry["step"])
    c = np.empty(P, dtype=np.float32)
    check(lib().mlck_read_entry(blob.h, C.byref(e), compute_bytes, None, None, None, _ptr(c, f32p)))
    return dict(compute=c)


def check_coverage(blobs, op_count: int, compute_bytes: int):
    """SparseCheckpoint::check_coverage (snapshot.hpp:322-334)."""
    arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
    check(lib().mlck_check_coverage(arr, len(blobs), op_count, compute_bytes))


class GradLog:
    """Per-iteration operator gradients on the device (Adam-replay input)."""

    def __init__(self, ctx: Context, param_counts, capacity_iterations: int):
        self.ctx = ctx
        self.param_counts = [int(p) for p in param_counts]
        pc = np.ascontiguousarray(self.param_counts, dtype=np.uint64)
        self.h = vp()
        check(lib().mlck_gradlog_create(ctx.h, len(pc), _ptr(pc, u64p), capacity_iterations, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().mlck_gradlog_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def put(self, iteration: int, op: int, grad):
        g = _f32(grad)
        check(lib().mlck_gradlog_put(self.h, iteration, op, _ptr(g, f32p)))

    def slot(self, iteration: int, op: int) -> int:
        p = vp()
        check(lib().mlck_gradlog_slot(self.h, iteration, op, C.byref(p)))
        return p.value

    def fill_synthetic(self, first_iteration: int, n_iterations: int, seed: int):
        check(lib().mlck_gradlog_fill_synthetic(self.h, first_iteration, n_iterations, seed))

    def capture(self, iteration: int, op: int, device_src: int):
        """Copy a trainer-owned device gradient into the log (ctx stream)."""
        check(lib().mlck_gradlog_capture(self.h, iteration, op, device_src))

    @property
    def nbytes(self) -> int:
        return int(lib().mlck_gradlog_bytes(self.h))


def sparse_to_dense_convert(out: DeviceState, blobs, window_start: int, wsparse: int, data_seed: int,
                            gradlog: GradLog | None, opt: Optimizer | None = None):
    """sparse_to_dense_convert (recovery.hpp:180-227) with logged-gradient replay."""
    arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
    opt = opt or Optimizer.adam()
    check(lib().mlck_sparse_to_dense_convert(out.h, arr, len(blobs), window_start, wsparse, data_seed,
                                             gradlog.h if gradlog is not None else None, C.byref(opt)))


def localized_recover(out: DeviceState, scope, blobs, window_start: int, wsparse: int, data_seed: int,
                      gradlog: GradLog | None, target_iteration: int, opt: Optimizer | None = None):
    """localized_recover (recovery.hpp:240-289): conversion of the operators in
    `scope` plus the lost iterations up to target_iteration, from the
    gradient log; only the scope's operators of `out` are written."""
    ids = np.ascontiguousarray(np.array(list(scope), dtype=np.uint32))
    arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
    opt = opt or Optimizer.adam()
    check(lib().mlck_localized_recover(out.h, _ptr(ids, u32p), ids.size, arr, len(blobs), window_start, wsparse,
                                       data_seed, gradlog.h if gradlog is not None else None, target_iteration, C.byref(opt)))


def localized_recover_segment(out: DeviceState, stage_lo: int, stage_hi: int, stage_of_op, n_stages: int, blobs,
                              window_start: int, wsparse: int, data_seed: int, log: "UpstreamLog | None",
                              n_global_microbatches: int, gradlog: GradLog | None, target_iteration: int,
                              opt: Optimizer | None = None):
    """localized_recover(engine, RecoverySegment{stage_lo, stage_hi}, ckpt, logs,
    target) (recovery.hpp:240-244): the scope is Engine::stage_of_op in the
    segment's stage range; the boundary inputs it consumes must be in `log`."""
    st = np.ascontiguousarray(np.array(list(stage_of_op), dtype=np.int32))
    arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
    opt = opt or Optimizer.adam()
    check(lib().mlck_localized_recover_segment(out.h, stage_lo, stage_hi, _ptr(st, i32p), n_stages, arr, len(blobs),
                                               window_start, wsparse, data_seed, log.h if log is not None else None,
                                               n_global_microbatches, gradlog.h if gradlog is not None else None,
                                               target_iteration, C.byref(opt)))


def conversion_plan(blobs, window_start: int, compute_bytes: int):
    """conversion_plan (recovery.hpp:123-137): [(record_index, replay_iteration,
    activating ids)] -- step k loads record k, replays window_start + k + 1."""
    arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
    counts = np.zeros(max(1, len(blobs)), dtype=np.uint64)
    total = C.c_uint64()
    check(lib().mlck_conversion_plan(arr, len(blobs), compute_bytes, None, 0, _ptr(counts, u64p), C.byref(total)))
    ids = np.zeros(max(1, total.value), dtype=np.uint32)
    check(lib().mlck_conversion_plan(arr, len(blobs), compute_bytes, _ptr(ids, u32p), ids.size,
                                     _ptr(counts, u64p), C.byref(total)))
    out, at = [], 0
    for k in range(len(blobs)):
        c = int(counts[k])
        out.append((k, window_start + k + 1, [int(x) for x in ids[at:at + c]]))
        at += c
    return out


def upstream_log_bytes(token_dim: int, pp_stages: int, microbatches: int, microbatch_size: int, dp_degree: int,
                       wsparse: int) -> int:
    """upstream_log_bytes (recovery.hpp:296-304)."""
    return int(lib().mlck_upstream_log_bytes(token_dim, pp_stages, microbatches, microbatch_size, dp_degree,
                                             wsparse))


def check_log_budget(token_dim: int, pp_stages: int, microbatches: int, microbatch_size: int, dp_degree: int,
                     wsparse: int, cpu_mem_per_node: float, nodes: int):
    """check_log_budget (recovery.hpp:308-317): ValueError when the host budget cannot hold the logs."""
    check(lib().mlck_check_log_budget(token_dim, pp_stages, microbatches, microbatch_size, dp_degree, wsparse,
                                      cpu_mem_per_node, nodes))


def optimizer_step_adam(ctx: Context, master: int, m: int, v: int, step: int, grad: int, n: int,
                        opt: Optimizer | None = None) -> int:
    """optimizer_step_adam (engine.hpp:738-753) on device pointers; returns step."""
    st = C.c_uint64(step)
    opt = opt or Optimizer.adam()
    check(lib().mlck_optimizer_step_adam(ctx.h, master, m, v, C.byref(st), grad, n, C.byref(opt)))
    return st.value


class UpstreamLog:
    """Boundary log (LogKey/UpstreamLog, engine.hpp:55-94) on a side stream.
    kind 0 = pinned host ring, 1 = device ring on `device`."""

    def __init__(self, ctx: Context, capacity_bytes: int, kind: int = 0, device: int = 0, external: int = 0):
        """kind 2: ring on caller-owned device memory at `external` (e.g. an
        IPC-opened peer buffer)."""
        self.ctx = ctx
        self.h = vp()
        if kind == 2:
            check(lib().mlck_log_create_external(ctx.h, external, capacity_bytes, C.byref(self.h)))
        else:
            check(lib().mlck_log_create(ctx.h, kind, device, capacity_bytes, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().mlck_log_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def put(self, iteration, micro_batch, boundary, direction, device_src: int, n_floats: int):
        check(lib().mlck_log_put(self.h, iteration, micro_batch, boundary, direction, device_src, n_floats))

    def at(self, iteration, micro_batch, boundary, direction) -> np.ndarray:
        n = C.c_uint64()
        check(lib().mlck_log_get(self.h, iteration, micro_batch, boundary, direction, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        check(lib().mlck_log_get(self.h, iteration, micro_batch, boundary, direction, _ptr(out, f32p), out.size,
                                 C.byref(n)))
        return out

    def get_device(self, iteration, micro_batch, boundary, direction, dst: int, cap: int) -> int:
        n = C.c_uint64()
        check(lib().mlck_log_get_device(self.h, iteration, micro_batch, boundary, direction, dst, cap,
                                        C.byref(n)))
        return n.value

    def __len__(self):
        return int(lib().mlck_log_count(self.h))

    def bytes(self) -> int:
        return int(lib().mlck_log_bytes(self.h))

    def entries(self):
        out = []
        for i in range(len(self)):
            it, mb, b, d, n = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint8(), C.c_uint64()
            check(lib().mlck_log_entry(self.h, i, C.byref(it), C.byref(mb), C.byref(b), C.byref(d), None, 0,
                                       C.byref(n)))
            data = np.empty(n.value, dtype=np.float32)
            check(lib().mlck_log_entry(self.h, i, C.byref(it), C.byref(mb), C.byref(b), C.byref(d),
                                       _ptr(data, f32p), data.size, C.byref(n)))
            out.append(((it.value, mb.value, b.value, d.value), data))
        return out

    def gc(self, persisted_window_start: int):
        """gc_logs (engine.hpp:90-94)."""
        check(lib().mlck_gc_logs(self.h, persisted_window_start))

    def sync(self):
        check(lib().mlck_log_sync(self.h))

    def set_async(self, on: bool):
        """ASYNC mode: put() does not order the ctx stream after the copy;
        fence() the stream that will overwrite a logged source."""
        check(lib().mlck_log_set_async(self.h, 1 if on else 0))

    def fence(self, stream: int | None = None):
        check(lib().mlck_log_fence(self.h, stream))


class Engine:
    """The miniature MoE trainer on the GPU (moelab::Engine, engine.hpp:150-730):
    run_iteration (producer of the boundary and gradient logs) and the
    recompute replay of conversion / localized recovery."""

    def __init__(self, ctx: Context, cfg: "EngineConfig | dict"):
        self.ctx = ctx
        self.cfg = cfg if isinstance(cfg, EngineConfig) else EngineConfig.from_dict(cfg)
        self.h = vp()
        check(lib().mlck_engine_create(ctx.h, C.byref(self.cfg), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().mlck_engine_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def op_count(self) -> int:
        return int(lib().mlck_engine_op_count(self.h))

    def param_counts(self) -> list:
        out = np.zeros(self.op_count, dtype=np.uint64)
        check(lib().mlck_engine_param_counts(self.h, _ptr(out, u64p)))
        return [int(x) for x in out]

    def stage_of_op(self, i: int) -> int:
        return int(lib().mlck_engine_stage_of_op(self.h, i))

    @staticmethod
    def _flags(frozen, n):
        if frozen is None:
            return None, None
        f = np.zeros(n, dtype=np.uint8)
        for i in frozen:
            f[i] = 1
        return f, _ptr(f, u8p)

    def run_iteration(self, st: DeviceState, frozen=None, log: "UpstreamLog | None" = None,
                      gradlog: GradLog | None = None):
        keep, fp = self._flags(frozen, self.op_count)
        check(lib().mlck_engine_run_iteration(self.h, st.h, fp, log.h if log is not None else None,
                                              gradlog.h if gradlog is not None else None))

    def replay_scoped_iteration(self, ops: DeviceState, iteration: int, stage_lo: int, stage_hi: int, frozen=None,
                                log: "UpstreamLog | None" = None):
        keep, fp = self._flags(frozen, self.op_count)
        check(lib().mlck_engine_replay_scoped_iteration(self.h, ops.h, iteration, stage_lo, stage_hi, fp,
                                                        log.h if log is not None else None))

    def sparse_to_dense_convert(self, out: DeviceState, blobs, window_start: int, wsparse: int, data_seed: int):
        """sparse_to_dense_convert (recovery.hpp:180-227) with the recompute replay."""
        arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
        check(lib().mlck_sparse_to_dense_convert_recompute(self.h, out.h, arr, len(blobs), window_start, wsparse,
                                                           data_seed))

    def localized_recover(self, out: DeviceState, stage_lo: int, stage_hi: int, blobs, window_start: int,
                          wsparse: int, data_seed: int, log: "UpstreamLog | None", target_iteration: int):
        """localized_recover (recovery.hpp:240-289) by recompute from the boundary log."""
        arr = (vp * max(1, len(blobs)))(*[b.h for b in blobs])
        check(lib().mlck_localized_recover_recompute(self.h, out.h, stage_lo, stage_hi, arr, len(blobs),
                                                     window_start, wsparse, data_seed,
                                                     log.h if log is not None else None, target_iteration))
