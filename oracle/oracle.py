"""ctypes loaders for the CPU checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference legs -- never by the product package.

* ``Oracle``  -- oracle/_build/libmoelab_oracle.so, the C restatement
  (oracle/moelab_oracle.c) of the reference checkpoint path.
* ``Reference`` -- oracle/_ref/libmoelab_ref.so, the UNMODIFIED reference
  headers (/root/reference/proj/include) compiled behind oracle/ref_shim.cpp.
  Present wherever it was built (it travels to the GPU box as a built file).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmoelab_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoelab_ref.so")

u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class MloEntry(C.Structure):
    _fields_ = [
        ("id", C.c_uint32), ("mode", C.c_uint8), ("param_count", C.c_uint64),
        ("step", C.c_uint64), ("master", f32p), ("m", f32p), ("v", f32p), ("compute", f32p),
    ]


class MloHeader(C.Structure):
    _fields_ = [
        ("kind", C.c_uint8), ("iteration", C.c_uint64), ("window_start", C.c_uint64),
        ("wsparse", C.c_uint32), ("slot", C.c_uint32), ("data_seed", C.c_uint64),
    ]


class MloParsedEntry(C.Structure):
    _fields_ = [
        ("id", C.c_uint32), ("mode", C.c_uint8), ("param_count", C.c_uint64),
        ("step", C.c_uint64), ("payload_offset", C.c_uint64),
    ]


class MloStateOp(C.Structure):
    _fields_ = [
        ("step", C.c_uint64), ("param_count", C.c_uint64),
        ("master", f32p), ("m", f32p), ("v", f32p),
    ]


ORACLE_ERRORS = {
    1: "container truncated",
    2: "container checksum mismatch",
    3: "container: bad magic",
    4: "container: unsupported version",
    5: "container: unsupported compute width",
}


@dataclass
class OpState:
    """One operator of a TrainState (engine.hpp:33-45)."""
    master: np.ndarray
    m: np.ndarray
    v: np.ndarray
    step: int = 0
    compute: np.ndarray | None = None  # values on the compute grid (float32)
    has_full_state: bool = True


@dataclass
class TrainState:
    ops: list = field(default_factory=list)
    iteration: int = 0
    data_seed: int = 0


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.mlo_fnv1a64.restype = C.c_uint64
        L.mlo_fnv1a64.argtypes = [u8p, C.c_size_t, C.c_uint64]
        L.mlo_quantize_value.argtypes = [C.c_float, C.c_int, f32p]
        L.mlo_quantize_array.argtypes = [f32p, C.c_size_t, C.c_int, f32p]
        L.mlo_pack_reduced.restype = C.c_uint16
        L.mlo_pack_reduced.argtypes = [C.c_float, C.c_int, C.c_int]
        L.mlo_unpack_reduced.restype = C.c_float
        L.mlo_unpack_reduced.argtypes = [C.c_uint16, C.c_int, C.c_int]
        L.mlo_encode_compute.restype = C.c_int64
        L.mlo_encode_compute.argtypes = [f32p, C.c_size_t, C.c_int, u8p]
        L.mlo_decode_compute.restype = C.c_int64
        L.mlo_decode_compute.argtypes = [u8p, C.c_size_t, C.c_int, f32p]
        L.mlo_record_size.restype = C.c_uint64
        L.mlo_record_size.argtypes = [C.POINTER(MloEntry), C.c_size_t, C.c_int]
        L.mlo_serialize_record.restype = C.c_int64
        L.mlo_serialize_record.argtypes = [C.POINTER(MloHeader), C.POINTER(MloEntry), C.c_size_t,
                                           C.c_int, u8p]
        L.mlo_parse_record.argtypes = [u8p, C.c_uint64, C.c_int, C.POINTER(MloHeader), u32p,
                                       C.POINTER(MloParsedEntry), C.c_uint32, u32p]
        L.mlo_adam_step.argtypes = [f32p, f32p, f32p, u64p, f32p, C.c_size_t, C.c_float,
                                    C.c_float, C.c_float, C.c_float]
        L.mlo_bias_correction.restype = C.c_float
        L.mlo_bias_correction.argtypes = [C.c_float, C.c_uint64]
        L.mlo_replay_op.argtypes = [f32p, f32p, f32p, u64p, f32p, C.c_uint32, C.c_size_t, C.c_int,
                                    C.c_float, C.c_float, C.c_float, C.c_float]
        L.mlo_state_size.restype = C.c_uint64
        L.mlo_state_size.argtypes = [C.POINTER(MloStateOp), C.c_size_t]
        L.mlo_serialize_state.restype = C.c_uint64
        L.mlo_serialize_state.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(MloStateOp),
                                          C.c_size_t, u8p]
        L.mlo_init_master.argtypes = [C.c_uint64, C.c_uint32, C.c_int32, f32p, C.c_size_t]
        L.mlo_synth_value.restype = C.c_float
        L.mlo_synth_value.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, C.c_float]
        L.mlo_synth_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_float, C.c_float, f32p, C.c_size_t]
        L.mlo_synth_fill_range.argtypes = [C.c_uint64, C.c_uint64, C.c_float, C.c_float, f32p, C.c_uint64,
                                           C.c_size_t]

    # ---- primitives
    def fnv1a64(self, data, seed: int = 0xcbf29ce484222325) -> int:
        a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        a = np.ascontiguousarray(a).view(np.uint8)
        return int(self.lib.mlo_fnv1a64(_ptr(a, u8p), a.size, seed))

    def quantize_value(self, x: float, compute_bytes: int) -> float:
        out = C.c_float()
        if self.lib.mlo_quantize_value(C.c_float(x), compute_bytes, C.byref(out)) != 0:
            raise ValueError(f"quantize: unsupported width {compute_bytes}")
        return out.value

    def quantize(self, vals: np.ndarray, compute_bytes: int) -> np.ndarray:
        """quantize_inplace (tensor.hpp:433-436) over an array."""
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        out = np.empty_like(vals)
        if self.lib.mlo_quantize_array(_ptr(vals, f32p), vals.size, compute_bytes, _ptr(out, f32p)) != 0:
            raise ValueError(f"quantize: unsupported width {compute_bytes}")
        return out

    def pack_reduced(self, x: float, e: int, m: int) -> int:
        return int(self.lib.mlo_pack_reduced(C.c_float(x), e, m))

    def unpack_reduced(self, c: int, e: int, m: int) -> float:
        return float(self.lib.mlo_unpack_reduced(c, e, m))

    def encode_compute(self, vals: np.ndarray, compute_bytes: int) -> bytes:
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        out = np.empty(vals.size * compute_bytes, dtype=np.uint8)
        n = self.lib.mlo_encode_compute(_ptr(vals, f32p), vals.size, compute_bytes, _ptr(out, u8p))
        if n < 0:
            raise ValueError("container: unsupported compute width")
        return out.tobytes()

    def decode_compute(self, codes: bytes, n: int, compute_bytes: int) -> np.ndarray:
        """read_compute (snapshot.hpp:95-111) over an array of codes."""
        a = np.frombuffer(codes, dtype=np.uint8)
        out = np.empty(n, dtype=np.float32)
        if self.lib.mlo_decode_compute(_ptr(a, u8p), n, compute_bytes, _ptr(out, f32p)) < 0:
            raise ValueError("container: unsupported compute width")
        return out

    # ---- container
    def _entries(self, entries, keep):
        arr = (MloEntry * max(1, len(entries)))()
        for i, e in enumerate(entries):
            ent = arr[i]
            ent.id, ent.mode, ent.param_count, ent.step = e["id"], e["mode"], e["param_count"], e.get("step", 0)
            for name in ("master", "m", "v", "compute"):
                a = e.get(name)
                if a is not None:
                    a = np.ascontiguousarray(a, dtype=np.float32)
                    keep.append(a)
                    setattr(ent, name, _ptr(a, f32p))
        return arr

    def serialize_record(self, header: dict, entries: list, compute_bytes: int) -> bytes:
        """entries: dicts with id, mode (0 Full/1 CO), param_count, step,
        master/m/v (Full) or compute (CO, grid values); sorted by id."""
        keep = []
        arr = self._entries(entries, keep)
        h = MloHeader(header.get("kind", 1), header["iteration"], header["window_start"],
                      header["wsparse"], header["slot"], header["data_seed"])
        size = self.lib.mlo_record_size(arr, len(entries), compute_bytes)
        out = np.empty(size, dtype=np.uint8)
        n = self.lib.mlo_serialize_record(C.byref(h), arr, len(entries), compute_bytes, _ptr(out, u8p))
        if n < 0:
            raise ValueError("container: unsupported compute width")
        assert n == size
        return out.tobytes()

    def parse_record(self, blob: bytes, compute_bytes: int):
        a = np.frombuffer(blob, dtype=np.uint8)
        h = MloHeader()
        n = C.c_uint32()
        ver = C.c_uint32()
        cap = 1 << 16
        ents = (MloParsedEntry * cap)()
        rc = self.lib.mlo_parse_record(_ptr(a, u8p), a.size, compute_bytes, C.byref(h), C.byref(n),
                                       ents, cap, C.byref(ver))
        if rc != 0:
            msg = ORACLE_ERRORS.get(rc, "error")
            if rc == 4:
                msg += f" {ver.value}"
            raise RuntimeError(msg)
        header = dict(kind=h.kind, iteration=h.iteration, window_start=h.window_start,
                      wsparse=h.wsparse, slot=h.slot, data_seed=h.data_seed)
        entries = [dict(id=ents[i].id, mode=ents[i].mode, param_count=ents[i].param_count,
                        step=ents[i].step, payload_offset=ents[i].payload_offset)
                   for i in range(n.value)]
        return header, entries

    # ---- optimizer
    def adam_step(self, master, m, v, step, grad, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        st = C.c_uint64(step)
        self.lib.mlo_adam_step(_ptr(master, f32p), _ptr(m, f32p), _ptr(v, f32p), C.byref(st),
                               _ptr(np.ascontiguousarray(grad, dtype=np.float32), f32p),
                               master.size, lr, b1, b2, eps)
        return st.value

    def bias_correction(self, beta: float, step: int) -> float:
        return float(self.lib.mlo_bias_correction(beta, step))

    def replay_op(self, master, m, v, step, grads, kind=0, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        grads = np.ascontiguousarray(grads, dtype=np.float32)
        st = C.c_uint64(step)
        n_steps = grads.shape[0] if grads.ndim == 2 else 0
        self.lib.mlo_replay_op(_ptr(master, f32p), _ptr(m, f32p), _ptr(v, f32p), C.byref(st),
                               _ptr(grads, f32p), n_steps, master.size, kind, lr, b1, b2, eps)
        return st.value

    # ---- dense image
    def serialize_state(self, state: TrainState) -> bytes:
        keep = []
        arr = (MloStateOp * max(1, len(state.ops)))()
        for i, op in enumerate(state.ops):
            for name in ("master", "m", "v"):
                a = np.ascontiguousarray(getattr(op, name), dtype=np.float32)
                keep.append(a)
                setattr(arr[i], name, _ptr(a, f32p))
            arr[i].step = op.step
            arr[i].param_count = op.master.size
        size = self.lib.mlo_state_size(arr, len(state.ops))
        out = np.empty(size, dtype=np.uint8)
        self.lib.mlo_serialize_state(state.iteration, state.data_seed, arr, len(state.ops), _ptr(out, u8p))
        return out.tobytes()

    # ---- synthetic inputs
    def init_master(self, seed, op_id, token_dim, n) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.mlo_init_master(seed, op_id, token_dim, _ptr(out, f32p), n)
        return out

    def synth(self, seed, stream, lo, hi, n, first=0) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.mlo_synth_fill_range(seed, stream, lo, hi, _ptr(out, f32p), first, n)
        return out


# --------------------------------------------------------------------------
# real reference (oracle/_ref)
# --------------------------------------------------------------------------
class MlrConfig(C.Structure):
    _fields_ = [
        ("layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
        ("shared_experts", C.c_int32), ("token_dim", C.c_int32), ("expert_hidden", C.c_int32),
        ("nonexpert_hidden", C.c_int32), ("residual", C.c_int32),
        ("expert_params", C.c_int64), ("nonexpert_params", C.c_int64), ("gate_params", C.c_int64),
        ("compute_bytes", C.c_int64), ("pp_stages", C.c_int32), ("dp_degree", C.c_int32),
        ("microbatches", C.c_int32), ("microbatch_size", C.c_int64), ("global_batch", C.c_int64),
        ("optimizer_kind", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float),
        ("beta2", C.c_float), ("eps", C.c_float), ("seed", C.c_uint64),
    ]


def toy_config(layers=1, stages=1, seed=1, experts=4, top_k=2, compute_bytes=2, token_dim=4,
               hidden=4, microbatches=2, mb_size=4, dp=1, optimizer_kind=0,
               expert_params=-1, nonexpert_params=-1, gate_params=-1, shared=0) -> MlrConfig:
    """test_recovery.cpp:14-29 toy_config (verify_toy.json shape at layers=3,
    stages=3); six_op_config (test_snapshot.cpp:13-28) is layers=1."""
    return MlrConfig(layers, experts, top_k, shared, token_dim, hidden, hidden, 1,
                     expert_params, nonexpert_params, gate_params, compute_bytes, stages, dp,
                     microbatches, mb_size, microbatches * mb_size * dp, optimizer_kind,
                     1e-3, 0.9, 0.999, 1e-8, seed)


class RefError(RuntimeError):
    pass


class Reference:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        cp = C.POINTER(MlrConfig)
        L.mlr_engine_create.restype = C.c_void_p
        L.mlr_engine_create.argtypes = [cp, C.c_char_p, C.c_size_t]
        L.mlr_engine_destroy.argtypes = [C.c_void_p]
        L.mlr_engine_run_iteration.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
        L.mlr_engine_iteration.restype = C.c_uint64
        L.mlr_engine_iteration.argtypes = [C.c_void_p]
        L.mlr_engine_data_seed.restype = C.c_uint64
        L.mlr_engine_data_seed.argtypes = [C.c_void_p]
        L.mlr_engine_op_count.restype = C.c_uint32
        L.mlr_engine_op_count.argtypes = [C.c_void_p]
        L.mlr_engine_param_count.restype = C.c_int64
        L.mlr_engine_param_count.argtypes = [C.c_void_p, C.c_uint32]
        L.mlr_engine_op_size.restype = C.c_uint64
        L.mlr_engine_op_size.argtypes = [C.c_void_p, C.c_uint32]
        L.mlr_engine_stage_of_op.restype = C.c_int32
        L.mlr_engine_stage_of_op.argtypes = [C.c_void_p, C.c_uint32]
        L.mlr_engine_get_op.argtypes = [C.c_void_p, C.c_uint32, f32p, f32p, f32p, u64p, f32p,
                                        C.POINTER(C.c_int32)]
        L.mlr_engine_set_op.argtypes = [C.c_void_p, C.c_uint32, f32p, f32p, f32p, C.c_uint64,
                                        C.c_uint64, C.c_int32]
        L.mlr_engine_set_iteration.argtypes = [C.c_void_p, C.c_uint64]
        L.mlr_engine_serialize_state.restype = C.c_size_t
        L.mlr_engine_serialize_state.argtypes = [C.c_void_p, u8p, C.c_size_t]
        L.mlr_engine_extract_grads.argtypes = [C.c_void_p, C.POINTER(f32p), C.c_char_p, C.c_size_t]
        L.mlr_schedule.argtypes = [C.c_void_p, C.c_int64, C.c_int64, u32p, u32p, u32p, C.c_char_p,
                                   C.c_size_t]
        L.mlr_snapshot.restype = C.c_int64
        L.mlr_snapshot.argtypes = [C.c_void_p, u32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                   C.c_uint8, C.c_uint64, C.c_uint32, u8p, C.c_size_t, C.c_char_p,
                                   C.c_size_t]
        L.mlr_dense_checkpoint.restype = C.c_int64
        L.mlr_dense_checkpoint.argtypes = [C.c_void_p, u8p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.mlr_parse_record.restype = C.c_int64
        L.mlr_parse_record.argtypes = [u8p, C.c_size_t, C.c_int64, u64p, u32p, C.c_char_p, C.c_size_t]
        L.mlr_convert.restype = C.c_int64
        L.mlr_convert.argtypes = [cp, C.c_uint64, C.c_uint32, C.POINTER(u8p), u64p, C.c_uint32,
                                  u8p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.mlr_localized_recover.restype = C.c_int64
        L.mlr_localized_recover.argtypes = [cp, C.c_uint64, C.c_uint32, C.POINTER(u8p), u64p, C.c_uint32,
                                            C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, u8p, C.c_size_t,
                                            C.c_char_p, C.c_size_t]
        L.mlr_check_coverage.argtypes = [C.c_uint32, C.POINTER(u8p), u64p, C.c_uint32, C.c_uint64,
                                         C.c_int64, C.c_char_p, C.c_size_t]
        L.mlr_log_create.restype = C.c_void_p
        L.mlr_log_destroy.argtypes = [C.c_void_p]
        L.mlr_log_count.restype = C.c_uint64
        L.mlr_log_count.argtypes = [C.c_void_p]
        L.mlr_log_bytes.restype = C.c_uint64
        L.mlr_log_bytes.argtypes = [C.c_void_p]
        L.mlr_log_entry.restype = C.c_int64
        L.mlr_log_entry.argtypes = [C.c_void_p, C.c_uint64, u64p, u32p, u32p, u8p, f32p, C.c_size_t]
        L.mlr_gc_logs.argtypes = [C.c_void_p, C.c_uint64]
        L.mlr_log_at.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint8,
                                 C.c_char_p, C.c_size_t]
        L.mlr_conversion_plan.restype = C.c_int64
        L.mlr_conversion_plan.argtypes = [C.c_uint64, C.c_uint32, C.POINTER(u8p), u64p, C.c_uint32, C.c_int64,
                                          u32p, C.c_size_t, u64p, u64p, C.c_char_p, C.c_size_t]
        L.mlr_check_log_budget.argtypes = [cp, C.c_int64, C.c_double, C.c_int32, C.c_char_p, C.c_size_t]
        L.mlr_upstream_log_bytes.restype = C.c_int64
        L.mlr_upstream_log_bytes.argtypes = [cp, C.c_int64]
        L.mlr_fnv1a64.restype = C.c_uint64
        L.mlr_fnv1a64.argtypes = [u8p, C.c_size_t, C.c_uint64]
        L.mlr_quantize_value.argtypes = [C.c_float, C.c_int, f32p, C.c_char_p, C.c_size_t]
        L.mlr_quantize_array.argtypes = [f32p, C.c_size_t, C.c_int, f32p, C.c_char_p, C.c_size_t]
        L.mlr_pack_array.argtypes = [f32p, C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_uint16)]
        L.mlr_unpack_array.argtypes = [C.POINTER(C.c_uint16), C.c_size_t, C.c_int, C.c_int, f32p]
        L.mlr_pack_reduced.restype = C.c_uint16
        L.mlr_pack_reduced.argtypes = [C.c_float, C.c_int, C.c_int]
        L.mlr_unpack_reduced.restype = C.c_float
        L.mlr_unpack_reduced.argtypes = [C.c_uint16, C.c_int, C.c_int]
        L.mlr_optimizer_step_adam.argtypes = [f32p, f32p, f32p, u64p, f32p, C.c_size_t, C.c_float,
                                              C.c_float, C.c_float, C.c_float, C.c_char_p, C.c_size_t]
        L.mlr_time_pack.restype = C.c_double
        L.mlr_time_pack.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                    C.c_int64, C.c_uint32, u64p, C.POINTER(C.c_double)]
        L.mlr_time_replay.restype = C.c_double
        L.mlr_time_replay.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_double)]

    @staticmethod
    def _err():
        return C.create_string_buffer(1024)

    def _check(self, rc, err):
        if rc != 0:
            raise RefError(err.value.decode())


class RefEngine:
    """Handle on a reference moelab::Engine (engine.hpp:152)."""

    def __init__(self, ref: Reference, cfg: MlrConfig):
        self.ref, self.cfg = ref, cfg
        err = ref._err()
        self.h = ref.lib.mlr_engine_create(C.byref(cfg), err, 1024)
        if not self.h:
            raise RefError(err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.mlr_engine_destroy(self.h)
            self.h = None

    @property
    def iteration(self) -> int:
        return int(self.ref.lib.mlr_engine_iteration(self.h))

    @property
    def data_seed(self) -> int:
        return int(self.ref.lib.mlr_engine_data_seed(self.h))

    @property
    def op_count(self) -> int:
        return int(self.ref.lib.mlr_engine_op_count(self.h))

    def param_count(self, i: int) -> int:
        return int(self.ref.lib.mlr_engine_param_count(self.h, i))

    def stage_of_op(self, i: int) -> int:
        return int(self.ref.lib.mlr_engine_stage_of_op(self.h, i))

    def run_iteration(self, log=None):
        err = self.ref._err()
        self.ref._check(self.ref.lib.mlr_engine_run_iteration(self.h, log.h if log is not None else None, err, 1024), err)

    def get_op(self, i: int) -> OpState:
        n = int(self.ref.lib.mlr_engine_op_size(self.h, i))
        a = [np.empty(n, dtype=np.float32) for _ in range(4)]
        st = C.c_uint64()
        hf = C.c_int32()
        self.ref.lib.mlr_engine_get_op(self.h, i, *(_ptr(x, f32p) for x in a[:3]), C.byref(st),
                                       _ptr(a[3], f32p), C.byref(hf))
        return OpState(a[0], a[1], a[2], st.value, a[3], bool(hf.value))

    def set_op(self, i: int, master, m, v, step, has_full=True):
        master, m, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (master, m, v))
        self.ref.lib.mlr_engine_set_op(self.h, i, _ptr(master, f32p), _ptr(m, f32p), _ptr(v, f32p),
                                       master.size, step, int(has_full))

    def state(self) -> TrainState:
        return TrainState([self.get_op(i) for i in range(self.op_count)], self.iteration, self.data_seed)

    def serialize_state(self) -> bytes:
        n = self.ref.lib.mlr_engine_serialize_state(self.h, None, 0)
        out = np.empty(n, dtype=np.uint8)
        self.ref.lib.mlr_engine_serialize_state(self.h, _ptr(out, u8p), n)
        return out.tobytes()

    def extract_grads(self) -> list:
        grads = [np.empty(self.param_count(i), dtype=np.float32) for i in range(self.op_count)]
        arr = (f32p * len(grads))(*[_ptr(g, f32p) for g in grads])
        err = self.ref._err()
        self.ref._check(self.ref.lib.mlr_engine_extract_grads(self.h, arr, err, 1024), err)
        return grads

    def schedule(self, wsparse: int, o_active: int):
        n = self.op_count
        ids = np.zeros(wsparse * n, dtype=np.uint32)
        na = np.zeros(wsparse, dtype=np.uint32)
        nc = np.zeros(wsparse, dtype=np.uint32)
        err = self.ref._err()
        self.ref._check(self.ref.lib.mlr_schedule(self.h, wsparse, o_active, _ptr(ids, u32p), _ptr(na, u32p),
                                                  _ptr(nc, u32p), err, 1024), err)
        slots = []
        for k in range(wsparse):
            row = ids[k * n:(k + 1) * n]
            slots.append((list(map(int, row[:na[k]])), list(map(int, row[na[k]:na[k] + nc[k]]))))
        return slots

    def snapshot(self, active, compute_only, slot_index, kind=1, window_start=0, wsparse=1) -> bytes:
        a = np.asarray(active, dtype=np.uint32)
        c = np.asarray(compute_only, dtype=np.uint32)
        err = self.ref._err()
        args = (self.h, _ptr(a, u32p), a.size, _ptr(c, u32p), c.size, slot_index, kind, window_start, wsparse)
        n = self.ref.lib.mlr_snapshot(*args, None, 0, err, 1024)
        if n < 0:
            raise RefError(err.value.decode())
        out = np.empty(n, dtype=np.uint8)
        self.ref.lib.mlr_snapshot(*args, _ptr(out, u8p), n, err, 1024)
        return out.tobytes()

    def dense_checkpoint(self) -> bytes:
        err = self.ref._err()
        n = self.ref.lib.mlr_dense_checkpoint(self.h, None, 0, err, 1024)
        if n < 0:
            raise RefError(err.value.decode())
        out = np.empty(n, dtype=np.uint8)
        self.ref.lib.mlr_dense_checkpoint(self.h, _ptr(out, u8p), n, err, 1024)
        return out.tobytes()


class RefLog:
    """Handle on a reference moelab::UpstreamLog (engine.hpp:63-86)."""

    def __init__(self, ref: Reference):
        self.ref = ref
        self.h = ref.lib.mlr_log_create()

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.mlr_log_destroy(self.h)
            self.h = None

    def __len__(self):
        return int(self.ref.lib.mlr_log_count(self.h))

    def entries(self):
        out = []
        for i in range(len(self)):
            it, mb, b, d = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint8()
            n = self.ref.lib.mlr_log_entry(self.h, i, C.byref(it), C.byref(mb), C.byref(b), C.byref(d), None, 0)
            data = np.empty(n, dtype=np.float32)
            self.ref.lib.mlr_log_entry(self.h, i, C.byref(it), C.byref(mb), C.byref(b), C.byref(d),
                                       _ptr(data, f32p), n)
            out.append(((it.value, mb.value, b.value, d.value), data))
        return out

    def gc(self, persisted_window_start: int):
        self.ref.lib.mlr_gc_logs(self.h, persisted_window_start)

    def at(self, it, mb, boundary, direction):
        err = self.ref._err()
        self.ref._check(self.ref.lib.mlr_log_at(self.h, it, mb, boundary, direction, err, 1024), err)


def ref_convert(ref: Reference, cfg: MlrConfig, window_start: int, wsparse: int, blobs: list) -> bytes:
    arrs = [np.frombuffer(b, dtype=np.uint8) for b in blobs]
    ptrs = (u8p * max(1, len(arrs)))(*[_ptr(a, u8p) for a in arrs])
    sizes = np.array([a.size for a in arrs], dtype=np.uint64)
    err = ref._err()
    args = (C.byref(cfg), window_start, wsparse, ptrs, _ptr(sizes, u64p), len(arrs))
    n = ref.lib.mlr_convert(*args, None, 0, err, 1024)
    if n < 0:
        raise RefError(err.value.decode())
    out = np.empty(n, dtype=np.uint8)
    ref.lib.mlr_convert(*args, _ptr(out, u8p), n, err, 1024)
    return out.tobytes()


def ref_localized_recover(ref: Reference, cfg: MlrConfig, window_start: int, wsparse: int, blobs: list, log,
                          stage_lo: int, stage_hi: int, target: int) -> bytes:
    """localized_recover (recovery.hpp:240-289) through oracle/_ref: the scope
    image (u64 iteration, u32 n, then per op: u32 id, u64 step, u64 P,
    master, m, v)."""
    arrs = [np.frombuffer(b, dtype=np.uint8) for b in blobs]
    ptrs = (u8p * max(1, len(arrs)))(*[_ptr(a, u8p) for a in arrs])
    sizes = np.array([a.size for a in arrs], dtype=np.uint64)
    err = ref._err()
    args = (C.byref(cfg), window_start, wsparse, ptrs, _ptr(sizes, u64p), len(arrs), log.h, stage_lo, stage_hi,
            target)
    n = ref.lib.mlr_localized_recover(*args, None, 0, err, 1024)
    if n < 0:
        raise RefError(err.value.decode())
    out = np.empty(n, dtype=np.uint8)
    ref.lib.mlr_localized_recover(*args, _ptr(out, u8p), n, err, 1024)
    return out.tobytes()


def ref_conversion_plan(ref: Reference, window_start: int, wsparse: int, blobs: list, compute_bytes: int):
    """conversion_plan (recovery.hpp:123-137): [(record_index, replay_iteration, activating ids)]."""
    bufs = [np.frombuffer(bytes(b), dtype=np.uint8) for b in blobs]
    ptrs = (u8p * max(1, len(bufs)))(*[_ptr(b, u8p) for b in bufs])
    sizes = np.array([b.size for b in bufs] or [0], dtype=np.uint64)
    n = max(1, wsparse)
    counts = np.zeros(n, dtype=np.uint64)
    its = np.zeros(n, dtype=np.uint64)
    ids = np.zeros(1 << 16, dtype=np.uint32)
    err = ref._err()
    tot = ref.lib.mlr_conversion_plan(window_start, wsparse, ptrs, _ptr(sizes, u64p), len(bufs), compute_bytes,
                                      _ptr(ids, u32p), ids.size, _ptr(counts, u64p), _ptr(its, u64p), err, 1024)
    if tot < 0:
        raise RefError(err.value.decode())
    out, at = [], 0
    for k in range(wsparse):
        c = int(counts[k])
        out.append((k, int(its[k]), [int(x) for x in ids[at:at + c]]))
        at += c
    return out


def ref_pack_reduced(ref: Reference, x: np.ndarray, ebits: int, mbits: int) -> np.ndarray:
    """pack_reduced (tensor.hpp:127-151) over float32 bits as they are (no
    float -> double round trip: signalling-NaN payloads survive)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.size, dtype=np.uint16)
    ref.lib.mlr_pack_array(_ptr(x, f32p), x.size, ebits, mbits, out.ctypes.data_as(C.POINTER(C.c_uint16)))
    return out


def ref_unpack_reduced(ref: Reference, codes: np.ndarray, ebits: int, mbits: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.uint16)
    out = np.empty(c.size, dtype=np.float32)
    ref.lib.mlr_unpack_array(c.ctypes.data_as(C.POINTER(C.c_uint16)), c.size, ebits, mbits, _ptr(out, f32p))
    return out


def ref_check_log_budget(ref: Reference, cfg: MlrConfig, wsparse: int, cpu_mem_per_node: float, nodes: int):
    err = ref._err()
    ref._check(ref.lib.mlr_check_log_budget(C.byref(cfg), wsparse, cpu_mem_per_node, nodes, err, 1024), err)


def ref_check_coverage(ref: Reference, wsparse: int, blobs: list, op_count: int, compute_bytes: int):
    arrs = [np.frombuffer(b, dtype=np.uint8) for b in blobs]
    ptrs = (u8p * max(1, len(arrs)))(*[_ptr(a, u8p) for a in arrs])
    sizes = np.array([a.size for a in arrs], dtype=np.uint64)
    err = ref._err()
    ref._check(ref.lib.mlr_check_coverage(wsparse, ptrs, _ptr(sizes, u64p), len(arrs), op_count,
                                          compute_bytes, err, 1024), err)


def ref_parse_record(ref: Reference, blob: bytes, compute_bytes: int):
    a = np.frombuffer(blob, dtype=np.uint8)
    it, sl = C.c_uint64(), C.c_uint32()
    err = ref._err()
    n = ref.lib.mlr_parse_record(_ptr(a, u8p), a.size, compute_bytes, C.byref(it), C.byref(sl), err, 1024)
    if n < 0:
        raise RefError(err.value.decode())
    return int(n), it.value, sl.value


def ref_build_schedule(ref: Reference, ops, compute_bytes, master_bytes, optimizer_bytes, bandwidth, t_iter,
                       ordering=0, allow_single=False):
    """build_schedule (schedule.hpp:177-209) of the compiled reference.  ops:
    dicts with cls (0 expert / 1 non-expert / 2 gate), params, hard, soft,
    ema, capacity.  Returns (wsparse, o_active, fits, [(active, compute_only)])."""
    L = ref.lib
    n = len(ops)
    if not getattr(L, "_bs_typed", False):
        f64p = C.POINTER(C.c_double)
        L.mlr_build_schedule.argtypes = [C.c_uint32, u8p, C.POINTER(C.c_int64), f64p, f64p, f64p, f64p, C.c_int64,
                                         C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int64,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32), u32p,
                                         u32p, u32p, C.c_char_p, C.c_size_t]
        L._bs_typed = True
    cls = np.array([o["cls"] for o in ops], dtype=np.uint8)
    params = np.array([o["params"] for o in ops], dtype=np.int64)
    cols = {k: np.array([float(o.get(k, 0.0)) for o in ops], dtype=np.float64)
            for k in ("hard", "soft", "ema", "capacity")}
    max_slots = n
    ids = np.zeros(max_slots * n, dtype=np.uint32)
    na = np.zeros(max_slots, dtype=np.uint32)
    nc = np.zeros(max_slots, dtype=np.uint32)
    w, o, fits = C.c_int64(), C.c_int64(), C.c_int32()
    err = C.create_string_buffer(1024)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = L.mlr_build_schedule(n, cls.ctypes.data_as(u8p), params.ctypes.data_as(C.POINTER(C.c_int64)),
                              dp(cols["hard"]), dp(cols["soft"]), dp(cols["ema"]), dp(cols["capacity"]),
                              compute_bytes, master_bytes, optimizer_bytes, bandwidth, t_iter, ordering,
                              int(allow_single), max_slots, C.byref(w), C.byref(o), C.byref(fits),
                              ids.ctypes.data_as(u32p), na.ctypes.data_as(u32p), nc.ctypes.data_as(u32p), err,
                              len(err))
    if rc != 0:
        msg = err.value.decode()
        raise (ValueError if "invalid" in msg or "non-positive" in msg or "no capacity" in msg
               or "no operators" in msg else RuntimeError)(msg)
    slots = []
    for k in range(w.value):
        row = ids[k * n:(k + 1) * n]
        slots.append((row[:na[k]].tolist(), row[na[k]:na[k] + nc[k]].tolist()))
    return w.value, o.value, bool(fits.value), slots


def load_reference():
    """Reference handle or None when oracle/_ref was not built here."""
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None
