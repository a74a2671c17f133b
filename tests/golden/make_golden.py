"""Generate the committed golden vectors from the REAL reference.

Run here (where /root/reference exists and oracle/_ref was built):
    make -C oracle && python tests/golden/make_golden.py

Each case drives the unmodified reference through oracle/_ref exactly like
the reference's own harnesses do (TrainRun, test_recovery.cpp:34-67;
capture_windows, verify.hpp:63-84): record state 0, then after every
iteration take the slot (s mod W) record into window floor(s/W)*W.  It stores
for every state s: the MLST dense image (engine.hpp:246-261), every operator's
master/m/v/step/compute, the serialized record (snapshot.hpp:115-144), the
gradients of iteration s+1 (extracted through the public API: beta1=0, lr=0
probe), the conversion result of every complete window
(recovery.hpp:180-227), and the upstream log (engine.hpp:381-411) when the
case logs.  The GPU parity tests read only these files (the GPU box has no
/root/reference).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import (Reference, RefEngine, RefLog, ref_convert, ref_localized_recover,  # noqa: E402
                           toy_config)

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # verify_toy.json shape (3 layers x 4 experts, 3 stages), W=3, O=ceil(18/3)
    "verify_toy": dict(cfg=dict(layers=3, stages=3, seed=1), W=3, O=6, T=9, log=True),
    # six_op_config (test_snapshot.cpp:13-34), Fig.5 slots, compute widths 1/4
    "six_op_cb1": dict(cfg=dict(layers=1, stages=1, seed=9, compute_bytes=1), W=3, O=2, T=6, log=False),
    "six_op_cb4": dict(cfg=dict(layers=1, stages=1, seed=9, compute_bytes=4), W=3, O=2, T=6, log=False),
    # SGD branch of apply_updates (engine.hpp:710-713)
    "toy_sgd": dict(cfg=dict(layers=1, stages=1, seed=5, optimizer_kind=1), W=3, O=2, T=6, log=False),
    # degenerate single-slot window (test_recovery.cpp:104-112)
    "w1": dict(cfg=dict(layers=1, stages=1, seed=5), W=1, O=6, T=4, log=False),
    # two data-parallel pipelines x 2 stages: replica-major micro-batch ids in the log
    "dp2_pp2": dict(cfg=dict(layers=2, stages=2, seed=3, dp=2, microbatches=2, mb_size=3), W=2, O=6, T=4,
                    log=True),
}


def capture(ref: Reference, name: str, spec: dict) -> dict:
    cfg = toy_config(**spec["cfg"])
    eng = RefEngine(ref, cfg)
    W, O, T = spec["W"], spec["O"], spec["T"]
    slots = eng.schedule(W, O)
    log = RefLog(ref) if spec["log"] else None
    d: dict = {}
    n_ops = eng.op_count
    windows: dict = {}

    def record():
        s = eng.iteration
        w, k = s // W * W, s % W
        blob = eng.snapshot(slots[k][0], slots[k][1], k, 1, w, W)
        windows.setdefault(w, []).append(blob)
        d[f"s{s}_blob"] = np.frombuffer(blob, dtype=np.uint8)
        d[f"s{s}_mlst"] = np.frombuffer(eng.serialize_state(), dtype=np.uint8)
        for i in range(n_ops):
            op = eng.get_op(i)
            d[f"s{s}_op{i}_master"] = op.master
            d[f"s{s}_op{i}_m"] = op.m
            d[f"s{s}_op{i}_v"] = op.v
            d[f"s{s}_op{i}_compute"] = op.compute
            d[f"s{s}_op{i}_step"] = np.array([op.step], dtype=np.uint64)
        if s < T:
            for i, g in enumerate(eng.extract_grads()):
                d[f"g{s + 1}_op{i}"] = g  # gradient applied by iteration s+1

    record()
    d["dense_s0"] = np.frombuffer(eng.dense_checkpoint(), dtype=np.uint8)
    while eng.iteration < T:
        eng.run_iteration(log)
        record()
    d[f"dense_s{T}"] = np.frombuffer(eng.dense_checkpoint(), dtype=np.uint8)

    converted = []
    for w, blobs in sorted(windows.items()):
        if len(blobs) == W:
            st = ref_convert(ref, cfg, w, W, blobs)
            d[f"conv_w{w}"] = np.frombuffer(st, dtype=np.uint8)
            converted.append(w)

    localized = []
    if log is not None:
        # localized recovery (recovery.hpp:240-289) of every stage (and the
        # trailing stage pair) from every complete window, to the window's end
        # and to the last logged iteration (lost-iteration catch-up)
        stages = spec["cfg"].get("stages", 1)
        ranges = [(s_, s_) for s_ in range(stages)] + ([(1, stages - 1)] if stages > 2 else [])
        for w in converted:
            for target in sorted({w + W, T}):
                for lo, hi in ranges:
                    img = ref_localized_recover(ref, cfg, w, W, windows[w], log, lo, hi, target)
                    d[f"loc_w{w}_t{target}_s{lo}_{hi}"] = np.frombuffer(img, dtype=np.uint8)
                    localized.append([w, target, lo, hi])
        ents = log.entries()
        d["log_keys"] = np.array([k for k, _ in ents], dtype=np.uint64).reshape(-1, 4)
        for j, (_, data) in enumerate(ents):
            d[f"log_{j}"] = data

    meta = dict(
        name=name, cfg={f: getattr(cfg, f) for f, _ in cfg._fields_}, W=W, O=O, T=T,
        n_ops=n_ops, param_counts=[eng.param_count(i) for i in range(n_ops)],
        stage_of_op=[eng.stage_of_op(i) for i in range(n_ops)],
        slots=slots, data_seed=eng.data_seed, converted_windows=converted,
        log=bool(spec["log"]), localized=localized,
    )
    return meta, d


def codec_vectors(ref: Reference) -> dict:
    """pack_reduced/quantize goldens incl. NaN, inf, subnormal, saturation."""
    import ctypes as C
    rng = np.random.default_rng(7)
    xs = np.concatenate([
        rng.uniform(-8, 8, 4000).astype(np.float32),
        rng.standard_normal(2000).astype(np.float32) * np.float32(1e-5),
        rng.standard_normal(1000).astype(np.float32) * np.float32(1e5),
        np.array([0.0, -0.0, 0.1, 65504.0, 65520.0, 65519.99, 1e6, -1e6, 240.0, 248.0, 232.0, 3e-7,
                  2.0 ** -24, 2.0 ** -25, 2.0 ** -26, 1.5 * 2.0 ** -24, 2.0 ** -9, 2.0 ** -10, 1e-45,
                  np.inf, -np.inf], dtype=np.float32),
        np.array([np.nan], dtype=np.float32),
        np.frombuffer(np.array([0xffc00001, 0x7f800001, 0x00000001, 0x80400000], dtype=np.uint32).tobytes(),
                      dtype=np.float32),
    ]).astype(np.float32)
    out = {"x": xs}
    fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
    for cb in (1, 2, 4):
        # array entry point: no float->double->float trip that would quiet sNaNs
        q = np.empty_like(xs)
        ref.lib.mlr_quantize_array(fp(xs), xs.size, cb, fp(q), None, 0)
        out[f"q{cb}"] = q
    out["pack16"] = np.array([ref.lib.mlr_pack_reduced(C.c_float(v), 5, 10) for v in out["q2"]], dtype=np.uint16)
    out["pack8"] = np.array([ref.lib.mlr_pack_reduced(C.c_float(v), 4, 3) for v in out["q1"]], dtype=np.uint16)
    up = ref.lib.mlr_unpack_array
    up.argtypes = [C.POINTER(C.c_uint16), C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_float)]
    for name, n, e, m in (("unpack16", 65536, 5, 10), ("unpack8", 256, 4, 3)):
        codes = np.arange(n, dtype=np.uint16)
        vals = np.empty(n, dtype=np.float32)
        up(codes.ctypes.data_as(C.POINTER(C.c_uint16)), n, e, m, fp(vals))  # sNaN-exact
        out[name] = vals
    return out


def fnv_vectors(ref: Reference) -> dict:
    rng = np.random.default_rng(11)
    out = {}
    sizes = [0, 1, 7, 8, 15, 16, 17, 31, 32, 33, 255, 1000, 4096, 65537, 300001]
    for i, n in enumerate(sizes):
        a = rng.integers(0, 256, n, dtype=np.uint8)
        out[f"data{i}"] = a
        out[f"hash{i}"] = np.array([ref.lib.mlr_fnv1a64(a.ctypes.data_as(__import__('ctypes').POINTER(
            __import__('ctypes').c_uint8)), n, 0xcbf29ce484222325)], dtype=np.uint64)
    return out


def adam_vectors(ref: Reference) -> dict:
    import ctypes as C
    rng = np.random.default_rng(5)
    n = 4096
    out = {}
    w = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = (rng.uniform(0, 1e-6, n)).astype(np.float32)
    out["w0"], out["m0"], out["v0"] = w.copy(), m.copy(), v.copy()
    step = C.c_uint64(3)
    f = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
    for s in range(5):
        g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        g[:8] = [0.0, -0.0, 1.0, -1.0, 1e-30, 3e-38, 1e30, -1e-20]
        out[f"g{s}"] = g
        ref.lib.mlr_optimizer_step_adam(f(w), f(m), f(v), C.byref(step), f(g), n, 1e-3, 0.9, 0.999, 1e-8,
                                        None, 0)
        out[f"w{s + 1}"], out[f"m{s + 1}"], out[f"v{s + 1}"] = w.copy(), m.copy(), v.copy()
    out["step0"] = np.array([3], dtype=np.uint64)
    return out


def main():
    ref = Reference()
    manifest = {"cases": {}, "files": {}}
    for name, spec in CASES.items():
        meta, d = capture(ref, name, spec)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **d)
        manifest["cases"][name] = meta
    for name, fn in (("codec", codec_vectors), ("fnv", fnv_vectors), ("adam", adam_vectors)):
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **fn(ref))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            with open(os.path.join(OUT, f), "rb") as fh:
                manifest["files"][f] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("wrote", sorted(manifest["files"]))


if __name__ == "__main__":
    main()
