"""Pins the CPU restatement (oracle/moelab_oracle.c) against the reference's
golden vectors (tests/golden, generated from the real reference) and, where
oracle/_ref was built, against the live reference.  CPU only."""
import numpy as np
import pytest

from golden_cases import CASE_NAMES, load_case, load_npz
from oracle.oracle import TrainState, OpState


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


# ---------------------------------------------------------------- codecs
def test_quantize_matches_reference_goldens(oracle):
    g = load_npz("codec")
    xs = g["x"]
    for cb in (1, 2, 4):
        q = oracle.quantize(xs, cb)  # array path: sNaN payloads survive
        # compare bit patterns: NaN payloads and signed zeros must match too
        assert np.array_equal(bits(q), bits(g[f"q{cb}"])), cb


def test_quantize_pins(oracle):
    # test_tensor.cpp:37-41
    assert oracle.quantize_value(0.1, 2) == np.float32(0.0999755859375)
    with pytest.raises(ValueError):
        oracle.quantize_value(1.0, 3)  # test_tensor.cpp:66-68


def test_pack_unpack_match_goldens(oracle):
    g = load_npz("codec")
    p16 = np.array([oracle.pack_reduced(float(v), 5, 10) for v in g["q2"]], dtype=np.uint16)
    p8 = np.array([oracle.pack_reduced(float(v), 4, 3) for v in g["q1"]], dtype=np.uint16)
    assert np.array_equal(p16, g["pack16"])
    assert np.array_equal(p8, g["pack8"])
    assert p8.max() <= 0xff  # test_tensor.cpp:79
    # array decode (read_compute): sNaN payloads survive, unlike a ctypes float return
    u16 = oracle.decode_compute(np.arange(65536, dtype=np.uint16).tobytes(), 65536, 2)
    assert np.array_equal(bits(u16), bits(g["unpack16"]))
    u8 = oracle.decode_compute(np.arange(256, dtype=np.uint8).tobytes(), 256, 1)
    assert np.array_equal(bits(u8), bits(g["unpack8"]))


# ---------------------------------------------------------------- fnv
def test_fnv_matches_goldens(oracle):
    g = load_npz("fnv")
    i = 0
    while f"data{i}" in g:
        assert oracle.fnv1a64(g[f"data{i}"]) == int(g[f"hash{i}"][0])
        i += 1
    assert oracle.fnv1a64(b"") == 0xcbf29ce484222325


# ---------------------------------------------------------------- adam
def test_adam_matches_goldens(oracle):
    g = load_npz("adam")
    w, m, v = g["w0"].copy(), g["m0"].copy(), g["v0"].copy()
    step = int(g["step0"][0])
    for s in range(5):
        step = oracle.adam_step(w, m, v, step, g[f"g{s}"])
        assert np.array_equal(bits(w), bits(g[f"w{s + 1}"]))
        assert np.array_equal(bits(m), bits(g[f"m{s + 1}"]))
        assert np.array_equal(bits(v), bits(g[f"v{s + 1}"]))
    assert step == 8


def test_adam_pins(oracle):
    # test_engine.cpp:213-246
    w, m, v = (np.array([x], dtype=np.float32) for x in (1.0, 0.0, 0.0))
    st = oracle.adam_step(w, m, v, 0, np.zeros(1, np.float32))
    assert (w[0], m[0], v[0], st) == (1.0, 0.0, 0.0, 1)
    w, m, v = (np.array([x], dtype=np.float32) for x in (1.0, 0.0, 0.0))
    oracle.adam_step(w, m, v, 0, np.ones(1, np.float32))
    assert abs(float(w[0]) - (1.0 - 0.001)) <= 1e-7


# ---------------------------------------------------------------- container
@pytest.mark.parametrize("name", CASE_NAMES)
def test_serialize_record_matches_reference(oracle, name):
    c = load_case(name)
    for s in range(c.T + 1):
        blob = oracle.serialize_record(c.header(s), c.record_entries(s), c.compute_bytes)
        assert blob == c.blob(s), (name, s)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_parse_record_roundtrip(oracle, name):
    c = load_case(name)
    for s in range(c.T + 1):
        blob = c.blob(s)
        h, ents = oracle.parse_record(blob, c.compute_bytes)
        assert h == c.header(s)
        want = c.record_entries(s)
        assert [(e["id"], e["mode"], e["param_count"]) for e in ents] == \
               [(e["id"], e["mode"], e["param_count"]) for e in want]


def test_parse_errors(oracle):
    c = load_case("six_op_cb4")
    blob = bytearray(c.blob(1))
    blob[len(blob) // 2] ^= 0x40  # test_snapshot.cpp:139-142
    with pytest.raises(RuntimeError, match="checksum"):
        oracle.parse_record(bytes(blob), 4)
    with pytest.raises(RuntimeError, match="truncated"):
        oracle.parse_record(b"\x00" * 5, 4)
    # bad magic with a valid trailer
    body = b"XXXX" + c.blob(1)[4:-8]
    bad = body + oracle.fnv1a64(body).to_bytes(8, "little")
    with pytest.raises(RuntimeError, match="bad magic"):
        oracle.parse_record(bad, 4)
    body = c.blob(1)[:4] + (7).to_bytes(4, "little") + c.blob(1)[8:-8]
    bad = body + oracle.fnv1a64(body).to_bytes(8, "little")
    with pytest.raises(RuntimeError, match="unsupported version 7"):
        oracle.parse_record(bad, 4)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_serialize_state_matches_reference(oracle, name):
    c = load_case(name)
    for s in range(c.T + 1):
        st = TrainState([OpState(**{k: v for k, v in c.op(s, i).items() if k != "compute"})
                         for i in range(c.n_ops)], s, c.data_seed)
        assert oracle.serialize_state(st) == c.mlst(s)


def oracle_convert(oracle, c, w) -> bytes:
    """Merge + logged-gradient Adam replay == sparse_to_dense_convert."""
    W = c.W
    full_slot = {}
    for k in range(W):
        for i in c.slot(k)[0]:
            full_slot[i] = k
    ops = []
    opt = c.optimizer
    for i in range(c.n_ops):
        k = full_slot[i]
        o = c.op(w + k, i)
        master, m, v = o["master"].copy(), o["m"].copy(), o["v"].copy()
        if W > 1:
            grads = np.stack([c.grads(w + j + 1, i) for j in range(k, W)]) if k < W else None
            step = oracle.replay_op(master, m, v, o["step"], grads, opt["kind"], opt["lr"], opt["beta1"],
                                    opt["beta2"], opt["eps"])
        else:
            step = o["step"]
        ops.append(OpState(master, m, v, step))
    it = w + W if W > 1 else w
    return oracle.serialize_state(TrainState(ops, it, c.data_seed))


@pytest.mark.parametrize("name", CASE_NAMES)
def test_merge_replay_equals_reference_conversion(oracle, name):
    c = load_case(name)
    assert c.meta["converted_windows"]
    for w in c.meta["converted_windows"]:
        assert oracle_convert(oracle, c, w) == c.converted(w), (name, w)
        # and the conversion equals the uninterrupted run (test_recovery.cpp:77-90)
        it = w + c.W if c.W > 1 else w
        assert c.converted(w) == c.mlst(it)


@pytest.mark.parametrize("name", ["verify_toy", "dp2_pp2"])
def test_localized_replay_equals_reference_localized_recovery(oracle, name):
    """The logged-gradient restatement of localized_recover (recovery.hpp:
    240-289): each scope operator's Full payload of the window, stepped with
    optimizer_step_adam on the gradients of iterations a+k+1 .. max(a+W,
    target), equals the reference's localized recovery -- which itself equals
    the uninterrupted run at the target (test_recovery.cpp:190-284)."""
    c = load_case(name)
    opt = c.optimizer
    assert c.localized()
    for (w, target, lo, hi) in c.localized():
        it, ref = c.localized_image(w, target, lo, hi)
        assert it == target
        end = max(w + c.W, target)
        for i in c.scope(lo, hi):
            k = next(k for k in range(c.W) if i in c.slot(k)[0])
            o = c.op(w + k, i)
            master, m, v = o["master"].copy(), o["m"].copy(), o["v"].copy()
            grads = np.stack([c.grads(j, i) for j in range(w + k + 1, end + 1)])
            step = oracle.replay_op(master, m, v, o["step"], grads, opt["kind"], opt["lr"], opt["beta1"],
                                    opt["beta2"], opt["eps"])
            rs, rmaster, rm, rv = ref[i]
            assert step == rs
            for a, b in ((master, rmaster), (m, rm), (v, rv)):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (name, w, target, lo, hi, i)
            tgt = c.op(target, i)
            assert np.array_equal(rmaster.view(np.uint32), tgt["master"].view(np.uint32))


def test_live_reference_localized_recovery(reference):
    """The committed localized-recovery goldens reproduce from oracle/_ref."""
    from oracle.oracle import RefEngine, RefLog, ref_localized_recover, toy_config
    c = load_case("verify_toy")
    cfg = toy_config(layers=3, stages=3, seed=1)
    e = RefEngine(reference, cfg)
    log = RefLog(reference)
    windows = {}
    slots = e.schedule(c.W, c.meta["O"])
    while True:
        s = e.iteration
        w, k = s // c.W * c.W, s % c.W
        windows.setdefault(w, []).append(e.snapshot(slots[k][0], slots[k][1], k, 1, w, c.W))
        if s == c.T:
            break
        e.run_iteration(log)
    w, target, lo, hi = c.localized()[-1]
    img = ref_localized_recover(reference, cfg, w, c.W, windows[w], log, lo, hi, target)
    assert img == c.d[f"loc_w{w}_t{target}_s{lo}_{hi}"].tobytes()


# ---------------------------------------------------------------- live reference
def test_live_reference_random_blobs(oracle, reference):
    """Random states through both serialize paths at odd sizes and widths."""
    from oracle.oracle import RefEngine, toy_config
    rng = np.random.default_rng(3)
    for cb in (1, 2, 4):
        cfg = toy_config(layers=1, stages=1, seed=4, compute_bytes=cb, expert_params=37,
                         nonexpert_params=101, gate_params=5)
        e = RefEngine(reference, cfg)
        for i in range(e.op_count):
            n = int(rng.integers(1, 300))
            e.set_op(i, rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32),
                     rng.uniform(0, 1, n).astype(np.float32), int(rng.integers(0, 100)))
        active, co = [0, 3], [1, 2, 4, 5]
        blob = e.snapshot(active, co, 1, 1, 10, 3)
        ents = []
        for i in sorted(active + co):
            o = e.get_op(i)
            if i in active:
                ents.append(dict(id=i, mode=0, param_count=o.master.size, step=o.step, master=o.master, m=o.m,
                                 v=o.v))
            else:
                ents.append(dict(id=i, mode=1, param_count=o.compute.size, compute=o.compute))
        hdr = dict(kind=1, iteration=e.iteration, window_start=10, wsparse=3, slot=1, data_seed=e.data_seed)
        assert oracle.serialize_record(hdr, ents, cb) == blob


def test_live_reference_errors(reference):
    from oracle.oracle import RefEngine, RefError, toy_config, ref_parse_record
    e = RefEngine(reference, toy_config())
    with pytest.raises(RefError, match="unknown operator"):  # test_snapshot.cpp:198-204
        e.snapshot([42], [], 0)
    blob = bytearray(e.snapshot([0, 1], [2, 3, 4, 5], 0))
    blob[len(blob) // 2] ^= 0x40
    with pytest.raises(RefError, match="checksum"):
        ref_parse_record(reference, bytes(blob), 2)
