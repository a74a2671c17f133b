"""GPU parity at the BASELINE.json shapes, not only at golden
sizes:

  configs[0]  8 experts x 2^21 (+ NE, G), W=5, O=2: every record of a window
              and the converted dense state against the REAL reference
              (oracle/_ref) running the same state;
  configs[1]  the DeepSeek-MoE layer's slot-0 record (2,040,228,799 B) and
  configs[2]  a Mixtral EP shard's slot-0 record (16 x 176,160,768 params,
              12.7 GB: offsets past 2^32) byte for byte against the oracle's
              serialize_record layout, streamed in pieces, plus the trailer
              against the oracle's FNV chained over the pieces;
  configs[3]  a W=6 window of full-size operators (4 experts of 7,898,100,
              the NE block of 80,140,000, the gate) converted, and localized
              recovery with 3 lost iterations: every master/m/v bit against
              the oracle's Adam trajectory of the same synthetic run;
  configs[4]  one iteration of an interior stage's [4096 x 2048] f32
              boundary entries through both log kinds, byte-exact.
"""
import numpy as np
import pytest

from oracle.oracle import RefEngine, ref_convert, toy_config

pytestmark = pytest.mark.gpu

PIECE = 1 << 26  # floats per generated piece (256 MiB)


@pytest.fixture(scope="module")
def mk():
    from paper_2412_15411_b200 import mlck
    return mlck


@pytest.fixture(scope="module")
def ctx(mk):
    c = mk.Context(0)
    yield c
    c.close()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def schedule(ordered, W, O):
    """generate_schedule (schedule.hpp:153-172)."""
    n = len(ordered)
    return [(ordered[k * O:min((k + 1) * O, n)], ordered[min((k + 1) * O, n):]) for k in range(W)]


class RecordCheck:
    """Streams the expected MLCK v1 bytes (snapshot.hpp:120-142) of a record
    of a synthetic state (mlck_state_fill_synthetic == the oracle's synth
    streams 3i, 3i+1, 3i+2) and compares them with the device record piece by
    piece; the FNV-1a-64 trailer is chained over the same pieces."""

    def __init__(self, ctx, oracle, blob, cb):
        self.ctx, self.o, self.cb = ctx, oracle, cb
        self.ptr, self.size = blob.device_ptr, blob.size
        self.pos, self.h = 0, 0xcbf29ce484222325

    def put(self, data: bytes):
        got = self.ctx.download(self.ptr + self.pos, len(data))
        assert got == data, f"record bytes differ in [{self.pos}, {self.pos + len(data)})"
        self.h = self.o.fnv1a64(np.frombuffer(data, np.uint8), seed=self.h)
        self.pos += len(data)

    def finish(self):
        assert self.size == self.pos + 8
        assert self.ctx.download(self.ptr + self.pos, 8) == self.h.to_bytes(8, "little"), "trailer"


def check_synthetic_record(ctx, oracle, blob, pcs, slot, slot_index, iteration, window_start, W, seed, step, cb,
                           data_seed):
    import struct
    active, co = slot
    ents = sorted([(i, 0) for i in active] + [(i, 1) for i in co])
    rc = RecordCheck(ctx, oracle, blob, cb)
    rc.put(struct.pack("<IIBQQIIQI", 0x4B434C4D, 1, 1, iteration, window_start, W, slot_index, data_seed,
                       len(ents)))
    for i, mode in ents:
        P = pcs[i]
        rc.put(struct.pack("<IBQ", i, mode, P) + (struct.pack("<Q", step) if mode == 0 else b""))
        if mode == 0:
            for stream, lo, hi in ((3 * i, -0.25, 0.25), (3 * i + 1, -1e-3, 1e-3), (3 * i + 2, 0.0, 1e-6)):
                for f in range(0, P, PIECE):
                    rc.put(oracle.synth(seed, stream, lo, hi, min(PIECE, P - f), first=f).tobytes())
        else:
            for f in range(0, P, PIECE):
                m = oracle.synth(seed, 3 * i, -0.25, 0.25, min(PIECE, P - f), first=f)
                rc.put(oracle.encode_compute(oracle.quantize(m, cb), cb))
    rc.finish()


# ---------------------------------------------------------------- configs[1], configs[2]
@pytest.mark.parametrize("workload", ["deepseek_moe_layer", "mixtral_8x7b_ep"])
def test_full_size_slot0_record_vs_oracle(mk, ctx, oracle, workload):
    if workload == "deepseek_moe_layer":
        pcs = [7_898_100] * 64 + [80_140_000, 100_000]
        W, O = 6, 11
    else:
        pcs = [176_160_768] * 16
        W, O = 4, 4
    cb = 2
    slots = schedule(list(range(len(pcs))), W, O)
    st = mk.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=21, step=10)
    st.set_meta(1000, 7)
    blob = mk.snapshot_record(st, *slots[0], 0, 1, 1000, W)
    want = 45 + 8 + sum(13 + 8 + 12 * pcs[i] for i in slots[0][0]) + sum(13 + cb * pcs[i] for i in slots[0][1])
    assert blob.size == want
    if workload == "deepseek_moe_layer":
        assert blob.size == 2_040_228_799  # SURVEY 8(d) slot-0 size
    else:
        assert blob.size > 1 << 32
    check_synthetic_record(ctx, oracle, blob, pcs, slots[0], 0, 1000, 1000, W, 21, 10, cb, 7)
    blob.close()
    st.close()


# ---------------------------------------------------------------- configs[3]
def host_trajectory(oracle, P, i, seed, gseed, n_ops, first_it, n_it, step0):
    """The oracle's Adam steps of operator i over iterations first_it ..
    first_it + n_it - 1 from its synthetic start (mlo_adam_step, the
    reference's arithmetic, engine.hpp:738-753)."""
    w = oracle.synth(seed, 3 * i, -0.25, 0.25, P)
    m = oracle.synth(seed, 3 * i + 1, -1e-3, 1e-3, P)
    v = oracle.synth(seed, 3 * i + 2, 0.0, 1e-6, P)
    step = step0
    for it in range(first_it, first_it + n_it):
        g = oracle.synth(gseed, 1_000_000 + it * n_ops + i, -1e-2, 1e-2, P)
        step = oracle.adam_step(w, m, v, step, g)
    return w, m, v, step


def test_full_size_window_conversion_and_localized_recovery(mk, ctx, oracle):
    """A W=6 window of full-size configs[3] operators, captured from a device
    training run (apply_updates on logged gradients), converted and
    localized-recovered; the result equals the oracle's uninterrupted run."""
    pcs = [7_898_100] * 4 + [80_140_000, 100_000]
    n, W, a, seed, gseed, extra = len(pcs), 6, 1000, 31, 41, 3
    slots = schedule(list(range(n)), W, 1)  # op k is Full in slot k: W-k replay steps
    st = mk.DeviceState(ctx, pcs, 2)
    st.fill_synthetic(seed=seed, step=10)
    g = mk.GradLog(ctx, pcs, W + extra)
    g.fill_synthetic(a + 1, W + extra, seed=gseed)
    blobs = []
    for k in range(W):  # capture_windows: record of state a+k, then train iteration a+k+1
        st.set_meta(a + k, 7)
        blobs.append(mk.snapshot_record(st, *slots[k], k, 1, a, W))
        st.apply_updates(range(n), g, a + k + 1)
    out = mk.DeviceState(ctx, pcs, 2)
    mk.sparse_to_dense_convert(out, blobs, a, W, 7, g)
    assert out.meta() == (a + W, 7)
    for i in range(n):
        w, m, v, step = host_trajectory(oracle, pcs[i], i, seed, gseed, n, a + 1, W, 10)
        got = out.download_op(i)
        assert got.step == step == 10 + W
        for x, y in ((got.master, w), (got.m, m), (got.v, v)):
            assert np.array_equal(bits(x), bits(y)), i
        assert np.array_equal(bits(got.compute), bits(oracle.quantize(w, 2))), i
    # localized recovery of a scope, 3 lost iterations past the window
    scope = [1, 3, 4]
    rec = mk.DeviceState(ctx, pcs, 2)
    mk.localized_recover(rec, scope, blobs, a, W, 7, g, a + W + extra)
    for i in scope:
        w, m, v, step = host_trajectory(oracle, pcs[i], i, seed, gseed, n, a + 1, W + extra, 10)
        got = rec.download_op(i)
        assert got.step == step
        for x, y in ((got.master, w), (got.m, m), (got.v, v)):
            assert np.array_equal(bits(x), bits(y)), i
    for b in blobs:
        b.close()


@pytest.mark.parametrize("seed", range(8))
def test_random_windows_conversion_and_recovery(mk, ctx, oracle, seed):
    """Random windows at small sizes: 2-20 operators of 1 to 200K parameters
    (odd sizes: the replay's 4-element units end mid-unit), W = 1-8 (W = 1 is
    the reference's degenerate window: no replay), compute width 1/2/4, 0-3
    lost iterations past the window and a random scope; conversion and
    localized recovery against the oracle's Adam trajectory, bit for bit."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 21))
    W = int(rng.integers(1, 9))
    O = -(-n // W)  # every operator Full in exactly one slot
    pcs = [int(rng.choice([rng.integers(1, 11), rng.integers(100, 5000), rng.integers(100_000, 200_000)]))
           for _ in range(n)]
    cb = int(rng.choice([1, 2, 4]))
    a, sseed, gseed, extra = int(rng.integers(0, 10_000)), 60 + seed, 70 + seed, int(rng.integers(0, 4))
    order = [int(x) for x in rng.permutation(n)]
    slots = schedule(order, W, O)
    st = mk.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=sseed, step=3)
    g = mk.GradLog(ctx, pcs, W + extra)
    g.fill_synthetic(a + 1, W + extra, seed=gseed)
    blobs = []
    for k in range(W):
        st.set_meta(a + k, 5)
        blobs.append(mk.snapshot_record(st, *slots[k], k, 1, a, W))
        st.apply_updates(range(n), g, a + k + 1)
    out = mk.DeviceState(ctx, pcs, cb)
    mk.sparse_to_dense_convert(out, blobs, a, W, 5, g)
    # W = 1: the single record already is the dense checkpoint (recovery.hpp:192-201)
    n_conv = 0 if W == 1 else W
    assert out.meta() == (a + n_conv, 5)
    for i in range(n):
        w, m, v, step = host_trajectory(oracle, pcs[i], i, sseed, gseed, n, a + 1, n_conv, 3)
        got = out.download_op(i)
        assert got.step == step, (seed, i)
        for x, y in ((got.master, w), (got.m, m), (got.v, v)):
            assert np.array_equal(bits(x), bits(y)), (seed, i)
        assert np.array_equal(bits(got.compute), bits(oracle.quantize(w, cb))), (seed, i)
    scope = sorted(int(x) for x in rng.choice(n, int(rng.integers(1, n + 1)), replace=False))
    rec = mk.DeviceState(ctx, pcs, cb)
    mk.localized_recover(rec, scope, blobs, a, W, 5, g, a + W + extra)
    for i in scope:
        w, m, v, step = host_trajectory(oracle, pcs[i], i, sseed, gseed, n, a + 1, W + extra, 3)
        got = rec.download_op(i)
        assert got.step == step, (seed, i)
        for x, y in ((got.master, w), (got.m, m), (got.v, v)):
            assert np.array_equal(bits(x), bits(y)), (seed, i)
    for b in blobs:
        b.close()
    for x in (st, out, rec, g):
        x.close()


# ---------------------------------------------------------------- configs[0]
def test_configs0_window_against_the_reference(mk, ctx, reference):
    """configs[0]: 8 experts + NE + G at 2^21 params each, W=5, O=2, the
    reference's own engine (oracle/_ref): its records and conversion vs ours
    on the same states and gradients."""
    P = 1 << 21
    cfg = toy_config(layers=1, experts=8, top_k=2, expert_params=P, nonexpert_params=P, gate_params=P, seed=3)
    eng = RefEngine(reference, cfg)
    n = eng.op_count
    W, O = 5, 2
    slots = schedule(list(range(n)), W, O)
    g = mk.GradLog(ctx, [P] * n, W)
    blobs, raw = [], []
    for k in range(W):
        state = eng.state()
        st = mk.DeviceState(ctx, [P] * n, 2)
        for i, op in enumerate(state.ops):
            st.upload_op(i, op.master, op.m, op.v, op.step)
        st.set_meta(eng.iteration, eng.data_seed)
        want = eng.snapshot(*slots[k], k, 1, 0, W)
        b = mk.snapshot_record(st, *slots[k], k, 1, 0, W)
        got = b.to_host()
        assert len(got) == len(want) and got == want, k
        blobs.append(b)
        raw.append(want)
        for i, gr in enumerate(eng.extract_grads()):  # the iteration's weight gradients
            g.put(eng.iteration + 1, i, gr)
        eng.run_iteration()
        st.close()
    out = mk.DeviceState(ctx, [P] * n, 2)
    mk.sparse_to_dense_convert(out, blobs, 0, W, eng.data_seed, g)
    assert out.serialize_state() == ref_convert(reference, cfg, 0, W, raw)


# ---------------------------------------------------------------- configs[4]
@pytest.mark.parametrize("kind", [0, 1])
def test_configs4_boundary_entries(mk, ctx, kind):
    """One iteration of an interior stage (dp2 x pp4, M=8): 8 fwd + 8 bwd
    entries of [4096 x 2048] f32 (33,554,432 B), byte-exact back."""
    n = 4096 * 2048
    rng = np.random.default_rng(kind)
    log = mk.UpstreamLog(ctx, 16 * 4 * n + (1 << 20), kind=kind, device=0)
    datas, ptrs = [], []
    for j in range(16):
        a = rng.standard_normal(n).astype(np.float32)
        datas.append(a)
        ptrs.append(ctx.upload(a))
    for mb in range(8):
        log.put(7, mb, 1, 0, ptrs[2 * mb], n)
        log.put(7, mb, 1, 1, ptrs[2 * mb + 1], n)
    log.sync()
    assert len(log) == 16 and log.bytes() == 16 * 4 * n
    for mb in range(8):
        assert log.at(7, mb, 1, 0).tobytes() == datas[2 * mb].tobytes()
        assert log.at(7, mb, 1, 1).tobytes() == datas[2 * mb + 1].tobytes()
    for p in ptrs:
        ctx.free(p)
    log.close()
