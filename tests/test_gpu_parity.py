"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bit-exact everywhere (Adam tolerance: 0
ulp, asserted on raw bits)."""
import numpy as np
import pytest

from golden_cases import CASE_NAMES, load_case, load_npz

pytestmark = pytest.mark.gpu


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


def upload_state(mk, ctx, c, s):
    st = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    for i in range(c.n_ops):
        o = c.op(s, i)
        st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
    st.set_meta(s, c.data_seed)
    return st


# ---------------------------------------------------------------- FNV (K2)
def test_fnv_goldens(mk, ctx):
    g = load_npz("fnv")
    i = 0
    while f"data{i}" in g:
        data = g[f"data{i}"]
        ptr = ctx.upload(data) if data.size else ctx.alloc(16)
        assert ctx.fnv1a64(ptr, data.size) == int(g[f"hash{i}"][0]), data.size
        ctx.free(ptr)
        i += 1


# sizes around the kernel's units: a 128-byte row (one thread), a 256-row TMA
# box, a 64 KiB chunk, a wave of 3 x 148 chunks
@pytest.mark.parametrize("n", [127, 128, 129, 255, 256, 32767, 32768, 32769, 65535, 65536, 65537, 131200,
                               444 * 65536, 444 * 65536 + 5, 16383, 16384, 16385, 1 << 20, 5 * (1 << 20) + 77,
                               64 * (1 << 20) + 13])
def test_fnv_large_vs_oracle(mk, ctx, oracle, n):
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, n, dtype=np.uint8)
    # long runs of equal bytes exercise the carry chain differently
    data[n // 3: n // 3 + 5000] = 0xff
    data[n // 2: n // 2 + 5000] = 0
    ptr = ctx.upload(data)
    try:
        assert ctx.fnv1a64(ptr, n) == oracle.fnv1a64(data)
        # unaligned start (parse of a sub-range)
        assert ctx.fnv1a64(ptr + 3, n - 3) == oracle.fnv1a64(data[3:])
        # 16-byte aligned sub-range: the tensor-map path on another base
        assert ctx.fnv1a64(ptr + 16, n - 16) == oracle.fnv1a64(data[16:])
        assert ctx.fnv1a64(ptr, n, seed=12345) == oracle.fnv1a64(data, seed=12345)
    finally:
        ctx.free(ptr)


# ---------------------------------------------------------------- codecs
def test_codec_goldens(mk, ctx):
    g = load_npz("codec")
    x = np.ascontiguousarray(g["x"], dtype=np.float32)
    dx = ctx.upload(x)
    out = ctx.alloc(x.nbytes)
    try:
        for cb in (1, 2, 4):
            ctx.quantize(dx, out, x.size, cb)
            q = np.frombuffer(ctx.download(out, x.nbytes), dtype=np.float32)
            assert np.array_equal(bits(q), bits(g[f"q{cb}"])), cb
        dq = ctx.upload(np.ascontiguousarray(g["q2"]))
        ctx.encode_compute(dq, out, x.size, 2)
        codes = np.frombuffer(ctx.download(out, 2 * x.size), dtype=np.uint16)
        assert np.array_equal(codes, g["pack16"])
        dq1 = ctx.upload(np.ascontiguousarray(g["q1"]))
        ctx.encode_compute(dq1, out, x.size, 1)
        codes = np.frombuffer(ctx.download(out, x.size), dtype=np.uint8)
        assert np.array_equal(codes.astype(np.uint16), g["pack8"])
        allc = ctx.upload(np.arange(65536, dtype=np.uint16))
        dec = ctx.alloc(65536 * 4)
        ctx.decode_compute(allc, dec, 65536, 2)
        assert np.array_equal(bits(np.frombuffer(ctx.download(dec, 65536 * 4), np.float32)),
                              bits(g["unpack16"]))
        c8 = ctx.upload(np.arange(256, dtype=np.uint8))
        ctx.decode_compute(c8, dec, 256, 1)
        assert np.array_equal(bits(np.frombuffer(ctx.download(dec, 256 * 4), np.float32)), bits(g["unpack8"]))
        for p in (dq, dq1, allc, dec, c8):
            ctx.free(p)
    finally:
        ctx.free(dx)
        ctx.free(out)
    with pytest.raises(ValueError, match="unsupported width"):
        ctx.quantize(0, 0, 1, 3)


# ---------------------------------------------------------------- Adam
def test_adam_goldens(mk, ctx):
    g = load_npz("adam")
    w, m, v = (ctx.upload(g[k]) for k in ("w0", "m0", "v0"))
    step = int(g["step0"][0])
    n = g["w0"].size
    for s in range(5):
        gp = ctx.upload(g[f"g{s}"])
        step = mk.optimizer_step_adam(ctx, w, m, v, step, gp, n)
        ctx.synchronize()
        ctx.free(gp)
        for ptr, key in ((w, "w"), (m, "m"), (v, "v")):
            got = np.frombuffer(ctx.download(ptr, 4 * n), dtype=np.float32)
            assert np.array_equal(bits(got), bits(g[f"{key}{s + 1}"])), (s, key)
    assert step == 8
    for p in (w, m, v):
        ctx.free(p)


# ---------------------------------------------------------------- K1 snapshot
# snapshot transports (-1 = auto): 1 = pack kernel + copy-engine push beside
# the FNV kernel (auto for peer replicas), 0 = pack-kernel replica stores
# (auto for local replicas), 5 = FNV-kernel replica stores, 3 = SM push on
# reserved SMs beside the FNV kernel, 2 = fused gather+store+hash kernel,
# 4 = copy-engine push after the hash
MODES = [-1, 1, 5, 3, 2, 0, 4]


@pytest.fixture
def mode(request, ctx):
    ctx.set_replica_mode(request.param)
    yield request.param
    ctx.set_replica_mode(-1)


@pytest.mark.parametrize("mode", MODES, indirect=True)
@pytest.mark.parametrize("name", CASE_NAMES)
def test_snapshot_matches_reference_bytes(mk, ctx, name, mode):
    c = load_case(name)
    for s in range(c.T + 1):
        st = upload_state(mk, ctx, c, s)
        active, co = c.slot(s % c.W)
        blob = mk.snapshot_record(st, active, co, s % c.W, 1, s // c.W * c.W, c.W)
        assert blob.to_host() == c.blob(s), (name, s)
        # the same record through the host-buffer entry point (e2e path)
        assert mk.snapshot_record_host(st, active, co, s % c.W, 1, s // c.W * c.W, c.W) == c.blob(s)
        assert st.serialize_state() == c.mlst(s)


@pytest.mark.parametrize("name", ["verify_toy", "six_op_cb1", "six_op_cb4"])
def test_dense_checkpoint_matches_reference(mk, ctx, name):
    c = load_case(name)
    for s in (0, c.T):
        st = upload_state(mk, ctx, c, s)
        assert mk.dense_checkpoint(st).to_host() == c.d[f"dense_s{s}"].tobytes()


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_snapshot_replicas_identical(mk, ctx, mode):
    c = load_case("verify_toy")
    st = upload_state(mk, ctx, c, 4)
    out = mk.Blob(ctx, 1 << 16)
    r1, r2 = ctx.alloc(1 << 16), ctx.alloc(1 << 16)
    out.add_replica(r1, 1 << 16)
    out.add_replica(r2, 1 << 16)
    active, co = c.slot(1)
    mk.snapshot_record(st, active, co, 1, 1, 3, 3, out)
    ref = c.blob(4)
    assert out.to_host() == ref
    assert ctx.download(r1, len(ref)) == ref
    assert ctx.download(r2, len(ref)) == ref
    with pytest.raises(ValueError, match="replica capacity"):
        small = mk.Blob(ctx, 1 << 16)
        small.add_replica(r1, 64)
        mk.snapshot_record(st, active, co, 1, 1, 3, 3, small)
    # a capacity past the replica's own allocation is refused when the replica is added
    big = ctx.alloc(2 << 20)
    with pytest.raises(ValueError, match="exceeds its allocation"):
        mk.Blob(ctx, 1 << 16).add_replica(big + (1 << 20), 2 << 20)
    with pytest.raises(ValueError, match="exceeds its allocation"):
        mk.Blob(ctx, 1 << 16).add_replica_witness(big + (1 << 20), 2 << 20)
    ctx.free(big)
    ctx.free(r1)
    ctx.free(r2)


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_snapshot_large_replicas_vs_oracle(mk, ctx, oracle, mode):
    """A ~200 MB record (several 64 MiB pack pieces under transport 1) with
    two replicas, byte for byte against the oracle."""
    pcs = [5_000_001, 3_999_999, 2_500_003, 777]
    st = mk.DeviceState(ctx, pcs, 2)
    st.fill_synthetic(seed=5, step=9)
    st.set_meta(77, 3)
    active, co = [0, 2], [1, 3]
    ents = []
    for i in range(len(pcs)):
        P = pcs[i]
        master = oracle.synth(5, 3 * i, -0.25, 0.25, P)
        if i in active:
            ents.append(dict(id=i, mode=0, param_count=P, step=9, master=master,
                             m=oracle.synth(5, 3 * i + 1, -1e-3, 1e-3, P),
                             v=oracle.synth(5, 3 * i + 2, 0.0, 1e-6, P)))
        else:
            ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, 2)))
    ref = oracle.serialize_record(dict(kind=1, iteration=77, window_start=75, wsparse=4, slot=2, data_seed=3),
                                  ents, 2)
    cap = len(ref) + 4096
    out = mk.Blob(ctx, cap)
    reps = [ctx.alloc(cap), ctx.alloc(cap)]
    for r in reps:
        out.add_replica(r, cap)
    mk.snapshot_record(st, active, co, 2, 1, 75, 4, out)
    assert out.to_host() == ref
    assert mk.snapshot_record_host(st, active, co, 2, 1, 75, 4) == ref  # host replica, pushed in pieces
    for r in reps:
        assert ctx.download(r, len(ref)) == ref
        ctx.free(r)
    st.close()


@pytest.mark.parametrize("reserve", [0, 144])
def test_fused_snapshot_on_few_sms_and_unaligned_replicas(mk, ctx, oracle, reserve):
    """The fused snapshot (transport 2: TMA loads from the arena, hash, TMA
    stores) on all SMs and on 4 SMs (chunk tickets: any grid), with a replica
    at an allocation's base and one 48 bytes into it (TMA store maps start
    anywhere 16-byte aligned), every copy against the oracle's
    serialize_record; ~60 MB records, entries at odd offsets.  Unaligned
    replicas are refused by add_replica."""
    pcs = [3_000_001, 4_999_999, 1_000_003, 333]
    st = mk.DeviceState(ctx, pcs, 2)
    st.fill_synthetic(seed=21, step=4)
    st.set_meta(50, 9)
    active, co = [1, 3], [0, 2]
    ents = []
    for i in range(len(pcs)):
        P = pcs[i]
        master = oracle.synth(21, 3 * i, -0.25, 0.25, P)
        if i in active:
            ents.append(dict(id=i, mode=0, param_count=P, step=4, master=master,
                             m=oracle.synth(21, 3 * i + 1, -1e-3, 1e-3, P),
                             v=oracle.synth(21, 3 * i + 2, 0.0, 1e-6, P)))
        else:
            ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, 2)))
    ref = oracle.serialize_record(dict(kind=1, iteration=50, window_start=48, wsparse=4, slot=2, data_seed=9),
                                  ents, 2)
    cap = len(ref) + 4096
    ctx.set_replica_mode(2)
    ctx.set_hash_reserve(reserve)
    try:
        for offset in (0, 48):
            out = mk.Blob(ctx, cap)
            buf = ctx.alloc(cap + 64)
            out.add_replica(buf + offset, cap)
            mk.snapshot_record(st, active, co, 2, 1, 48, 4, out)
            assert out.to_host() == ref, (reserve, offset)
            assert ctx.download(buf + offset, len(ref)) == ref, (reserve, offset)
            out.close()
            ctx.free(buf)
    finally:
        ctx.set_replica_mode(-1)
        ctx.set_hash_reserve(0)
        st.close()


@pytest.mark.parametrize("cb", [1, 2, 4])
def test_fused_snapshot_many_boundaries(mk, ctx, oracle, cb):
    """Transport 2 on a record of 40 operators of 100K-400K parameters: ~80
    segment boundaries, each a pre-gathered patch chunk between runs of
    TMA-loaded chunks at every shift; bytes against the oracle, and the local
    replica; the fused kernel (not the pack fallback) did it."""
    rng = np.random.default_rng(40 + cb)
    pcs = [int(x) for x in rng.integers(100_000, 400_000, 40)]
    st = mk.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=5 + cb, step=3)
    st.set_meta(30, 2)
    active = sorted(int(x) for x in rng.choice(40, 12, replace=False))
    co = [i for i in range(40) if i not in active]
    ents = []
    for i in range(40):
        P = pcs[i]
        master = oracle.synth(5 + cb, 3 * i, -0.25, 0.25, P)
        if i in active:
            ents.append(dict(id=i, mode=0, param_count=P, step=3, master=master,
                             m=oracle.synth(5 + cb, 3 * i + 1, -1e-3, 1e-3, P),
                             v=oracle.synth(5 + cb, 3 * i + 2, 0.0, 1e-6, P)))
        else:
            ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, cb)))
    ref = oracle.serialize_record(dict(kind=1, iteration=30, window_start=30, wsparse=3, slot=0, data_seed=2),
                                  ents, cb)
    cap = len(ref) + 4096
    ctx.set_replica_mode(2)
    try:
        out = mk.Blob(ctx, cap)
        rep = ctx.alloc(cap)
        out.add_replica(rep, cap)
        ctx.set_timing(True)
        mk.snapshot_record(st, active, co, 0, 1, 30, 3, out)
        labels = [name for name, _ in ctx.timings()]
        ctx.set_timing(False)
        assert "pack_fnv" in labels and "pack" not in labels, labels
        assert out.to_host() == ref
        assert ctx.download(rep, len(ref)) == ref
        out.close()
        ctx.free(rep)
    finally:
        ctx.set_replica_mode(-1)
        st.close()


@pytest.mark.parametrize("seed", range(9))
def test_fused_snapshot_random_layouts(mk, ctx, oracle, seed):
    """Transport 2 on random record layouts: operators of 1-3000 parameters
    mixed with 50K-600K ones (runs at every shift; seeds 0-5, the fused
    kernel), 2000 operators of 1-150 parameters (a record made of patch
    chunks; seeds 6-7) and a one-parameter record under one row (seed 8) --
    those two take the pack path; random Full / compute-only split and compute
    width, a replica 0 or 16 bytes into its buffer; every byte of the record
    and the replica against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    if seed < 6:
        n = int(rng.integers(3, 24))
        pcs = [int(rng.integers(1, 3000)) if rng.random() < 0.5 else int(rng.integers(50_000, 600_000))
               for _ in range(n)]
    elif seed < 8:
        n = 2000
        pcs = [int(x) for x in rng.integers(1, 150, n)]
    else:
        n, pcs = 1, [1]
    cb = int(rng.choice([1, 2, 4]))
    st = mk.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=seed, step=5)
    st.set_meta(12, 1 + seed)
    active = sorted(int(x) for x in rng.choice(n, int(rng.integers(1, n + 1)), replace=False))
    co = [i for i in range(n) if i not in active]
    ents = []
    for i in range(n):
        P = pcs[i]
        master = oracle.synth(seed, 3 * i, -0.25, 0.25, P)
        if i in active:
            ents.append(dict(id=i, mode=0, param_count=P, step=5, master=master,
                             m=oracle.synth(seed, 3 * i + 1, -1e-3, 1e-3, P),
                             v=oracle.synth(seed, 3 * i + 2, 0.0, 1e-6, P)))
        else:
            ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, cb)))
    ref = oracle.serialize_record(dict(kind=1, iteration=12, window_start=10, wsparse=3, slot=2, data_seed=1 + seed),
                                  ents, cb)
    cap = len(ref) + 4096
    off = 16 * int(rng.integers(0, 2))
    ctx.set_replica_mode(2)
    try:
        out = mk.Blob(ctx, cap)
        buf = ctx.alloc(cap + 64)
        out.add_replica(buf + off, cap)
        ctx.set_timing(True)
        mk.snapshot_record(st, active, co, 2, 1, 10, 3, out)
        path = "fused" if "pack_fnv" in [name for name, _ in ctx.timings()] else "pack"
        ctx.set_timing(False)
        print(f"seed {seed}: {n} operators, {len(ref)} bytes, cb {cb}, replica +{off}: {path}")
        assert path == ("fused" if seed < 6 else "pack")
        assert out.to_host() == ref, path
        assert ctx.download(buf + off, len(ref)) == ref, path
        out.close()
        ctx.free(buf)
    finally:
        ctx.set_replica_mode(-1)
        st.close()


def test_replay_fast_paths_match_ieee_intrinsics(mk, ctx):
    """The conversion's hoisted-reciprocal division and spelled-out square root
    equal __fdiv_rn / __fsqrt_rn: 2^28 divisions over every exponent pair of
    their range, and all 2^32 float32 patterns for the square root."""
    assert ctx.fastmath_check(1 << 28, seed=7) == (0, 0)


def test_concurrent_contexts_hash_correctly(mk):
    """Two contexts on one device snapshot ~0.5 GB records at once: the hash
    kernels take turns on the device (each needs its whole grid resident)
    and both records match their one-context bytes."""
    a, b = mk.Context(0), mk.Context(0)
    pcs = [20_000_000, 20_000_000]
    sts = []
    for c, seed in ((a, 3), (b, 4)):
        st = mk.DeviceState(c, pcs, 2)
        st.fill_synthetic(seed=seed, step=5)
        st.set_meta(10, 1)
        sts.append(st)
    ref = [mk.snapshot_record(st, [0], [1], 0, 1, 10, 2).to_host() for st in sts]
    outs = [mk.Blob(st.ctx, len(ref[0]) + 4096) for st in sts]
    for _ in range(3):
        for st, o in zip(sts, outs):
            mk.snapshot_record(st, [0], [1], 0, 1, 10, 2, o)  # asynchronous on each context's stream
    a.synchronize()
    b.synchronize()
    assert [o.to_host() for o in outs] == ref
    for o in outs:  # blobs and states before their contexts
        o.close()
    for st in sts:
        st.close()
    a.close()
    b.close()


def test_snapshot_errors(mk, ctx):
    c = load_case("six_op_cb4")
    st = upload_state(mk, ctx, c, 1)
    with pytest.raises(ValueError, match="unknown operator 42"):  # test_snapshot.cpp:198-204
        mk.snapshot_record(st, [42], [], 0)
    st.set_step(3, 0, has_full_state=False)
    with pytest.raises(RuntimeError, match="has no full state"):
        mk.snapshot_record(st, [3], [], 0)
    with pytest.raises(RuntimeError, match="is frozen"):  # test_snapshot.cpp:154-160
        mk.dense_checkpoint(st)


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_snapshot_large_synthetic_vs_oracle(mk, ctx, oracle, mode):
    """Odd sizes and every compute width at MB scale against the oracle."""
    rng = np.random.default_rng(2)
    for cb in (1, 2, 4):
        pcs = [int(x) for x in rng.integers(100_000, 700_000, 7)] + [1, 3, 5]
        st = mk.DeviceState(ctx, pcs, cb)
        st.fill_synthetic(seed=99 + cb, step=17)
        st.set_meta(123, 7)
        active, co = [0, 3, 8], [1, 2, 4, 5, 6, 7, 9]
        blob = mk.snapshot_record(st, active, co, 2, 1, 120, 6)
        ents = []
        for i in sorted(active + co):
            P = pcs[i]
            master = oracle.synth(99 + cb, 3 * i, -0.25, 0.25, P)
            if i in active:
                ents.append(dict(id=i, mode=0, param_count=P, step=17, master=master,
                                 m=oracle.synth(99 + cb, 3 * i + 1, -1e-3, 1e-3, P),
                                 v=oracle.synth(99 + cb, 3 * i + 2, 0.0, 1e-6, P)))
            else:
                ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, cb)))
        ref = oracle.serialize_record(dict(kind=1, iteration=123, window_start=120, wsparse=6, slot=2,
                                           data_seed=7), ents, cb)
        got = blob.to_host()
        assert len(got) == len(ref)
        assert got == ref, cb


# ---------------------------------------------------------------- parse
@pytest.mark.parametrize("name", ["verify_toy", "six_op_cb1", "six_op_cb4"])
def test_parse_record_matches_oracle(mk, ctx, oracle, name):
    c = load_case(name)
    for s in range(c.T + 1):
        b = mk.Blob.from_host(ctx, c.blob(s))
        h, ents = mk.parse_record(b, c.compute_bytes)
        oh, oents = oracle.parse_record(c.blob(s), c.compute_bytes)
        assert h == oh and ents == oents
        for e in ents[:3]:
            got = mk.read_entry(b, e, c.compute_bytes)
            o = c.op(s, e["id"])
            if e["mode"] == 0:
                assert np.array_equal(bits(got["master"]), bits(o["master"]))
            else:
                assert np.array_equal(bits(got["compute"]), bits(o["compute"]))


def test_parse_errors(mk, ctx, oracle):
    c = load_case("six_op_cb4")
    blob = bytearray(c.blob(1))
    blob[len(blob) // 2] ^= 0x40
    with pytest.raises(RuntimeError, match="container checksum mismatch"):
        mk.parse_record(mk.Blob.from_host(ctx, bytes(blob)), 4)
    with pytest.raises(RuntimeError, match="container truncated"):
        mk.parse_record(mk.Blob.from_host(ctx, b"\x01\x02\x03"), 4)
    body = b"XXXX" + c.blob(1)[4:-8]
    bad = body + oracle.fnv1a64(body).to_bytes(8, "little")
    with pytest.raises(RuntimeError, match="bad magic"):
        mk.parse_record(mk.Blob.from_host(ctx, bad), 4)
    body = c.blob(1)[:4] + (7).to_bytes(4, "little") + c.blob(1)[8:-8]
    bad = body + oracle.fnv1a64(body).to_bytes(8, "little")
    with pytest.raises(RuntimeError, match="unsupported version 7"):
        mk.parse_record(mk.Blob.from_host(ctx, bad), 4)
    body = c.blob(1)[:-100]
    bad = body + oracle.fnv1a64(body).to_bytes(8, "little")
    with pytest.raises(RuntimeError, match="container truncated"):
        mk.parse_record(mk.Blob.from_host(ctx, bad), 4)


def _ref_parse_verdicts(records, cb, q):
    """The compiled reference's parse of each record, in a child process whose
    address space is capped: a mutated count makes the reference allocate
    (and zero) a vector of that many entries, which must fail as bad_alloc
    instead of exhausting the host."""
    import resource

    resource.setrlimit(resource.RLIMIT_AS, (4 << 30, 4 << 30))
    from oracle.oracle import RefError, load_reference, ref_parse_record

    ref = load_reference()
    out = []
    for rec in records:
        try:
            out.append(ref_parse_record(ref, rec, cb))
        except RefError as e:
            out.append(str(e))
        except MemoryError:
            out.append("std::bad_alloc")
    q.put(out)


@pytest.mark.parametrize("name", ["verify_toy", "six_op_cb1", "six_op_cb4", "dp2_pp2"])
def test_parse_fuzz_matches_reference(mk, ctx, oracle, reference, name):
    """parse_record (snapshot.hpp:146-197) on 150 mutated copies of a real
    record -- random byte flips (header, entry table, payloads), truncations
    and extensions, each re-sealed with a valid FNV trailer so the structural
    checks run -- against the compiled reference's parse of the same bytes:
    the same error text, or the same entry count, iteration and slot.  Where
    a mutated count makes the reference's own vector allocation throw, any
    error is the same verdict."""
    import multiprocessing as mproc

    c = load_case(name)
    cb = c.compute_bytes
    rng = np.random.default_rng(sum(map(ord, name)))
    base = c.blob(1)[:-8]
    records = []
    for trial in range(150):
        body = bytearray(base)
        kind = trial % 3
        if kind == 0:  # flips, mostly in the header and entry table
            for _ in range(int(rng.integers(1, 4))):
                pos = int(rng.integers(0, min(len(body), 160))) if rng.random() < 0.8 else int(rng.integers(0, len(body)))
                body[pos] ^= 1 << int(rng.integers(0, 8))
        elif kind == 1:  # truncated
            body = body[:int(rng.integers(0, len(body)))]
        else:  # extended
            body += bytes(rng.integers(0, 256, int(rng.integers(1, 64)), dtype=np.uint8))
        records.append(bytes(body) + oracle.fnv1a64(bytes(body)).to_bytes(8, "little"))
    mp = mproc.get_context("spawn")
    q = mp.Queue()
    proc = mp.Process(target=_ref_parse_verdicts, args=(records, cb, q))
    proc.start()
    wants = q.get(timeout=300)
    proc.join(timeout=60)
    outcomes = {"ok": 0, "error": 0}
    for trial, (rec, want) in enumerate(zip(records, wants)):
        try:
            hdr, ents = mk.parse_record(mk.Blob.from_host(ctx, rec), cb)
            got = (len(ents), hdr["iteration"], hdr["slot"])
        except (mk.MlckRuntime, mk.MlckInvalid) as e:
            got = str(e)
        if isinstance(want, str):
            alloc = "bad_alloc" in want or "_M_default_append" in want or "length" in want
            assert isinstance(got, str) and (alloc or want in got), (trial, want, got)
            outcomes["error"] += 1
        else:
            assert got == tuple(want), (trial, want, got)
            outcomes["ok"] += 1
    assert outcomes["error"] > 0


def test_check_coverage(mk, ctx):
    c = load_case("six_op_cb4")  # test_snapshot.cpp:170-196
    blobs = [mk.Blob.from_host(ctx, c.blob(k)) for k in range(3)]
    mk.check_coverage(blobs, c.n_ops, 4)
    bad = [blobs[0], blobs[1], blobs[1]]
    with pytest.raises(RuntimeError, match="window coverage violated for operator 2: 2 full payloads"):
        mk.check_coverage(bad, c.n_ops, 4)


# ---------------------------------------------------------------- K3 conversion
def gradlog_for(mk, ctx, c, w):
    g = mk.GradLog(ctx, c.meta["param_counts"], max(c.W, 1))
    for it in range(w + 1, w + c.W + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    return g


@pytest.mark.parametrize("name", CASE_NAMES)
def test_conversion_matches_reference(mk, ctx, name):
    c = load_case(name)
    opt = c.optimizer
    o = mk.Optimizer(opt["kind"], opt["lr"], opt["beta1"], opt["beta2"], opt["eps"])
    for w in c.meta["converted_windows"]:
        blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
        g = gradlog_for(mk, ctx, c, w) if c.W > 1 else None
        out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
        mk.sparse_to_dense_convert(out, blobs, w, c.W, c.data_seed, g, o)
        assert out.serialize_state() == c.converted(w), (name, w)
        # compute weights are refreshed from the converted masters
        it = w + c.W if c.W > 1 else w
        for i in range(c.n_ops):
            assert np.array_equal(bits(out.download_op(i).compute), bits(c.op(it, i)["compute"]))


def test_conversion_from_device_snapshots(mk, ctx):
    """Snapshot on the GPU, convert on the GPU: end-to-end window."""
    c = load_case("verify_toy")
    w = 3
    blobs = []
    for k in range(c.W):
        st = upload_state(mk, ctx, c, w + k)
        a, co = c.slot(k)
        blobs.append(mk.snapshot_record(st, a, co, k, 1, w, c.W))
    g = gradlog_for(mk, ctx, c, w)
    out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    mk.sparse_to_dense_convert(out, blobs, w, c.W, c.data_seed, g)
    assert out.serialize_state() == c.mlst(w + c.W)


def test_conversion_errors(mk, ctx):
    c = load_case("six_op_cb4")
    blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(0)]
    g = gradlog_for(mk, ctx, c, 0)
    out = mk.DeviceState(ctx, c.meta["param_counts"], 4)
    with pytest.raises(RuntimeError, match="sparse checkpoint incomplete: 2 of 3 records"):
        mk.sparse_to_dense_convert(out, blobs[:2], 0, 3, c.data_seed, g)
    raw = bytearray(c.blob(1))
    raw[len(raw) // 3] ^= 0x10  # test_recovery.cpp:129-139
    bad = [blobs[0], mk.Blob.from_host(ctx, bytes(raw)), blobs[2]]
    with pytest.raises(RuntimeError, match=r"slot 1.*checksum"):
        mk.sparse_to_dense_convert(out, bad, 0, 3, c.data_seed, g)
    with pytest.raises(RuntimeError, match="conversion finished with frozen operator 4"):
        mk.sparse_to_dense_convert(out, [blobs[0], blobs[1], blobs[1]], 0, 3, c.data_seed, g)


# ---------------------------------------------------------------- localized recovery
@pytest.mark.parametrize("name", ["verify_toy", "dp2_pp2"])
def test_localized_recovery_matches_reference(mk, ctx, name):
    """localized_recover (recovery.hpp:240-289) of every stage, from every
    complete window, to the window's end and to the last logged iteration:
    bit-identical to the reference's own localized recovery."""
    c = load_case(name)
    P = c.meta["param_counts"]
    g = mk.GradLog(ctx, P, c.T)
    for it in range(1, c.T + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    cases = c.localized()
    assert cases
    for (w, target, lo, hi) in cases:
        blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
        out = mk.DeviceState(ctx, P, c.compute_bytes)
        scope = c.scope(lo, hi)
        mk.localized_recover(out, scope, blobs, w, c.W, c.data_seed, g, target)
        it, ref = c.localized_image(w, target, lo, hi)
        assert it == target
        for i in scope:
            step, master, m, v = ref[i]
            got = out.download_op(i)
            assert got.step == step, (name, w, target, lo, hi, i)
            for a, b in ((got.master, master), (got.m, m), (got.v, v)):
                assert np.array_equal(bits(a), bits(b)), (name, w, target, lo, hi, i)
            # the compute weights are those of the recovered masters
            assert np.array_equal(bits(got.compute), bits(c.op(target, i)["compute"]))


def test_localized_recovery_errors(mk, ctx):
    c = load_case("verify_toy")
    g = gradlog_for(mk, ctx, c, 3)
    blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(3)]
    out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    scope = c.scope(1, 1)
    with pytest.raises(RuntimeError, match="^sparse checkpoint incomplete$"):
        mk.localized_recover(out, scope, blobs[:2], 3, 3, c.data_seed, g, 6)
    raw = bytearray(c.blob(5))
    raw[17] ^= 0x01
    bad = blobs[:2] + [mk.Blob.from_host(ctx, bytes(raw))]
    with pytest.raises(RuntimeError, match=r"slot 2.*checksum"):
        mk.localized_recover(out, scope, bad, 3, 3, c.data_seed, g, 6)
    # a window without some scope operator's Full payload
    dup = [blobs[0], blobs[1], blobs[1]]
    frozen = [i for i in scope if i not in c.slot(0)[0] + c.slot(1)[0]]
    with pytest.raises(RuntimeError, match=f"localized recovery left operator {frozen[0]} frozen"):
        mk.localized_recover(out, scope, dup, 3, 3, c.data_seed, g, 6)
    with pytest.raises(ValueError, match="unknown operator"):
        mk.localized_recover(out, [10 ** 6], blobs, 3, 3, c.data_seed, g, 6)


# ---------------------------------------------------------------- training step
@pytest.mark.parametrize("name", ["verify_toy", "toy_sgd", "six_op_cb1"])
def test_apply_updates_matches_engine(mk, ctx, name):
    """Engine::apply_updates on device == the reference's next state."""
    c = load_case(name)
    opt = c.optimizer
    o = mk.Optimizer(opt["kind"], opt["lr"], opt["beta1"], opt["beta2"], opt["eps"])
    g = mk.GradLog(ctx, c.meta["param_counts"], 2)
    for s in range(c.T):
        st = upload_state(mk, ctx, c, s)
        for i in range(c.n_ops):
            g.put(s + 1, i, c.grads(s + 1, i))
        st.apply_updates(range(c.n_ops), g, s + 1, o)
        st.set_meta(s + 1, c.data_seed)
        assert st.serialize_state() == c.mlst(s + 1), (name, s)


# ---------------------------------------------------------------- K4 logging
@pytest.mark.parametrize("name", ["verify_toy", "dp2_pp2"])
@pytest.mark.parametrize("kind", [0, 1])
def test_upstream_log_matches_reference(mk, ctx, name, kind):
    c = load_case(name)
    ref = c.log_entries()
    log = mk.UpstreamLog(ctx, 1 << 22, kind=kind, device=0)
    # producers write in execution order; the reference map orders by key
    order = np.random.default_rng(1).permutation(len(ref))
    bufs = []
    for j in order:
        key, data = ref[j]
        p = ctx.upload(data)
        bufs.append(p)
        log.put(*key, p, data.size)
    log.sync()
    got = log.entries()
    assert [k for k, _ in got] == [k for k, _ in ref]
    for (_, a), (_, b) in zip(got, ref):
        assert np.array_equal(bits(a), bits(b))
    assert log.bytes() == sum(d.size * 4 for _, d in ref)
    k0 = ref[-1][0]
    assert np.array_equal(bits(log.at(*k0)), bits(ref[-1][1]))
    # gc_logs keeps iteration >= window start (engine.hpp:90-94)
    log.gc(3)
    assert all(k[0] >= 3 for k, _ in log.entries())
    log.gc(100)
    assert len(log) == 0
    with pytest.raises(RuntimeError, match="upstream log missing entry: iteration 1 micro-batch 0 boundary 0 fwd"):
        log.at(1, 0, 0, 0)
    for p in bufs:
        ctx.free(p)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("seed", range(3))
def test_upstream_log_random_puts_and_gc(mk, ctx, kind, seed):
    """UpstreamLog (engine.hpp:55-94) under random traffic: 300 puts of 1-20K
    floats on colliding keys (a repeated key overwrites, like the reference's
    map assignment), gc_logs at rising window starts, reads of present and
    missing keys -- against a dict model of the reference's std::map after
    every operation batch (key order, bytes, at(), bytes()); then a 1 MiB
    ring recycled many times over, collected, and refilled by one entry of its
    whole capacity (the allocator's holes coalesce)."""
    rng = np.random.default_rng(300 + seed)
    log = mk.UpstreamLog(ctx, 1 << 26, kind=kind, device=0)
    model, bufs, floor = {}, [], 0

    def check():
        log.sync()
        got = log.entries()
        want = sorted(model.items())
        assert [k for k, _ in got] == [k for k, _ in want]
        for (_, a), (_, b) in zip(got, want):
            assert np.array_equal(bits(a), bits(b))
        assert log.bytes() == sum(v.size * 4 for v in model.values())

    for step in range(300):
        if rng.random() < 0.05:
            floor += int(rng.integers(1, 3))
            log.gc(floor)
            model = {k: v for k, v in model.items() if k[0] >= floor}
        key = (int(rng.integers(floor, floor + 5)), int(rng.integers(0, 4)), int(rng.integers(0, 3)),
               int(rng.integers(0, 2)))
        data = rng.standard_normal(int(rng.integers(1, 20_000))).astype(np.float32)
        p = ctx.upload(data)
        bufs.append(p)
        log.put(*key, p, data.size)
        model[key] = data
        if step % 50 == 49:
            check()
            k = list(model)[int(rng.integers(0, len(model)))]
            assert np.array_equal(bits(log.at(*k)), bits(model[k]))
    check()
    with pytest.raises(RuntimeError, match="upstream log missing entry"):
        log.at(floor + 100, 0, 0, 1)
    log.close()
    # a 1 MiB ring recycled many times over (first-fit holes from overwrites and gc):
    # the same model, then everything collected and one entry of the whole ring
    cap = 1 << 20
    log = mk.UpstreamLog(ctx, cap, kind=kind, device=0)
    model, floor = {}, 0
    for step in range(600):
        if step % 10 == 9:
            floor += 1
            log.gc(floor)
            model = {k: v for k, v in model.items() if k[0] >= floor}
        key = (int(rng.integers(floor, floor + 3)), int(rng.integers(0, 4)), int(rng.integers(0, 3)),
               int(rng.integers(0, 2)))
        data = rng.standard_normal(int(rng.integers(1, 4_000))).astype(np.float32)
        live = sum(-(-v.size * 4 // 256) * 256 for k, v in model.items() if k != key)
        if live + data.size * 4 > cap // 2:
            continue
        p = ctx.upload(data)
        bufs.append(p)
        log.put(*key, p, data.size)
        model[key] = data
    check()
    log.gc(floor + 1000)
    assert len(log) == 0 and log.bytes() == 0
    whole = rng.standard_normal(cap // 4).astype(np.float32)
    p = ctx.upload(whole)
    bufs.append(p)
    log.put(floor + 1000, 0, 0, 0, p, whole.size)  # the free list coalesced back to one block
    log.sync()
    assert np.array_equal(bits(log.at(floor + 1000, 0, 0, 0)), bits(whole))
    log.close()
    for p in bufs:
        ctx.free(p)
