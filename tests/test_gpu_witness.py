"""Witnessed re-verification (mlck_ctx_set_witness, fnv.cuh automaton_and_ends, kernels.cu fnv_witness_kernel):
a record the hash kernel wrote keeps its segment starts, and parse_record /
check_coverage / conversion re-hash it against them.  The checksum must be
the exact FNV-1a-64 of the bytes in memory whatever happened to the record
or the witness afterwards."""
import numpy as np
import pytest

from golden_cases import load_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk():
    from paper_2412_15411_b200 import mlck
    return mlck


@pytest.fixture()
def ctx(mk):
    c = mk.Context(0)
    yield c
    c.close()


def synthetic_record(mk, ctx, pcs, slot, cb=2, seed=3):
    st = mk.DeviceState(ctx, pcs, cb)
    st.fill_synthetic(seed=seed, step=4)
    st.set_meta(9, 5)
    b = mk.snapshot_record(st, *slot, 0, 1, 9, 1)
    return st, b


# ragged record sizes around the 32-byte segment / 128-byte row / 64 KiB chunk units
@pytest.mark.parametrize("pcs,slot", [
    ([1], ([0], [])), ([3, 5], ([0], [1])), ([7, 1000, 33], ([1], [0, 2])),
    ([16383, 16384, 16385], ([0, 2], [1])), ([300_000, 77_777, 1], ([1], [0, 2])),
    ([5_000_003, 4_000_001], ([0], [1]))])
@pytest.mark.parametrize("mode", [0, 2])
def test_witnessed_parse_matches_oracle(mk, ctx, oracle, pcs, slot, mode):
    ctx.set_replica_mode(mode)
    st, b = synthetic_record(mk, ctx, pcs, slot)
    ctx.set_replica_mode(-1)
    assert b.witness_ptr != 0
    host = b.to_host()
    assert int.from_bytes(host[-8:], "little") == oracle.fnv1a64(np.frombuffer(host[:-8], np.uint8))
    used0, fb0 = ctx.witness_stats()
    mk.parse_record(b, 2)  # checksum verified against the witness (the binding parses twice: count, entries)
    used, fb = ctx.witness_stats()
    assert used > used0 and fb == fb0


def test_corrupted_byte_is_caught_with_a_witness(mk, ctx):
    st, b = synthetic_record(mk, ctx, [100_000, 50_000], ([0], [1]))
    n = b.size
    for off in (0, 45, 1000, n // 2, n - 9):
        host = bytearray(b.to_host())
        raw = host[off]
        ctx.memset(b.device_ptr + off, raw ^ 0x01, 1)
        with pytest.raises(RuntimeError, match="container checksum mismatch"):
            mk.parse_record(b, 2)
        ctx.memset(b.device_ptr + off, raw, 1)
        mk.parse_record(b, 2)


def test_stale_witness_falls_back_and_stays_exact(mk, ctx):
    st, b = synthetic_record(mk, ctx, [200_000, 3], ([0], [1]))
    w = b.witness_ptr
    # flip one witnessed start: the segment chain no longer closes
    word = np.frombuffer(ctx.download(w + 4 * 10, 4), np.uint8).copy()
    ctx.memset(w + 4 * 10 + 1, int(word[1]) ^ 0x5a, 1)
    used0, fb0 = ctx.witness_stats()
    mk.parse_record(b, 2)  # still verifies: the full hash takes over
    assert ctx.witness_stats()[1] > fb0
    # a stale witness and a corrupted record: still caught
    ctx.memset(b.device_ptr + 777, 0x11, 1)
    with pytest.raises(RuntimeError, match="container checksum mismatch"):
        mk.parse_record(b, 2)


def test_conversion_with_and_without_witness(mk, ctx):
    """The golden conversion through witnessed records, and with the witness
    off: identical bytes, equal to the reference's conversion."""
    c = load_case("verify_toy")
    w = 3
    g = mk.GradLog(ctx, c.meta["param_counts"], c.W)
    for it in range(w + 1, w + c.W + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    for on in (True, False):
        ctx.set_witness(on)
        blobs = []
        for k in range(c.W):
            s = w + k
            st = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
            for i in range(c.n_ops):
                o = c.op(s, i)
                st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
            st.set_meta(s, c.data_seed)
            blobs.append(mk.snapshot_record(st, *c.slot(k), k, 1, w, c.W))
            assert (blobs[-1].witness_ptr != 0) == on
        used0, _ = ctx.witness_stats()
        out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
        mk.sparse_to_dense_convert(out, blobs, w, c.W, c.data_seed, g)
        assert out.serialize_state() == c.converted(w)
        assert ctx.witness_stats()[0] - used0 == (c.W if on else 0)
    ctx.set_witness(True)


def test_host_records_have_no_witness(mk, ctx):
    c = load_case("verify_toy")
    b = mk.Blob.from_host(ctx, c.blob(3))
    assert b.witness_ptr == 0
    used0, _ = ctx.witness_stats()
    mk.parse_record(b, c.compute_bytes)
    assert ctx.witness_stats()[0] == used0


@pytest.mark.parametrize("mode", [-1, 0, 1, 2, 5])
def test_witness_travels_with_a_replica(mk, ctx, mode):
    """mlck_blob_add_replica_witness: each record's witness follows it to a
    buffer beside its replica; a blob wrapped over the replica (no copy)
    verifies on the witnessed path, and a corrupted replica is still caught."""
    pcs = [2_000_003, 700_001, 99]
    st = mk.DeviceState(ctx, pcs, 2)
    st.fill_synthetic(seed=8, step=2)
    st.set_meta(12, 4)
    cap = 40 << 20
    out = mk.Blob(ctx, cap)
    rep, wit = ctx.alloc(cap), ctx.alloc(mk.witness_bytes(cap))
    out.add_replica(rep, cap)
    out.add_replica_witness(wit, mk.witness_bytes(cap))
    ctx.set_replica_mode(mode)
    try:
        mk.snapshot_record(st, [0, 2], [1], 0, 1, 12, 2, out)
        ctx.synchronize()
        n = out.size
        view = mk.Blob.wrap(ctx, rep, n, wit)
        assert view.to_host() == out.to_host()
        used0, fb0 = ctx.witness_stats()
        mk.parse_record(view, 2)
        used, fb = ctx.witness_stats()
        assert used > used0 and fb == fb0  # the replica's own witness, no from-scratch hash
        raw = view.to_host()[n // 3]
        ctx.memset(rep + n // 3, raw ^ 0x40, 1)
        with pytest.raises(RuntimeError, match="container checksum mismatch"):
            mk.parse_record(view, 2)
        with pytest.raises(ValueError, match="read-only"):
            mk.snapshot_record(st, [0, 2], [1], 0, 1, 12, 2, view)
        view.close()
        with pytest.raises(ValueError, match="replica witness capacity"):
            small = mk.Blob(ctx, cap)
            small.add_replica_witness(wit, 64)
            mk.snapshot_record(st, [0, 2], [1], 0, 1, 12, 2, small)
    finally:
        ctx.set_replica_mode(-1)
        out.close()
        ctx.free(rep)
        ctx.free(wit)
        st.close()


def test_conversion_from_wrapped_replicas(mk, ctx):
    """The golden window converted from blobs wrapped over replica buffers and
    their witnesses: the reference's bytes, every record verified against its
    travelled witness."""
    c = load_case("verify_toy")
    w = 3
    g = mk.GradLog(ctx, c.meta["param_counts"], c.W)
    for it in range(w + 1, w + c.W + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    cap = 1 << 16
    views, keep = [], []
    for k in range(c.W):
        s = w + k
        st = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
        for i in range(c.n_ops):
            o = c.op(s, i)
            st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
        st.set_meta(s, c.data_seed)
        b = mk.Blob(ctx, cap)
        rep, wit = ctx.alloc(cap), ctx.alloc(mk.witness_bytes(cap))
        b.add_replica(rep, cap)
        b.add_replica_witness(wit, mk.witness_bytes(cap))
        mk.snapshot_record(st, *c.slot(k), k, 1, w, c.W, b)
        ctx.synchronize()
        views.append(mk.Blob.wrap(ctx, rep, b.size, wit))
        keep.append((st, b, rep, wit))
    used0, fb0 = ctx.witness_stats()
    out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    mk.sparse_to_dense_convert(out, views, w, c.W, c.data_seed, g)
    assert out.serialize_state() == c.converted(w)
    used, fb = ctx.witness_stats()
    assert used - used0 == c.W and fb == fb0
    for v in views:
        v.close()
    for st, b, rep, wit in keep:
        b.close()
        ctx.free(rep)
        ctx.free(wit)


def test_wrap_refuses_spans_past_their_allocation(mk, ctx):
    """mlck_blob_wrap: a record running past its allocation, or a witness
    buffer smaller than mlck_witness_bytes (the verifier reads whole chunks of
    it), is refused up front instead of read out of bounds."""
    c = load_case("verify_toy")
    rec = c.blob(3)
    n = len(rec)
    buf = ctx.alloc(n)
    wbuf = ctx.alloc(2 << 20)  # (device allocations are whole 2 MiB pages: point 64 B before the end)
    big_w = ctx.alloc(mk.witness_bytes(n))
    try:
        with pytest.raises(ValueError, match="run past their allocation"):
            mk.Blob.wrap(ctx, buf, n + (4 << 20))
        with pytest.raises(ValueError, match="mlck_witness_bytes"):
            mk.Blob.wrap(ctx, buf, n, wbuf + (2 << 20) - 64)
        view = mk.Blob.wrap(ctx, buf, n, big_w)  # fits: accepted (a stale witness only costs the full hash)
        view.close()
    finally:
        for p in (buf, wbuf, big_w):
            ctx.free(p)
