"""GPU checks of the drop-in boundary's newer entry points against the
reference: conversion_plan (recovery.hpp:123-137), the scalar codec forms
quantize_value / pack_reduced / unpack_reduced (tensor.hpp:99-183) and the
generic reduced formats, localized_recover with a RecoverySegment
(recovery.hpp:240-289), the log's ordered / async source contract, the
hash kernel on a reserved-SM grid (any grid size is correct), and snapshots
ordered on a caller's stream (mlck_ctx_set_stream, hash_async)."""
import numpy as np
import pytest

from golden_cases import load_case
from oracle.oracle import RefError, ref_conversion_plan, ref_pack_reduced, ref_unpack_reduced

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


# ---------------------------------------------------------------- conversion_plan
@pytest.mark.parametrize("name,w", [("verify_toy", 0), ("verify_toy", 3), ("six_op_cb1", 3), ("dp2_pp2", 0)])
def test_conversion_plan_matches_reference(mk, ctx, reference, name, w):
    c = load_case(name)
    raw = c.window_blobs(w)
    blobs = [mk.Blob.from_host(ctx, b) for b in raw]
    got = mk.conversion_plan(blobs, w, c.compute_bytes)
    want = ref_conversion_plan(reference, w, c.W, raw, c.compute_bytes)
    assert got == want


def test_conversion_plan_errors_are_unwrapped(mk, ctx, reference):
    """conversion_plan calls parse_record directly: the raw parse error, no
    'sparse checkpoint record (slot k)' prefix (recovery.hpp:130)."""
    c = load_case("verify_toy")
    raw = c.window_blobs(3)
    bad = bytearray(raw[1])
    bad[len(bad) // 2] ^= 0x20
    raw2 = [raw[0], bytes(bad), raw[2]]
    with pytest.raises(RefError) as ref_err:
        ref_conversion_plan(reference, 3, 3, raw2, c.compute_bytes)
    blobs = [mk.Blob.from_host(ctx, b) for b in raw2]
    with pytest.raises(RuntimeError) as ours:
        mk.conversion_plan(blobs, 3, c.compute_bytes)
    assert str(ours.value) == str(ref_err.value) == "container checksum mismatch"


# ---------------------------------------------------------------- scalar codecs
def special_floats():
    v = [0.0, -0.0, 1.0, -1.0, 65504.0, 65520.0, 65519.99, 240.0, 248.0, 239.9, 1e-8, -1e-8, 6e-8, 2 ** -24,
         2 ** -25, 2 ** -14, 2 ** -9, 2 ** -6, 2 ** -10, np.inf, -np.inf, 1e30, -1e30, 3.4e38]
    return np.array(v, dtype=np.float32)


@pytest.mark.parametrize("cb", [1, 2, 4])
def test_quantize_value_matches_reference(mk, ctx, reference, cb):
    rng = np.random.default_rng(cb)
    x = np.concatenate([special_floats(), rng.standard_normal(20000).astype(np.float32) * 10 ** rng.uniform(
        -9, 6, 20000).astype(np.float32), rng.integers(0, 2 ** 32, 20000, dtype=np.uint64).astype(np.uint32).view(
        np.float32)])
    got = ctx.quantize_values(x, cb)
    want = _ref_q(reference, x, cb)
    assert np.array_equal(bits(got), bits(want))
    with pytest.raises(ValueError, match="quantize: unsupported width 3"):
        ctx.quantize_values(x[:4], 3)


def _ref_q(reference, x, cb):
    """quantize_value over the array (mlr_quantize_array: bits as they are)."""
    import ctypes as C
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    err = C.create_string_buffer(256)
    fp = C.POINTER(C.c_float)
    assert reference.lib.mlr_quantize_array(x.ctypes.data_as(fp), x.size, cb, out.ctypes.data_as(fp), err, 256) == 0
    return out


@pytest.mark.parametrize("eb,mb", [(5, 10), (4, 3), (5, 2), (8, 7), (3, 4), (6, 9)])
def test_reduced_format_codecs_match_reference(mk, ctx, reference, eb, mb):
    """unpack_reduced of every code of the format and pack_reduced of every
    decoded value (and of raw floats) == the reference's."""
    n_codes = 1 << (1 + eb + mb)
    codes = np.arange(n_codes, dtype=np.uint16)
    got_f = ctx.unpack_reduced_values(codes, eb, mb)
    want_f = ref_unpack_reduced(reference, codes, eb, mb)
    assert np.array_equal(bits(got_f), bits(want_f))
    rng = np.random.default_rng(eb * 100 + mb)
    x = np.concatenate([want_f, special_floats(), rng.standard_normal(5000).astype(np.float32)])
    got_c = ctx.pack_reduced_values(x, eb, mb)
    want_c = ref_pack_reduced(reference, x, eb, mb)
    assert np.array_equal(got_c, want_c)


def test_reduced_format_bad_widths(mk, ctx):
    with pytest.raises(ValueError, match="unsupported widths"):
        ctx.pack_reduced_values(np.ones(4, np.float32), 9, 3)


# ---------------------------------------------------------------- RecoverySegment
def _gradlog(mk, ctx, c):
    g = mk.GradLog(ctx, c.meta["param_counts"], c.T)
    for it in range(1, c.T + 1):
        for i in range(c.n_ops):
            g.put(it, i, c.grads(it, i))
    return g


def _log_with_reference_entries(mk, ctx, c):
    """A device-ring upstream log holding the reference's own boundary entries."""
    ents = c.log_entries()
    need = sum(4 * d.size + 256 for _, d in ents) + (1 << 16)
    log = mk.UpstreamLog(ctx, need, kind=1, device=0)
    bufs = []
    for (it, mb, b, d), data in ents:
        p = ctx.upload(np.ascontiguousarray(data, dtype=np.float32))
        bufs.append(p)
        log.put(it, mb, b, d, p, data.size)
    log.sync()
    for p in bufs:
        ctx.free(p)
    return log


def test_localized_recover_segment_matches_reference(mk, ctx):
    """localized_recover(engine, RecoverySegment, ckpt, logs, target) with the
    reference's stage_of_op and its logged boundaries: bit-identical scope."""
    c = load_case("dp2_pp2")
    P = c.meta["param_counts"]
    g = _gradlog(mk, ctx, c)
    log = _log_with_reference_entries(mk, ctx, c)
    stage_of_op = c.meta["stage_of_op"]
    n_stages = max(stage_of_op) + 1
    n_gmb = int(c.meta["cfg"]["dp_degree"]) * int(c.meta["cfg"]["microbatches"])
    for (w, target, lo, hi) in c.localized():
        blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
        out = mk.DeviceState(ctx, P, c.compute_bytes)
        mk.localized_recover_segment(out, lo, hi, stage_of_op, n_stages, blobs, w, c.W, c.data_seed, log, n_gmb, g,
                                     target)
        it, ref = c.localized_image(w, target, lo, hi)
        assert out.meta()[0] == it == target
        for i in c.scope(lo, hi):
            step, master, m, v = ref[i]
            got = out.download_op(i)
            assert got.step == step
            for a, b in ((got.master, master), (got.m, m), (got.v, v)):
                assert np.array_equal(bits(a), bits(b)), (w, target, lo, hi, i)


def test_localized_recover_segment_needs_the_boundary_log(mk, ctx):
    c = load_case("dp2_pp2")
    g = _gradlog(mk, ctx, c)
    stage_of_op = c.meta["stage_of_op"]
    n_stages = max(stage_of_op) + 1
    n_gmb = int(c.meta["cfg"]["dp_degree"]) * int(c.meta["cfg"]["microbatches"])
    w, target, lo, hi = c.localized()[0]
    blobs = [mk.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
    out = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    empty = mk.UpstreamLog(ctx, 1 << 16, kind=0)
    if lo == 0 and hi == n_stages - 1:
        pytest.skip("segment spans every stage")
    with pytest.raises(RuntimeError, match=f"upstream log missing entry: iteration {w + 1} micro-batch 0 boundary"):
        mk.localized_recover_segment(out, lo, hi, stage_of_op, n_stages, blobs, w, c.W, c.data_seed, empty, n_gmb,
                                     g, target)
    with pytest.raises(ValueError, match="recovery segment"):
        mk.localized_recover_segment(out, 1, 0, stage_of_op, n_stages, blobs, w, c.W, c.data_seed, empty, n_gmb, g,
                                     target)


# ---------------------------------------------------------------- log source contract
def test_log_put_ordered_mode_allows_source_reuse(mk, ctx):
    """Default ORDERED mode: once put() returns, work queued on the ctx stream
    may overwrite the source -- the logged bytes are the ones put."""
    n = 1 << 22
    a = np.arange(n, dtype=np.float32)
    p = ctx.upload(a)
    log = mk.UpstreamLog(ctx, 8 * n + 4096, kind=0)
    log.put(1, 0, 0, 0, p, n)
    ctx.memset(p, 0xff, 4 * n)  # the next micro-batch reuses the buffer (ctx stream)
    log.put(1, 1, 0, 0, p, n)
    log.sync()
    assert np.array_equal(log.at(1, 0, 0, 0), a)
    assert np.array_equal(bits(log.at(1, 1, 0, 0)), np.full(n, 0xffffffff, np.uint32))
    ctx.free(p)


def test_log_async_mode_with_fence(mk, ctx):
    n = 1 << 20
    a = np.arange(n, dtype=np.float32) * 3
    p = ctx.upload(a)
    log = mk.UpstreamLog(ctx, 4 * n + 4096, kind=1, device=0)
    log.set_async(True)
    log.put(2, 0, 1, 1, p, n)
    log.fence()  # the ctx stream now follows the copy
    ctx.memset(p, 0, 4 * n)
    log.sync()
    assert np.array_equal(log.at(2, 0, 1, 1), a)
    ctx.free(p)


# ---------------------------------------------------------------- hash grid
@pytest.mark.parametrize("reserve", [0, 100, 140, 147])
def test_fnv_on_a_reserved_grid(mk, ctx, oracle, reserve):
    """Tickets hand the chunks out: the hash is exact on any number of SMs."""
    data = np.random.default_rng(reserve).integers(0, 256, 40 * 65536 + 11, dtype=np.uint8)
    p = ctx.upload(data)
    ctx.set_hash_reserve(reserve)
    try:
        assert ctx.fnv1a64(p, data.size) == oracle.fnv1a64(data)
    finally:
        ctx.set_hash_reserve(0)
        ctx.free(p)


def test_parse_beyond_the_old_caps(mk, ctx, oracle):
    """parse / coverage of 40 records (the round-1 path capped a call at 32)
    and a record of 70,000 entries (capped at 65,536)."""
    c = load_case("verify_toy")
    raw = c.window_blobs(3) * 14
    blobs = [mk.Blob.from_host(ctx, b) for b in raw[:40]]
    plan = mk.conversion_plan(blobs, 0, c.compute_bytes)
    assert len(plan) == 40
    # one record with 70,000 compute-only entries of one parameter each
    n = 70000
    hdr = dict(kind=1, iteration=5, window_start=5, wsparse=1, slot=0, data_seed=1)
    ents = [dict(id=i, mode=1, param_count=1, compute=np.array([0.5], np.float32)) for i in range(n)]
    blob = oracle.serialize_record(hdr, ents, 2)
    info, entries = mk.parse_record(mk.Blob.from_host(ctx, blob), 2)
    assert len(entries) == n and entries[-1]["id"] == n - 1


# ---------------------------------------------------------------- stream order
class _DevArray:
    """A raw device float32 span as a torch tensor (no copy)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


@pytest.mark.parametrize("mode", [-1, 0, 1, 5])
@pytest.mark.parametrize("hash_async", [False, True])
def test_snapshot_follows_the_user_stream(mk, ctx, oracle, mode, hash_async):
    """mlck_ctx_set_stream: a snapshot is ordered after the work already
    queued on the caller's stream (here a ~10 ms sleep, then an in-place write
    to operator 0's master and v), with the trailer hash on the same stream or
    on the context's side stream (mlck_ctx_set_hash_async); the record and its
    replica equal the oracle's serialize_record of the written state."""
    import torch

    pcs = [300_001, 1_000_003, 77]
    st = mk.DeviceState(ctx, pcs, 2)
    st.fill_synthetic(seed=4, step=6)
    st.set_meta(20, 3)
    ctx.synchronize()
    master0, _m0, v0, _codes = st.op_ptrs(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.set_replica_mode(mode)
    ctx.set_hash_async(hash_async)
    try:
        with torch.cuda.stream(stream):
            torch.cuda._sleep(20_000_000)
            torch.as_tensor(_DevArray(master0, pcs[0]), device="cuda").fill_(0.5)
            torch.as_tensor(_DevArray(v0, pcs[0]), device="cuda").mul_(2.0)
        cap = 16 << 20
        out = mk.Blob(ctx, cap)
        rep = ctx.alloc(cap)
        out.add_replica(rep, cap)
        mk.snapshot_record(st, [0, 2], [1], 1, 1, 19, 2, out)
        stream.synchronize()
        ctx.synchronize()
        ents = []
        for i, P in enumerate(pcs):
            master = oracle.synth(4, 3 * i, -0.25, 0.25, P)
            if i == 1:
                ents.append(dict(id=i, mode=1, param_count=P, compute=oracle.quantize(master, 2)))
                continue
            v = oracle.synth(4, 3 * i + 2, 0.0, 1e-6, P)
            if i == 0:
                master = np.full(P, 0.5, dtype=np.float32)
                v = v * np.float32(2.0)
            ents.append(dict(id=i, mode=0, param_count=P, step=6, master=master,
                             m=oracle.synth(4, 3 * i + 1, -1e-3, 1e-3, P), v=v))
        ref = oracle.serialize_record(dict(kind=1, iteration=20, window_start=19, wsparse=2, slot=1, data_seed=3),
                                      ents, 2)
        assert out.to_host() == ref
        assert ctx.download(rep, len(ref)) == ref
        assert out.replication() == 1
        out.close()
        ctx.free(rep)
    finally:
        ctx.set_stream(None)
        ctx.set_replica_mode(-1)
        ctx.set_hash_async(False)
        st.close()
