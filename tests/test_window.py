"""Window lifecycle and durability: the reference's
SparseCheckpoint bookkeeping (snapshot.hpp:300-335) and the "one persisted +
one in-flight" policy.  Policy tests run on CPU with stand-in
blobs; persistence and device-driven replication run on the GPU."""
import os

import numpy as np
import pytest

from golden_cases import load_case


class FakeBlob:
    """Stands in for mlck.Blob in the host-only policy tests."""

    def __init__(self, copies=0):
        self.copies = copies

    def replication(self):
        return self.copies


@pytest.fixture(scope="module")
def window():
    from paper_2412_15411_b200 import window
    return window


def test_sparse_checkpoint_counters(window):
    ck = window.SparseCheckpoint(6, 3, replication_target=2)
    blobs = [FakeBlob() for _ in range(3)]
    for b in blobs[:2]:
        ck.add_record(b)
    assert not ck.complete() and not ck.persisted()
    ck.add_record(blobs[2])
    assert ck.complete()
    ck.poll()
    assert ck.replication == [0, 0, 0] and not ck.persisted()
    for b in blobs:
        b.copies = 2
    ck.poll()
    assert ck.persisted()
    with pytest.raises(RuntimeError, match="window is full"):
        ck.add_record(FakeBlob())


def test_window_ring_keeps_one_persisted_and_collects_the_old(window):
    persisted = []
    ring = window.WindowRing(ctx=None, wsparse=2, replication_target=1, on_persist=persisted.append)
    b = {s: FakeBlob() for s in range(8)}
    # capture_windows: the record after state s goes to window floor(s / W) * W
    assert [ring.window_of(s) for s in range(5)] == [0, 0, 2, 2, 4]
    for s in range(4):
        ring.add_record(s, b[s])
    assert [w.window_start for w in ring.in_flight] == [0, 2]
    assert not ring.poll()  # nothing replicated yet
    b[0].copies = b[1].copies = 1
    assert ring.poll() and ring.persisted.window_start == 0 and persisted == [0]
    assert [w.window_start for w in ring.in_flight] == [2]
    # window 2 persists: window 0 is collected, its blobs go back to the pool
    b[2].copies = b[3].copies = 1
    assert ring.poll() and ring.persisted.window_start == 2 and persisted == [0, 2]
    assert ring.in_flight == [] and set(map(id, ring._free)) == {id(b[0]), id(b[1])}
    assert ring.acquire(16) in (b[0], b[1])
    with pytest.raises(RuntimeError, match="older than the persisted window"):
        ring.add_record(1, FakeBlob())


def test_window_ring_skips_a_stalled_window(window):
    # window 0 never replicates, window 2 does: 2 becomes the persisted one and
    # the stalled, older in-flight window is collected with it
    ring = window.WindowRing(ctx=None, wsparse=2, replication_target=1)
    bl = [FakeBlob() for _ in range(4)]
    for s in range(4):
        ring.add_record(s, bl[s])
    bl[2].copies = bl[3].copies = 1
    assert ring.poll() and ring.persisted.window_start == 2 and ring.in_flight == []


# ---------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def mk():
    from paper_2412_15411_b200 import mlck
    return mlck


@pytest.fixture(scope="module")
def ctx(mk):
    c = mk.Context(0)
    yield c
    c.close()


def upload_state(mk, ctx, c, s):
    st = mk.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
    for i in range(c.n_ops):
        o = c.op(s, i)
        st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
    st.set_meta(s, c.data_seed)
    return st


@pytest.mark.gpu
def test_blob_save_load_roundtrip(mk, ctx, oracle, tmp_path):
    # a multi-piece file (> 64 MiB) with an odd size, and the reference can parse it
    rng = np.random.default_rng(3)
    data = rng.integers(0, 256, (64 << 20) + (1 << 20) + 5, dtype=np.uint8).tobytes()
    b = mk.Blob.from_host(ctx, data)
    path = str(tmp_path / "big.bin")
    assert b.save(path) == len(data)
    assert os.path.getsize(path) == len(data)
    assert mk.Blob.load(ctx, path).to_host() == data
    c = load_case("verify_toy")
    rec = mk.Blob.from_host(ctx, c.blob(4))
    rec.save(str(tmp_path / "rec.mlck"))
    with open(tmp_path / "rec.mlck", "rb") as f:
        raw = f.read()
    assert raw == c.blob(4)
    assert oracle.parse_record(raw, c.compute_bytes) == mk.parse_record(mk.Blob.load(ctx, str(tmp_path / "rec.mlck")),
                                                                         c.compute_bytes)
    with pytest.raises(RuntimeError, match="persist: cannot open"):
        mk.Blob.load(ctx, str(tmp_path / "missing.mlck"))


@pytest.mark.gpu
def test_replication_follows_the_device(mk, ctx):
    c = load_case("verify_toy")
    st = upload_state(mk, ctx, c, 4)
    out = mk.Blob(ctx, 1 << 16)
    assert out.replication() == 0  # nothing written yet
    reps = [ctx.alloc(1 << 16), ctx.alloc(1 << 16)]
    for r in reps:
        out.add_replica(r, 1 << 16)
    active, co = c.slot(1)
    mk.snapshot_record(st, active, co, 1, 1, 3, 3, out)
    ctx.synchronize()
    assert out.replication() == 2
    for r in reps:
        ctx.free(r)


@pytest.mark.gpu
def test_window_ring_end_to_end(mk, ctx, window, tmp_path):
    """Windows of real records: persisted once replicated (device replicas or
    durable files), saved, loaded back byte-exact and covering every operator."""
    c = load_case("verify_toy")
    W = c.W
    persisted = []
    ring = window.WindowRing(ctx, W, replication_target=1, on_persist=persisted.append)
    keep = []
    for s in range(2 * W):
        st = upload_state(mk, ctx, c, s)
        keep.append(st)
        blob = ring.acquire(1 << 16)
        if s < W:  # window 0 replicates to device buffers, window W does not
            blob.add_replica(ctx.alloc(1 << 16), 1 << 16)
        active, co = c.slot(s % W)
        mk.snapshot_record(st, active, co, s % W, 1, s // W * W, W, blob)
        ring.add_record(s, blob)
    ctx.synchronize()
    # window W has no replicas: only window 0 persists through the device
    assert ring.poll() and ring.persisted.window_start == 0 and persisted == [0]
    win = ring.in_flight[0]
    assert win.window_start == W and win.complete() and not win.persisted()
    # a durable file copy of each record counts toward the target
    d = str(tmp_path / "w")
    win.save(d)
    assert ring.poll() and ring.persisted.window_start == W and persisted == [0, W]
    assert len(ring._free) == W  # window 0's blobs are back in the pool
    loaded = window.SparseCheckpoint.load(ctx, d, replication_target=1)
    assert loaded.window_start == W and loaded.persisted()
    assert [b.to_host() for b in loaded.blobs] == [c.blob(s) for s in range(W, 2 * W)]
    loaded.check_coverage(c.n_ops, c.compute_bytes)
