"""Multi-GPU replica placement on real devices: each rank packs
its expert shard's record (`take_sparse_snapshot` on `slot ∩ shard`,
`snapshot.hpp:204-241`) and the replicas land in its ring peers' HBM over
NVLink (CUDA IPC, `placement.ring_targets`).  Every peer's copy must equal the
sender's record byte for byte, under every replica transport; the record must
equal the oracle's serialize_record of the same shard state, and its trailer
the CPU oracle's FNV-1a-64 (`digest.hpp:18-25`).

One process per GPU; gloo carries only the IPC handles and the host copies the
checker compares (the data path itself has no collective).  The "2rank-1gpu"
cases put two ranks on one GPU (CUDA IPC between processes on the same
device): the same handle exchange, ring placement, capacity checks, witness
travel and mapping teardown, so a single-GPU run exercises the protocol too.

CASES: (world, devices)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

E = 8  # experts per layer (configs[0] shape), sizes not multiples of 4 so payloads sit at odd offsets


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _record_bytes(pcs, a, c, cb):
    return 45 + 8 + sum(13 + 8 + 12 * pcs[i] for i in a) + sum(13 + cb * pcs[i] for i in c)


CASES = [(2, 2), (4, 4), (2, 1)]
IDS = ["2gpu", "4gpu", "2rank-1gpu"]


def _worker(rank, world, port, q, ndev):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok, msg, cur_mode = True, "", None
    try:
        from oracle.oracle import Oracle
        from paper_2412_15411_b200 import mlck
        from paper_2412_15411_b200 import placement as pl

        cb = 2
        classes = ["E"] * E + ["NE", "G"]
        pcs = [40_001 + 4_099 * i for i in range(E)] + [70_003, 517]
        owned = pl.shard_operators(classes, E, world, rank)
        ctx = mlck.Context(rank % ndev)
        st = mlck.DeviceState(ctx, pcs, cb)
        st.fill_synthetic(seed=11, step=3)
        st.set_meta(40, 11)
        active = owned[:2]
        compute_only = owned[2:]
        # one capacity for every rank's buffers: a sender's record must fit its peers' receive buffers
        cap = _record_bytes(pcs, range(len(pcs)), [], cb) + 4096
        r = pl.replicas(world)
        recv = [ctx.alloc(cap) for _ in range(r)]

        def all_gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        targets = pl.exchange_handles(all_gather, [ctx.ipc_export(p) for p in recv], rank, world)
        opened = [ctx.ipc_open(h) for h, _peer in targets]
        # a replica claiming more than the peer allocated is refused before any write
        probe = mlck.Blob(ctx, 256)
        try:
            probe.add_replica(opened[0], cap + (8 << 20))
            ok, msg = False, f"rank {rank}: oversized replica capacity accepted"
        except mlck.MlckInvalid as e:
            if "exceeds its IPC mapping" not in str(e):
                ok, msg = False, f"rank {rank}: unexpected error text: {e}"
        probe.close()
        blob = mlck.Blob(ctx, cap)
        for p in opened:
            blob.add_replica(p, cap)
        orc = Oracle()
        # the shard record the reference's take_sparse_snapshot + serialize_record makes from the same
        # state on slot ∩ shard (fill_synthetic follows the oracle's synth streams 3i, 3i+1, 3i+2)
        ents = []
        for i in sorted(active + compute_only):
            P = pcs[i]
            master = orc.synth(11, 3 * i, -0.25, 0.25, P)
            if i in active:
                ents.append(dict(id=i, mode=0, param_count=P, step=3, master=master,
                                 m=orc.synth(11, 3 * i + 1, -1e-3, 1e-3, P), v=orc.synth(11, 3 * i + 2, 0.0, 1e-6, P)))
            else:
                ents.append(dict(id=i, mode=1, param_count=P, compute=orc.quantize(master, cb)))
        ref = orc.serialize_record(dict(kind=1, iteration=40, window_start=36, wsparse=4, slot=1, data_seed=11),
                                   ents, cb)
        for mode in (-1, 0, 1, 2, 3, 4, 5):
            cur_mode = mode
            for p in recv:
                ctx.memset(p, 0, cap)
            ctx.synchronize()
            dist.barrier()
            ctx.set_replica_mode(mode)
            mlck.snapshot_record(st, active, compute_only, 1, 1, 36, 4, blob)
            ctx.synchronize()
            dist.barrier()  # every sender's stores are complete before anyone reads
            mine = blob.to_host()
            assert len(mine) == _record_bytes(pcs, active, compute_only, cb)
            if mine != ref:
                ok, msg = False, f"mode {mode}: rank {rank} record differs from the reference's shard record"
            trailer = int.from_bytes(mine[-8:], "little")
            if trailer != orc.fnv1a64(np.frombuffer(mine[:-8], dtype=np.uint8)):
                ok, msg = False, f"mode {mode}: rank {rank} trailer differs from the oracle FNV"
            records = all_gather(mine)
            for j, src in enumerate(pl.ring_sources(rank, world)):
                want = records[src]
                if ctx.download(recv[j], len(want)) != want:
                    ok, msg = False, f"mode {mode}: rank {rank} replica {j} of rank {src} differs"
            dist.barrier()
        ctx.set_replica_mode(-1)
        # witnesses travel with the replicas (mlck_blob_add_replica_witness): a rank
        # verifies a peer's record on the witnessed path, straight from its inbound buffer
        wcap = mlck.witness_bytes(cap)
        recv_w = [ctx.alloc(wcap) for _ in range(r)]
        wtargets = pl.exchange_handles(all_gather, [ctx.ipc_export(p) for p in recv_w], rank, world)
        opened_w = [ctx.ipc_open(h) for h, _peer in wtargets]
        for p in opened_w:
            blob.add_replica_witness(p, wcap)
        mlck.snapshot_record(st, active, compute_only, 1, 1, 36, 4, blob)
        ctx.synchronize()
        dist.barrier()
        sizes = all_gather(blob.size)
        for j, src in enumerate(pl.ring_sources(rank, world)):
            view = mlck.Blob.wrap(ctx, recv[j], sizes[src], recv_w[j])
            used0, fb0 = ctx.witness_stats()
            mlck.parse_record(view, cb)
            used, fb = ctx.witness_stats()
            if not (used > used0 and fb == fb0):
                ok, msg = False, f"rank {rank}: replica {j} of rank {src} did not verify on its witness"
            view.close()
        dist.barrier()  # every peer is done reading its inbound buffers
        for p in opened_w:
            ctx.ipc_close(p)
        # closing the mappings drops the blob's replicas inside them: the next
        # record stays local instead of storing to unmapped memory
        for p in opened:
            ctx.ipc_close(p)
        mlck.snapshot_record(st, active, compute_only, 1, 1, 36, 4, blob)
        if blob.to_host() != ref or blob.replication() != 0:
            ok, msg = False, f"rank {rank}: replicas inside a closed IPC mapping were kept"
        blob.close()
        dist.barrier()
    except Exception as e:  # report, do not hang the other ranks' queue reads
        ok, msg = False, f"rank {rank}, mode {cur_mode}: {type(e).__name__}: {e}"
    q.put((rank, ok, msg))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ndev", CASES, ids=IDS)
def test_ring_replicas_byte_exact(world, ndev):
    if torch.cuda.device_count() < ndev:
        pytest.skip(f"needs {ndev} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, ndev)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [m for _, ok, m in res if not ok]
    assert not bad, bad


def _log_worker(rank, world, port, q, ndev):
    """Upstream logging into the ring successor's HBM (kind 2 over an IPC
    mapping, what bench.py's N>1 logging does): the entries read back through
    the log equal the reference's UpstreamLog bit for bit (engine.hpp:55-94)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok, msg = True, ""
    try:
        from golden_cases import load_case
        from paper_2412_15411_b200 import mlck

        ref = load_case("dp2_pp2").log_entries()
        cap = 1 << 22
        ctx = mlck.Context(rank % ndev)
        mine = ctx.alloc(cap)  # this rank hosts its predecessor's log
        handles = [None] * world
        dist.all_gather_object(handles, ctx.ipc_export(mine))
        peer = ctx.ipc_open(handles[(rank + 1) % world])
        log = mlck.UpstreamLog(ctx, cap, kind=2, external=peer)
        bufs = []
        for j in np.random.default_rng(rank).permutation(len(ref)):
            key, data = ref[j]
            p = ctx.upload(data)
            bufs.append(p)
            log.put(*key, p, data.size)
        log.sync()
        got = log.entries()
        if [k for k, _ in got] != [k for k, _ in ref]:
            ok, msg = False, f"rank {rank}: key order differs"
        elif not all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for (_, a), (_, b) in zip(got, ref)):
            ok, msg = False, f"rank {rank}: entry bytes differ"
        log.close()
        dist.barrier()
        for p in bufs:
            ctx.free(p)
        ctx.ipc_close(peer)
        dist.barrier()
    except Exception as e:
        ok, msg = False, f"rank {rank}: {type(e).__name__}: {e}"
    q.put((rank, ok, msg))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ndev", CASES, ids=IDS)
def test_upstream_log_in_peer_hbm(world, ndev):
    if torch.cuda.device_count() < ndev:
        pytest.skip(f"needs {ndev} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_log_worker, args=(r, world, port, q, ndev)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [m for _, ok, m in res if not ok]
    assert not bad, bad
