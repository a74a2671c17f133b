"""Multi-GPU host logic on CPU: expert sharding, ring replica placement and
the IPC-handle exchange, run under torch.distributed gloo with 2 and 4
processes (the data path itself has no collective)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_15411_b200 import placement as pl


def test_ring_targets_and_sources_are_inverse():
    for world in (1, 2, 3, 4, 8):
        r = pl.replicas(world)
        assert r == (0 if world == 1 else min(2, world - 1))
        for rank in range(world):
            for peer, j in pl.ring_targets(rank, world):
                assert peer != rank
                assert pl.ring_sources(peer, world)[j] == rank
        # every receive buffer has exactly one sender
        senders = sorted((p, j) for rank in range(world) for p, j in pl.ring_targets(rank, world))
        assert senders == sorted((p, j) for p in range(world) for j in range(r))


def test_expert_sharding_is_a_partition():
    E, layers, world = 64, 3, 8
    classes = (["E"] * E + ["NE", "G"]) * layers
    owned = [set(pl.shard_operators(classes, E, world, r)) for r in range(world)]
    assert set().union(*owned) == set(range(len(classes)))
    assert sum(len(o) for o in owned) == len(classes)
    assert all(len([i for i in o if classes[i] == "E"]) == E * layers // world for o in owned)


def test_shard_slot_restricts_public_slot():
    slot = ([0, 1, 2, 3], [4, 5, 6])
    assert pl.shard_slot(slot, {1, 3, 5}) == ([1, 3], [5])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = pl.replicas(world)
    local = [f"h{rank}.{j}".encode().ljust(64, b"\0") for j in range(r)]

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    got = pl.exchange_handles(all_gather, local, rank, world)
    # the handle I open on peer p must be the buffer p reserved for me
    ok = all(h.rstrip(b"\0") == f"h{p}.{pl.ring_sources(p, world).index(rank)}".encode() for h, p in got)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok, len(got)))


@pytest.mark.parametrize("world", [2, 4])
def test_handle_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert all(n == min(2, world - 1) for _, _, n in res)
