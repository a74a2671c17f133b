"""Host-side placement for the multi-GPU checkpoint path.

* Expert parallelism: expert e of a layer goes to GPU e*G//E (contiguous
  blocks); non-expert and gate operators live on GPU 0.
* Replica placement: every GPU pushes its record to r = min(2, G-1) ring
  successors (g+1, g+2 mod G) -- the paper's r=2 replication (PAPER.md:364,
  snapshot.hpp:303 replication_target).  Each GPU hosts one receive buffer
  per ring predecessor; buffer j on GPU p receives from sender p-(j+1).
* The only exchange is the receive buffers' CUDA IPC handles (all_gather of
  64-byte handles); no collective touches the data.
"""
from __future__ import annotations


def replicas(world: int) -> int:
    return 0 if world <= 1 else min(2, world - 1)


def ring_targets(rank: int, world: int) -> list[tuple[int, int]]:
    """(peer rank, receive-buffer index on that peer) for each replica."""
    return [((rank + k) % world, k - 1) for k in range(1, replicas(world) + 1)]


def ring_sources(rank: int, world: int) -> list[int]:
    """Sender rank of each local receive buffer (index j)."""
    return [(rank - (j + 1)) % world for j in range(replicas(world))]


def expert_owner(expert: int, experts: int, world: int) -> int:
    return expert * world // experts


def shard_operators(op_classes: list[str], experts_per_layer: int, world: int, rank: int) -> list[int]:
    """Operator ids (layer-major: E experts, NE, G per layer; core.hpp:105-134)
    owned by `rank`."""
    out = []
    for i, cls in enumerate(op_classes):
        layer_pos = i % (experts_per_layer + 2)
        if cls == "E":
            if expert_owner(layer_pos, experts_per_layer, world) == rank:
                out.append(i)
        elif rank == 0:
            out.append(i)
    return out


def shard_slot(slot: tuple[list[int], list[int]], owned: set[int]) -> tuple[list[int], list[int]]:
    """The shard record: take_sparse_snapshot(engine, ScheduleSlot{active & shard,
    compute_only & shard}, k) -- public-API restriction, so shard parity is exact."""
    a, c = slot
    return [i for i in a if i in owned], [i for i in c if i in owned]


def exchange_handles(all_gather, local_handles: list[bytes], rank: int, world: int) -> list[tuple[bytes, int]]:
    """Gather every rank's receive-buffer handles; return (handle, peer) for
    this rank's replica targets, in replica order."""
    table = all_gather(local_handles)
    return [(table[peer][j], peer) for peer, j in ring_targets(rank, world)]
