"""Development probe: the N > 1 snapshot step of bench.py (mixtral EP records,
ring replicas through CUDA IPC) with per-step pack / push / fnv timings per
rank, for transports 1 (copy engines beside the hash) and 4 (after the hash).

  torchrun --nproc-per-node 4 scripts/push_probe.py   [PROBE_BACKEND=gloo|nccl]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import bench
from paper_2412_15411_b200 import mlck, placement

world, rank, local = bench.dist_env()
backend = os.environ.get("PROBE_BACKEND", "gloo")
torch.cuda.set_device(local)
dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)} if backend == "nccl" else {}))


def all_gather(obj):
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


ctx = mlck.Context(local)
wl = bench.mixtral_ep() if world > 1 else bench.deepseek_layer()
slots = bench.schedule(wl)
sizes = [bench.record_bytes(wl, s) for s in slots]
cap = max(sizes)
r = min(2, world - 1) if world > 1 else 1
st = mlck.DeviceState(ctx, wl["param_counts"], wl["cb"])
st.fill_synthetic(seed=7 + rank, step=10)
st.set_meta(1000, 7)
W = wl["W"]
blobs = [mlck.Blob(ctx, cap) for _ in range(W)]
if world == 1:  # local replica per slot, as bench.py at N=1
    for b in blobs:
        b.add_replica(ctx.alloc(cap), cap)
else:
    recv = [ctx.alloc(cap) for _ in range(r)]
    targets = placement.exchange_handles(all_gather, [ctx.ipc_export(p) for p in recv], rank, world)
    for handle, _peer in targets:
        ptr = ctx.ipc_open(handle)
        for b in blobs:
            b.add_replica(ptr, cap)


def step(i):
    k = i % W
    a, c = slots[k]
    mlck.snapshot_record(st, a, c, k, 1, 1000, W, blobs[k])


for mode in [int(m) for m in os.environ.get("PROBE_MODES", "1,4,1").split(",")]:
    ctx.set_replica_mode(mode)
    for i in range(3):
        step(i)
    ctx.synchronize()
    dist.barrier()
    ctx.set_timing(True)
    samp = os.environ.get("PROBE_SAMPLER", "0")
    import contextlib
    cm = bench.ClockSampler(local) if samp == "all" or (samp == "0rank" and rank == 0) else contextlib.nullcontext()
    with cm:
        ctx.event_record(0)
        for i in range(8):
            step(i)
        ctx.event_record(1)
        ctx.synchronize()
    tim = ctx.timings()
    ctx.set_timing(False)
    ms = ctx.event_ms(0, 1) / 8
    by = {}
    for n, t in tim:
        by.setdefault(n, []).append(round(t, 2))
    gbs = [round(r * sizes[i % W] / (t / 1000) / 1e9) for i, t in enumerate(by.get("push", []))]
    print(f"[{backend}] rank {rank} mode {mode} step {ms:.2f} ms {by} push GB/s {gbs}", flush=True)
    dist.barrier()
dist.destroy_process_group()
