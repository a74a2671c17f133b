"""Stress: many fused snapshots (transport 2) of a DeepSeek-MoE-layer-shaped
state, every record's trailer and every 25th record's bytes (and its local
replica) compared with the same slot's record built by transport 0 (the
pack kernel + FNV kernel: independent code paths).  Prints one JSON line."""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_15411_b200 import mlck  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 600
wl = bench.deepseek_layer()
pcs, cb, W = wl["param_counts"], wl["cb"], wl["W"]
slots = bench.schedule(wl)
ctx = mlck.Context(0)
st = mlck.DeviceState(ctx, pcs, cb)
st.fill_synthetic(seed=7, step=10)
st.set_meta(1000, 7)
cap = max(bench.record_bytes(wl, s) for s in slots) + 4096
ctx.set_replica_mode(0)
ref = []
for k in range(W):
    a, c = slots[k]
    b = mlck.snapshot_record(st, a, c, k, 1, 1000, W)
    host = b.to_host()
    ref.append((hashlib.sha256(host).hexdigest(), host[-8:], len(host)))
    b.close()
ctx.set_replica_mode(2)
blob = mlck.Blob(ctx, cap)
rep = ctx.alloc(cap)
blob.add_replica(rep, cap)
bad, full = 0, 0
t0 = time.time()
for i in range(iters):
    k = i % W
    a, c = slots[k]
    mlck.snapshot_record(st, a, c, k, 1, 1000, W, blob)
    n = ref[k][2]
    if ctx.download(blob.device_ptr + n - 8, 8) != ref[k][1]:
        bad += 1
    if i % 25 == 0:
        full += 1
        if hashlib.sha256(blob.to_host()).hexdigest() != ref[k][0]:
            bad += 1
        if hashlib.sha256(ctx.download(rep, n)).hexdigest() != ref[k][0]:
            bad += 1
print(json.dumps({"iterations": iters, "full_compares": full, "mismatches": bad, "seconds": time.time() - t0}))
