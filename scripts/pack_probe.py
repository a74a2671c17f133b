"""Development probe: pack kernel time for the bench's N=1 slot mix (record
plus one local replica), per variant library (MLCK_B200_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2412_15411_b200 import mlck

ctx = mlck.Context(0)
wl = bench.deepseek_layer()
slots = bench.schedule(wl)
sizes = [bench.record_bytes(wl, s) for s in slots]
cap = max(sizes)
st = mlck.DeviceState(ctx, wl["param_counts"], wl["cb"])
st.fill_synthetic(seed=7, step=10)
st.set_meta(1000, 7)
blobs = [mlck.Blob(ctx, cap) for _ in slots]
for b in blobs:
    b.add_replica(ctx.alloc(cap), cap)
for rep in range(2):
    ctx.set_timing(True)
    for i in range(12):
        a, c = slots[i % len(slots)]
        mlck.snapshot_record(st, a, c, i % len(slots), 1, 1000, len(slots), blobs[i % len(slots)])
    t = ctx.timings()
    ctx.set_timing(False)
pack = [ms for n, ms in t if n == "pack"]
fnv = [ms for n, ms in t if n == "fnv"]
print(f"pack {sum(pack) / len(pack):.3f} ms  fnv {sum(fnv) / len(fnv):.3f} ms")
