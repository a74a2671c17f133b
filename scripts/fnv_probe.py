"""Development probe: FNV kernel throughput and its profile counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_15411_b200 import mlck

ctx = mlck.Context(0)
for mb in (16, 256, 1024):
    n = mb << 20
    st = mlck.DeviceState(ctx, [n // 12], 4)
    st.fill_synthetic(1, 1)
    ptr = st.op_ptrs(0)[0]
    ctx.synchronize()
    h0 = ctx.fnv1a64(ptr, n)
    ctx.event_record(0)
    reps = 3
    for _ in range(reps):
        ctx.fnv1a64(ptr, n)
    ctx.event_record(1)
    ms = ctx.event_ms(0, 1) / reps
    h1, prof = ctx.fnv1a64_profile(ptr, n)
    ch = max(1, prof["chunks"])
    print(f"{mb} MB: {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s  same={h0 == h1}  per-chunk: "
          f"probes {prof['lookback_probes'] / ch:.2f} spins {prof['spin_rereads'] / ch:.1f} "
          f"thread0 cycles/chunk: rounds {prof['cycles_rounds'] / ch:.0f} wait {prof['cycles_wait'] / ch:.0f} "
          f"final {prof['cycles_final'] / ch:.0f} other {prof['cycles_other'] / ch:.0f} "
          f"| lb: idle {prof['lb_idle'] / ch:.0f} probe {prof['lb_probe'] / ch:.0f} "
          f"spin {prof['lb_spin'] / ch:.0f} compose {prof['lb_compose'] / ch:.0f} pub {prof['lb_publish'] / ch:.0f} "
          f"total {prof['lb_total'] / ch:.0f}")
    print("   compute detail/chunk: refill %.0f data_wait %.0f final_hash %.0f" % tuple(
        prof[k] / ch for k in ["cyc_refill", "cyc_data_wait", "cyc_final_hash"]))
    st.close()

# per-chunk trace on 64 MB
n = 64 << 20
CH = int(os.environ.get("FNV_CHUNK", "65536"))
st = mlck.DeviceState(ctx, [n // 12], 4)
st.fill_synthetic(1, 1)
ptr = st.op_ptrs(0)[0]
chunks = (n + CH - 1) // CH
tr = np.zeros(chunks * 12, dtype=np.uint64)
ctx.fnv1a64_profile(ptr, n, trace=tr)
tr = tr.reshape(chunks, 12).astype(np.int64)
t0 = tr[:, 0].min()
np.set_printoptions(linewidth=200)
print("columns: start, agg0, res0, agg1, res1, agg2, res2, agg3, res3, end (us rel. to first start), sm")
for c in [c for c in list(range(0, 8)) + list(range(1000, 1008)) + list(range(3000, 3004)) if c < chunks]:
    row = tr[c]
    print(c, [(int(x - t0) // 100) / 10 for x in row[:10]], int(row[10]))
dur = (tr[:, 9] - tr[:, 0]) / 1000
print("chunk lifetime us: median %.1f p90 %.1f max %.1f" % (np.median(dur), np.percentile(dur, 90), dur.max()))
for r in range(4):
    w = (tr[:, 2 + 2 * r] - tr[:, 1 + 2 * r]) / 1000
    c = (tr[:, 1 + 2 * r] - (tr[:, 2 * r] if r else tr[:, 0])) / 1000
    print(f"round {r}: compute-to-publish median {np.median(c):.2f} us, lookback wait median {np.median(w):.2f} us p90 {np.percentile(w, 90):.2f}")
# dependency: time res(c, r) vs agg(c-1, r)
lag = (tr[1:, 2] - tr[:-1, 1]) / 1000
print("res0(c) - agg0(c-1) median %.2f us" % np.median(lag))
# wave analysis (slot-major order: wave = G consecutive chunks)
G = int(os.environ.get("FNV_GRID", "148"))
for w in [3, 6, 9, 12]:
    if (w + 1) * G > chunks:
        break
    rows = tr[w * G:(w + 1) * G]
    for r in range(4):
        agg = (rows[:, 1 + 2 * r] - t0) / 1000
        res = (rows[:, 2 + 2 * r] - t0) / 1000
        print(f"wave {w} round {r}: agg min {agg.min():.1f} med {np.median(agg):.1f} max {agg.max():.1f} "
              f"(argmax cta {int(np.argmax(agg))}) | res min {res.min():.1f} med {np.median(res):.1f} max {res.max():.1f}")
# one SM's chunks: the turn structure (times relative to the first start, us)
sm = int(tr[100, 10])
rows = tr[tr[:, 10] == sm]
rows = rows[np.argsort(rows[:, 0])]
print(f"SM {sm}: chunk events (start, agg0, res0, agg1, res1, agg2, res2, agg3, res3, end)")
for rw in rows[:9]:
    print([round((int(x) - t0) / 1000, 1) for x in rw[:10]])
