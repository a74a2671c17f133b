"""Localized recovery by recompute: per-target error vs the uninterrupted run."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_cases import load_case
from paper_2412_15411_b200 import mlck

def nerr(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    s = np.max(np.abs(b)); return float(np.max(np.abs(a - b)) / s) if s > 0 else float(np.max(np.abs(a - b)))

c = load_case("dp2_pp2")
ctx = mlck.Context(0)
eng = mlck.Engine(ctx, c.meta["cfg"])
log = mlck.UpstreamLog(ctx, 1 << 24, kind=1, device=0)
keys = []
for (it, mb, b, d), data in c.log_entries():
    p = ctx.upload(np.ascontiguousarray(data, np.float32)); log.put(it, mb, b, d, p, data.size); keys.append((it, mb, b, d))
log.sync()
print("log keys", sorted(set(k[0] for k in keys)), len(keys))
for w in (0, 2):
    for target in range(w + c.W, c.T + 1):
        for lo in (0, 1):
            blobs = [mlck.Blob.from_host(ctx, b) for b in c.window_blobs(w)]
            out = mlck.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
            eng.localized_recover(out, lo, lo, blobs, w, c.W, c.data_seed, log, target)
            errs = []
            for i in c.scope(lo, lo):
                got, want = out.download_op(i), c.op(target, i)
                errs.append(max(nerr(got.master, want["master"]), nerr(got.m, want["m"]), nerr(got.v, want["v"])))
            print("w", w, "target", target, "stage", lo, "max nerr vs run", max(errs), [round(e, 8) for e in errs])
