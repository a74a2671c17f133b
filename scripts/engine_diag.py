"""Diagnostics: GPU toy engine vs the golden reference, one iteration."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_cases import load_case
from paper_2412_15411_b200 import mlck

name = sys.argv[1] if len(sys.argv) > 1 else "verify_toy"
c = load_case(name)
ctx = mlck.Context(0)
eng = mlck.Engine(ctx, c.meta["cfg"])
print("cfg", c.meta["cfg"], "n_ops", c.n_ops, "P", c.meta["param_counts"][:8])
g = mlck.GradLog(ctx, c.meta["param_counts"], 4)
log = mlck.UpstreamLog(ctx, 1 << 24, kind=0)
s = 0
st = mlck.DeviceState(ctx, c.meta["param_counts"], c.compute_bytes)
for i in range(c.n_ops):
    o = c.op(s, i)
    st.upload_op(i, o["master"], o["m"], o["v"], o["step"])
st.set_meta(s, c.data_seed)
eng.run_iteration(st, log=log, gradlog=g)
for i in range(c.n_ops):
    P = c.meta["param_counts"][i]
    gd = np.frombuffer(ctx.download(g.slot(s + 1, i), 4 * P), np.float32)
    gw = c.grads(s + 1, i)
    d = np.abs(gd - gw)
    rel = d.max() / max(1e-30, np.abs(gw).max())
    bad = np.nonzero(gd != gw)[0]
    print(f"op {i} stage {eng.stage_of_op(i)} grad maxabs {np.abs(gw).max():.3e} maxdiff {d.max():.3e} rel {rel:.2e} "
          f"ndiff {bad.size} first {bad[:6].tolist()} got {gd[bad[:3]].tolist()} want {gw[bad[:3]].tolist()}")
got = dict(log.entries())
want = dict(c.log_entries()) if "log_keys" in c.d else {}
for k in sorted(want)[:6]:
    if k[0] != 1: continue
    print("log", k, "got" if k in got else "MISSING", None if k not in got else float(np.abs(got[k] - want[k]).max()))
