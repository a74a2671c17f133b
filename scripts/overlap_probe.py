"""Development probe: does a memory-bound Adam kernel co-run with the hash
kernel (hash on one context stream, Adam on another)?  Prints the times of
each alone and of both launched together."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15411_b200 import mlck

a, b = mlck.Context(0), mlck.Context(0)
n = 1713239274
hs = mlck.DeviceState(a, [n // 12 + 1], 4)
hs.fill_synthetic(1, 1)
hptr = hs.op_ptrs(0)[0]
P = 200_000_000
st = mlck.DeviceState(b, [P], 4)
st.fill_synthetic(2, 3)
gs = mlck.DeviceState(b, [P], 4)
gs.fill_synthetic(3, 3)
w, m, v, _ = st.op_ptrs(0)
g = gs.op_ptrs(0)[0]
a.synchronize(); b.synchronize()


def adam():
    mlck.optimizer_step_adam(b, w, m, v, 5, g, P)


def run(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a.synchronize(); b.synchronize()
        t = time.perf_counter()
        fn()
        a.synchronize(); b.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


t_f = run(lambda: a.fnv1a64(hptr, n))
t_a = run(adam)


def both():
    adam()
    a.fnv1a64(hptr, n)


def both2():
    for _ in range(3):
        adam()
    a.fnv1a64(hptr, n)


t_c = run(both)
t_a3 = run(lambda: [adam() for _ in range(3)])
t_c3 = run(both2)
print(f"hash alone {t_f:.2f} ms, adam alone {t_a:.2f} ms, both {t_c:.2f} ms (sum {t_f + t_a:.2f}); "
      f"3 adams {t_a3:.2f}, 3 adams + hash {t_c3:.2f} (sum {t_f + t_a3:.2f})")
