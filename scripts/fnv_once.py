"""One FNV launch over 256 MB of synthetic device bytes (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15411_b200 import mlck
ctx = mlck.Context(0)
n = 256 << 20
st = mlck.DeviceState(ctx, [n // 12], 4)
st.fill_synthetic(1, 1)
ptr = st.op_ptrs(0)[0]
for _ in range(3):
    h = ctx.fnv1a64(ptr, n)
print(hex(h))
