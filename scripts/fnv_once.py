"""Development: one FNV launch over N MB of synthetic state (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_15411_b200 import mlck

ctx = mlck.Context(0)
n = int(sys.argv[1] if len(sys.argv) > 1 else 256) << 20
st = mlck.DeviceState(ctx, [n // 12], 4)
st.fill_synthetic(1, 1)
ptr = st.op_ptrs(0)[0]
for _ in range(3):
    h = ctx.fnv1a64(ptr, n)
ctx.synchronize()
print(hex(h))
