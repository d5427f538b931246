"""K1 timing: set_instance (validation + build_ordering + site-major transpose) on a device
cost matrix, best of 3 wall times.  python tools/time_k1.py [npts] ; PMB_K1=radix forces the radix path."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
p = max(1, n // 100)
costs = synth.euclid_costs(n, 12345, device="cuda")
ctx = pm.Context(0)
best = 1e9
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.set_instance(costs, n, n, p)
    best = min(best, time.perf_counter() - t0)
so, inc = ctx.get_tables()
h = hash(so[:50].tobytes()) ^ hash(inc[-50:].tobytes())
print(f"n=m={n} K1={os.environ.get('PMB_K1', 'auto')}: set_instance {best * 1e3:.2f} ms  tables-hash {h & 0xffffffff:08x}")
