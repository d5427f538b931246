"""Timeline of the host-buffer evaluation call (pm_evaluate) at a BASELINE shape:
torch.profiler (CUPTI) records the library's copies and kernels; prints each
activity's start/end relative to the call's host entry.
python tools/e2e_timeline.py [syn20k|syn5k|pmed40] [calls]"""
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

cfg = bench.config_for(sys.argv[1] if len(sys.argv) > 1 else "syn20k")
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = m = cfg["npts"]
p, count = cfg["p"], cfg["count"]
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, m, p)
pop = synth.random_population(m, p, count, seed=7)
host = torch.from_numpy(pop.view(np.int64)).pin_memory().numpy().view(np.uint64)
for _ in range(3):
    ctx.evaluate(host)
torch.cuda.synchronize()
walls = []
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(calls):
        t0 = time.perf_counter()
        ctx.evaluate(host)
        walls.append((time.perf_counter() - t0) * 1e6)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t_first = ev[0].time_range.start if ev else 0
print("host wall per call (us):", ", ".join(f"{w:.1f}" for w in walls))
for e in ev:
    print(f"{e.time_range.start - t_first:10.1f} {e.time_range.end - t_first:10.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
