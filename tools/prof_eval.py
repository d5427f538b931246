"""Minimal driver for ncu captures: build one instance, evaluate one population
a few times with the chosen kernel.  python tools/prof_eval.py [config] [scan|gather|auto] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

cfg = bench.config_for(sys.argv[1] if len(sys.argv) > 1 else "syn20k")
kind = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = m = cfg["npts"]
p, count = cfg["p"], cfg["count"]
wp = (m + 63) // 64
ctx = pm.Context(0)
if kind != "auto":
    ctx.set_eval_kernel({"scan": pm.EVAL_SCAN, "gather": pm.EVAL_GATHER}[kind])
costs = synth.euclid_costs(n, 12345, device="cuda")
ctx.set_instance(costs, n, m, p)
del costs
pop = synth.random_population(m, p, count, seed=7)
words = torch.from_numpy(pop.view(np.int64)).cuda()
out = torch.empty(count, dtype=torch.int64, device="cuda")
for _ in range(reps):
    ctx.evaluate_device(words, out, count, wp, check=True)
torch.cuda.synchronize()
print("ok", cfg["workload"], kind, int(out[:4].sum().item()))
