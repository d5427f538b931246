"""k_scan2 (two clients per lane) vs the default K2: identical costs, kernel times.
python tools/scan2_check.py [config] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

cfg = bench.config_for(sys.argv[1] if len(sys.argv) > 1 else "syn20k")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = m = cfg["npts"]
p, count = cfg["p"], cfg["count"]
wp = (m + 63) // 64
ctx = pm.Context(0)
ctx.set_eval_kernel(pm.EVAL_SCAN)
s = torch.cuda.Stream()
ctx.set_stream(s)
ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, m, p)
pop = synth.random_population(m, p, count, seed=7)
words = torch.from_numpy(pop.view(np.int64)).cuda()
out = torch.empty(count, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for rnd in range(2):
    for v in ("0", "12", "16", "0"):
        os.environ["PMB_SCAN2"] = v
        with torch.cuda.stream(s):
            ctx.evaluate_device(words, out, count, wp, check=True)
            res.setdefault(v, out.clone())
            ctx.set_profiling(True)
            ctx.profile_read()
            for _ in range(reps):
                flush.zero_()
                ctx.evaluate_device(words, out, count, wp, check=False)
            ms, nl = ctx.profile_read()
            ctx.set_profiling(False)
        ctx.check_errors()
        same = torch.equal(res[v], res["0"])
        print(f"{cfg['workload'][:6]} PMB_SCAN2={v:>2}: {ms / nl:.4f} ms  same_as_default={same}", flush=True)
