"""BASELINE config 5: p sweep at n=m=10000 -- scan vs gather kernel time, the AUTO
choice, evals/s and the SURVEY 8(d) roofline fraction per p.  Prints a markdown
table (profiles/r01_p_sweep.md).  python tools/sweep.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
peak, src = bench.peaks()
n = m = 10000
count = 4096
wp = (m + 63) // 64
costs = synth.euclid_costs(n, 12345, device="cuda")
ctx = pm.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
print(f"| p | E[k*] meas. | B_eval (MB) | scan ms | gather ms | AUTO | evals/s (AUTO) | roofline frac (of {peak:.0f} GB/s, {src.split()[0]}) |")
print("|---|---|---|---|---|---|---|---|")
rows = []
for p in (10, 20, 50, 100, 200, 500, 1000):
    ctx.set_instance(costs, n, m, p)
    pop = synth.random_population(m, p, count, seed=7)
    words = torch.from_numpy(pop.view(np.int64)).cuda()
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    sumk = torch.empty(count, dtype=torch.int64, device="cuda")
    ctx.scan_depths_device(words, sumk, count, wp)
    ksum = int(sumk.sum().item())
    b_eval = (12 * ksum + 8 * wp * count) / count
    t = {}
    res = {}
    for kind, k in (("scan", pm.EVAL_SCAN), ("gather", pm.EVAL_GATHER)):
        ctx.set_eval_kernel(k)
        with torch.cuda.stream(s):
            ctx.evaluate_device(words, out, count, wp, check=True)
            res[kind] = out.clone()
            ctx.set_profiling(True)
            ctx.profile_read()
            for _ in range(reps):
                flush.zero_()
                ctx.evaluate_device(words, out, count, wp, check=False)
            ms, nl = ctx.profile_read()
            ctx.set_profiling(False)
        t[kind] = ms / nl
    assert torch.equal(res["scan"], res["gather"])
    auto = "scan" if ctx.auto_eval_kernel() == 1 else "gather"
    ctx.set_eval_kernel(pm.EVAL_AUTO)
    ev = count / (t[auto] / 1e3)
    frac = ev * b_eval / (peak * 1e9)
    rows.append(dict(p=p, mean_kstar=ksum / count / n, b_eval_mb=b_eval / 1e6, scan_ms=t["scan"],
                     gather_ms=t["gather"], auto=auto, evals_per_s=ev, roofline_frac=frac))
    print(f"| {p} | {ksum / count / n:.2f} | {b_eval / 1e6:.3f} | {t['scan']:.3f} | {t['gather']:.3f} | {auto} | "
          f"{ev:,.0f} | {frac:.2f} |", flush=True)
print("\n```json\n" + json.dumps(rows) + "\n```")
