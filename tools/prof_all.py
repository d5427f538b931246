"""Driver that launches every kernel of the library once at a BASELINE shape, for
one ncu capture of each (tools/profile_all.sh):
  * OR-Library-shaped graph, n=900 (pmed40's size): Floyd-Warshall closure
    kernels, then K1 (validation, sort, site-major transpose) via pm_set_instance_orlib;
  * the paper's GA shape (nb=60, nt=256, p=90): K3 kernels with the reference's
    exact population draw (k_unrank) and the device draw (k_draw_population);
  * syn5k: K2b gather (k_open_lists, k_gather), pm_min_cost_sum;
  * a payload-key instance (costs near 2^58): the tile-sort fallback k_build_rows.
python tools/prof_all.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402


def graph_text(n, extra, seed, wmax=100):
    """Random spanning tree plus extra edges (the shape of the OR-Library pmed graphs)."""
    rng = np.random.default_rng(seed)
    lines = []
    for v in range(2, n + 1):
        lines.append(f"{int(rng.integers(1, v))} {v} {int(rng.integers(1, wmax + 1))}")
    for _ in range(extra):
        u, v = rng.integers(1, n + 1, size=2)
        if u != v:
            lines.append(f"{int(u)} {int(v)} {int(rng.integers(1, wmax + 1))}")
    return f"{n} {len(lines)} 90\n" + "\n".join(lines) + "\n"


ctx = pm.Context(0)
ctx.set_instance_orlib(graph_text(900, 15300, 5))
for pop in ("reference", "device"):
    cfg = pm.ga_config(nb=60, nt=256, evolve_limit=2, saturation=3, seed=1, population=pop)
    r = ctx.run_ga(cfg)
    print("ga", pop, r["best_cost"], r["kernels_executed"])

n = m = 5000
ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, m, 50)
popw = synth.random_population(m, 50, 1024, seed=7)
words = torch.from_numpy(popw.view(np.int64)).cuda()
out = torch.empty(1024, dtype=torch.int64, device="cuda")
ctx.set_eval_kernel(pm.EVAL_GATHER)
ctx.evaluate_device(words, out, 1024, (m + 63) // 64, check=True)
print("min_cost_sum", int(ctx.min_cost_sum(popw[:64]).sum()))

big = (np.arange(7 * 300, dtype=np.int64).reshape(7, 300) * 7919 % 4093) + (1 << 58)
ctx.set_instance(torch.from_numpy(big).cuda(), 7, 300, 11)
assert ctx.table_info().dist_bytes == 8
torch.cuda.synchronize()
print("ok")
