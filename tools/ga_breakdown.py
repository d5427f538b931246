"""Where a generation's time goes at the paper's GA shape (n=m=900, p=90, nb=60, nt=256):
run_ga with the crossover rounds and/or mutation attempts switched off, and the K2 launches
of one generation timed alone.  python tools/ga_breakdown.py [reference|device] [gens]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

popmode = sys.argv[1] if len(sys.argv) > 1 else "device"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 30
n, p, nb, nt = 900, 90, 60, 256
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, n, p)


def rate(**kw):
    cfg = pm.ga_config(nb=nb, nt=nt, evolve_limit=gens, saturation=gens + 1, seed=1, population=popmode, **kw)
    ctx.run_ga(cfg)  # warm-up
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        r = ctx.run_ga(cfg)
        best = min(best, (time.perf_counter() - t0) / r["kernels_executed"])
    return best * 1e3


full = rate()
nocx = rate(crossover_iters=0)
nomut = rate(mutation_iters=0)
none = rate(crossover_iters=0, mutation_iters=0)
print(f"{popmode}: ms/gen full {full:.3f}  no-crossover {nocx:.3f}  no-mutation {nomut:.3f}  neither {none:.3f}")
print(f"  crossover rounds {full - nocx:.3f} ms, mutation {full - nomut:.3f} ms, rest {none:.3f} ms")
# the evaluations of one generation alone: 9 batches of nb*nt and one of 8*nb*nt
wp = (n + 63) // 64
s = torch.cuda.Stream()
ctx.set_stream(s)
pop = synth.random_population(n, p, 8 * nb * nt, seed=7)
words = torch.from_numpy(pop.view(np.int64)).cuda()
out = torch.empty(8 * nb * nt, dtype=torch.int64, device="cuda")
with torch.cuda.stream(s):
    for _ in range(3):
        ctx.evaluate_device(words, out, nb * nt, wp, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        for _ in range(9):
            ctx.evaluate_device(words, out, nb * nt, wp, check=False)
        ctx.evaluate_device(words, out, 8 * nb * nt, wp, check=False)
    e1.record(s)
    torch.cuda.synchronize()
print(f"  evaluations of one generation alone (transpose + K2): {e0.elapsed_time(e1) / 10:.3f} ms")
