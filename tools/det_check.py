"""Determinism probe: the same GA config several times in one process; prints
per-generation bests (compare across processes too).
python tools/det_check.py npts p nb nt gens population [repeats]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

npts, p, nb, nt, gens = (int(x) for x in sys.argv[1:6])
popmode = sys.argv[6]
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(npts, 12345, device="cuda"), npts, npts, p)
for _ in range(reps):
    r = ctx.run_ga(pm.ga_config(nb=nb, nt=nt, evolve_limit=gens, saturation=gens + 1, seed=1, population=popmode))
    print(popmode, r["best_cost"], list(r["per_kernel_best_costs"]))
