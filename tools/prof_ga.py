"""GA timing driver: python tools/prof_ga.py [syn20k|pmed40] [generations] [population]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "syn20k"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 3
popmode = sys.argv[3] if len(sys.argv) > 3 else "device"
n, p, nb = {"syn20k": (20000, 200, 16), "pmed40": (900, 90, 60), "pmed1": (100, 5, 60)}[cfgname]
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, n, p)
cfg = pm.ga_config(nb=nb, nt=256, evolve_limit=gens, saturation=gens + 1, seed=1, population=popmode)
reps = int(os.environ.get("PROF_GA_REPS", "1"))  # >1: the first run warms up (table, buffers)
for _ in range(reps):
    t0 = time.perf_counter()
    r = ctx.run_ga(cfg)
    dt = time.perf_counter() - t0
print(f"{cfgname} {popmode}: {r['kernels_executed']} gens in {dt:.3f}s ({r['kernels_executed']/r['wall_time']:.2f} gens/s, "
      f"evolve {r['evolve_time']:.3f}s) best {r['best_cost']}")
