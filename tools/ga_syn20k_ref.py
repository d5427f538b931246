import sys, time, os
sys.path.insert(0, os.getcwd())
import paper_1610_10061_b200 as pm
from paper_1610_10061_b200 import synth
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(20000, 12345, device="cuda"), 20000, 20000, 200)
for pop in ("reference", "device"):
    cfg = pm.ga_config(nb=16, nt=256, evolve_limit=10, saturation=11, seed=1, population=pop)
    t0 = time.perf_counter(); r = ctx.run_ga(cfg); t1 = time.perf_counter()
    r2 = ctx.run_ga(cfg); t2 = time.perf_counter()
    print(pop, "first run %.2fs" % (t1 - t0), "second %.2fs" % (t2 - t1), "gens/s %.2f" % (r2["kernels_executed"] / r2["wall_time"]), "best", r2["best_cost"], r["best_cost"] == r2["best_cost"])
