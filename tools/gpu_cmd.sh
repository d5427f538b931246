#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
python - <<'PY'
import sys, time
sys.path.insert(0, '.')
import paper_1610_10061_b200 as pm
from paper_1610_10061_b200 import synth
ctx = pm.Context(0)
ctx.set_instance(synth.euclid_costs(900, 12345, device="cuda"), 900, 900, 90)
for mode in ("device", "reference"):
    ctx.run_ga(pm.ga_config(nb=60, nt=256, evolve_limit=2, saturation=3, seed=2, population=mode))
    r = ctx.run_ga(pm.ga_config(nb=60, nt=256, evolve_limit=10, saturation=11, seed=1, population=mode))
    print(mode, "gens/s", r["kernels_executed"] / r["wall_time"], "evolve/gen ms", 1e3 * r["evolve_time"] / r["kernels_executed"])
PY
