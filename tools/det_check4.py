"""evolve_blocks at the paper's GA shape (60 x 256, 900/90) against the
reference's evolve_block, block by block; reports mismatching blocks/threads."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_10061_b200 as pm  # noqa: E402
from oracle.oracle import RefLib  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

npts, p, nb, nt = 900, 90, 60, 256
cx = int(sys.argv[1]) if len(sys.argv) > 1 else -1
mu = int(sys.argv[2]) if len(sys.argv) > 2 else -1
costs = synth.euclid_costs(npts, 12345)
ctx = pm.Context(0)
ctx.set_instance(costs, npts, npts, p)
ri = RefLib().create(npts, npts, p, costs)
blocks = synth.random_population(npts, p, nb * nt, seed=9)
cfg = pm.ga_config(nb=nb, nt=nt, seed=1, crossover_iters=None if cx < 0 else cx, mutation_iters=None if mu < 0 else mu)
got, bc, bt = ctx.evolve_blocks(blocks, cfg, 0)
bad = []
for b in range(nb):
    rc, want, wbest, wcost, wthread = ri.evolve_block(blocks[b * nt:(b + 1) * nt], nt, nb, 1, 0, b, cx, mu)
    diff = np.nonzero((got[b * nt:(b + 1) * nt] != want).any(axis=1))[0]
    if len(diff) or bc[b] != wcost:
        bad.append((b, list(diff[:8]), int(bc[b]), wcost))
print("cx", cx, "mu", mu, "mismatching blocks:", len(bad), bad[:5])
