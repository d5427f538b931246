"""Drive every kernel family once on small shapes against the bounds-checked
build (`make bounds`: device PMB_CHECKs trap on an index outside its buffer;
compute-sanitizer is not available on the GPU pool): K1 (counting-sort and
radix paths, wide-key payload path, heavy ties), K2 scan (split shapes and
the 24-warp variant), K2b gather, min_cost_sum, K3 evolve_blocks, run_ga with
the host and the device population draw, the OR-Library Floyd--Warshall
closure.  Results are still checked against the oracle.

  make bounds
  PMB_LIBRARY=$PWD/paper_1610_10061_b200/libpmedian_b200_bounds.so python tools/bounds_check.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1610_10061_b200 as pm  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from test_ingest import random_graph  # noqa: E402

o = Oracle()


def check_eval(ctx, n, m, p, costs, count, seed):
    so, inc = o.build_ordering(n, m, p, costs)
    got_so, got_inc = ctx.get_tables()
    assert (got_so == so).all() and (got_inc == inc).all(), (n, m, p)
    pop = o.random_population(m, p, count, seed=seed)
    rc, want, _, _ = o.evaluate(so, inc, m, pop)
    assert rc == 0
    for kind in (pm.EVAL_SCAN, pm.EVAL_GATHER):
        ctx.set_eval_kernel(kind)
        assert (ctx.evaluate(pop) == want).all(), (n, m, p, kind)
    ctx.set_eval_kernel(pm.EVAL_AUTO)
    assert (ctx.min_cost_sum(pop) == want).all()


def main():
    which = sys.argv[1:] or ["eval", "wide", "k1", "prep", "walks", "ga", "orlib"]
    with pm.Context(0) as ctx:
        if "eval" in which:
            for n, m, p, count in ((5, 4, 2, 3), (130, 200, 20, 100), (300, 300, 30, 256), (600, 700, 7, 70)):
                costs = o.synth_euclid(n) if n == m else o.random_costs(n + m, n, m, 1000)
                ctx.set_instance(costs, n, m, p)
                check_eval(ctx, n, m, p, costs, count, seed=n)
            print("eval ok", flush=True)
        if "wide" in which:
            # long CTA segments: the 24-warp K2 variant (one 768-thread CTA per SM)
            n = m = 4200
            p, count = 400, 4640
            costs = o.synth_euclid(n)
            ctx.set_instance(costs, n, m, p)
            so, inc = o.build_ordering(n, m, p, costs)
            pop = o.random_population(m, p, count, seed=11)
            rc, want, _, _ = o.evaluate(so, inc, m, pop)
            ctx.set_eval_kernel(pm.EVAL_SCAN)
            assert (ctx.evaluate(pop) == want).all()
            ctx.set_eval_kernel(pm.EVAL_AUTO)
            print("wide ok", flush=True)
        if "k1" in which:
            for k1 in ("count", "radix"):
                os.environ["PMB_K1"] = k1
                costs = o.random_costs(3, 70, 90, 1 << 40)  # wide keys: payload path
                ctx.set_instance(costs, 70, 90, 9)
                check_eval(ctx, 70, 90, 9, costs, 64, seed=5)
                costs = o.random_costs(4, 80, 120, 30)      # heavy ties
                ctx.set_instance(costs, 80, 120, 12)
                check_eval(ctx, 80, 120, 12, costs, 64, seed=6)
            os.environ.pop("PMB_K1")
            print("k1 ok", flush=True)
        if "prep" in which:
            # n * m > 2^20: the fused prep pass (u16 row copy with a padded
            # stride when m % 8 != 0, u16 site-major table), both K1 paths
            for n, m, p, mx in ((1100, 1100, 50, None), (1001, 1203, 40, 1000), (1030, 1030, 20, 70000)):
                costs = o.synth_euclid(n) if mx is None else o.random_costs(n + 7, n, m, mx)
                for k1 in ("count", "radix"):
                    os.environ["PMB_K1"] = k1
                    ctx.set_instance(costs, n, m, p)
                    check_eval(ctx, n, m, p, costs, 96, seed=m)
                os.environ.pop("PMB_K1")
            print("prep ok", flush=True)
        if "walks" in which:
            import torch
            n = m = 600
            costs = o.synth_euclid(n)
            ctx.set_instance(costs, n, m, 30)
            pop = o.random_population(m, 30, 100, seed=4)
            w = torch.from_numpy(pop.view(np.int64)).cuda()
            gs = torch.zeros(4, dtype=torch.int64, device="cuda")
            cm = torch.zeros(n, dtype=torch.int32, device="cuda")
            ctx.scan_walks_device(w, gs, cm, 100, pop.shape[1])
            so, inc = o.build_ordering(n, m, 30, costs)
            _, _, _, sk = o.evaluate(so, inc, m, pop, want_sum_k=True)
            assert int(gs.sum()) >= int(sk.max()) and int(cm.max()) <= m - 30 + 1
            print("walks ok", flush=True)
        if "ga" in which:
            n = m = 200
            costs = o.synth_euclid(n)
            ctx.set_instance(costs, n, m, 20)
            blocks = o.random_population(m, 20, 2 * 32, seed=9)
            cfg = pm.ga_config(nb=2, nt=32, seed=3)
            out, bc, bt = ctx.evolve_blocks(blocks, cfg, 1, 0)
            for b in range(2):
                assert ctx.evaluate(out[b * 32 + bt[b]][None, :])[0] == bc[b]
            for device_draw in (False, True):
                cfg = pm.ga_config(nb=4, nt=32, evolve_limit=3, saturation=10, seed=2,
                                   population="device" if device_draw else "reference")
                r = ctx.run_ga(cfg)
                assert ctx.evaluate(r["best"][None, :])[0] == r["best_cost"]
            print("ga ok", flush=True)
        if "orlib" in which:
            text = random_graph(5, 60, 90, oracle=o)
            ctx.set_instance_orlib(text, p=6)
            print("orlib ok", flush=True)
    print(f"bounds driver ok ({pm.LIB_PATH})")


if __name__ == "__main__":
    main()
