"""Regression tests for the round-1 advisor findings, each against
the oracle or the reference's semantics:

* K1's radix kernel with zero radix passes (an all-zero cost matrix, m > 64:
  the counting sort hands the one m-site bucket back to it);
* K1's payload-key kernel over rows longer than one 1024-element tile (the
  digit-count clearing race);
* run_ga with an evolve_limit far above what saturation lets it reach (the
  per-kernel bests grow with the run, nothing is sized by evolve_limit);
* scan and gather launches over more than 65535 x 64 chromosomes (the grid's
  y limit).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _eval(ctx, pm, pop, kind):
    ctx.set_eval_kernel(kind)
    try:
        return ctx.evaluate(pop)
    finally:
        ctx.set_eval_kernel(pm.EVAL_AUTO)


def test_all_zero_costs_zero_radix_passes(ctx, pm, oracle):
    n, m, p = 9, 300, 10
    costs = np.zeros(n * m, dtype=np.int64)
    ctx.set_instance(costs, n, m, p)
    so, inc = oracle.build_ordering(n, m, p, costs)
    so2, inc2 = ctx.get_tables()
    assert (so == so2).all() and (inc == inc2).all()  # site order 0..W-1 in every row
    pop = oracle.random_population(m, p, 64, seed=2)
    for kind in (pm.EVAL_SCAN, pm.EVAL_GATHER):
        assert (_eval(ctx, pm, pop, kind) == 0).all()


def test_payload_keys_across_tiles(ctx, pm, oracle):
    n, m, p = 5, 3000, 30
    base = oracle.random_costs(21, n, m, 7)
    costs = (base.astype(np.int64) << np.int64(58)) // 5 + base  # ~2^60: payload keys, many ties
    ctx.set_instance(costs, n, m, p)
    assert ctx.table_info().dist_bytes == 8
    so, inc = oracle.build_ordering(n, m, p, costs)
    so2, inc2 = ctx.get_tables()
    assert (so == so2).all() and (inc == inc2).all()
    pop = oracle.random_population(m, p, 40, seed=6)
    want = oracle.evaluate(so, inc, m, pop)[1]
    for kind in (pm.EVAL_SCAN, pm.EVAL_GATHER):
        assert (_eval(ctx, pm, pop, kind) == want).all()


def test_run_ga_huge_evolve_limit_stops_on_saturation(ctx, pm, oracle):
    n = m = 60
    ctx.set_instance(oracle.synth_euclid(n, seed=3), n, m, 6)
    r = ctx.run_ga(pm.ga_config(nb=2, nt=8, evolve_limit=10**9, saturation=3, seed=11))
    k = int(r["kernels_executed"])
    assert 3 <= k < 10**6
    assert len(r["per_kernel_best_costs"]) == k
    pk = np.asarray(r["per_kernel_best_costs"])
    assert pk.min() == r["best_cost"]


def test_more_than_65535_groups(ctx, pm, oracle):
    """4,200,000 chromosomes of one word: 65,625 64-chromosome groups for the
    scan's transpose and more than 65535 chromosome rows for the gather."""
    n, m, p = 6, 64, 3
    costs = oracle.random_costs(5, n, m, 1000)
    ctx.set_instance(costs, n, m, p)
    so, inc = oracle.build_ordering(n, m, p, costs)
    count = 4_200_000
    pop = oracle.random_population(m, p, count, seed=7)  # exactly p open sites each
    rc, want, _, _ = oracle.evaluate(so, inc, m, pop)
    assert rc == 0
    for kind in (pm.EVAL_SCAN, pm.EVAL_GATHER):
        assert np.array_equal(_eval(ctx, pm, pop, kind), want), kind
