"""GPU edge cases beyond the reference's own tests: over-filled chromosomes
(popcount > p takes the gather kernel's general path), all-open chromosomes,
single-client / two-site instances, populations that are not a multiple of the
group width, and asynchronous device calls reporting errors later."""
import numpy as np
import pytest

from oracle.oracle import words_per

pytestmark = pytest.mark.gpu


def _overfilled(oracle, m, p, count, seed):
    pop = oracle.random_population(m, min(m - 1, 2 * p + 5), count, seed=seed)
    pop[0] = 0
    for j in range(m):  # all sites open
        pop[0, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
    return pop


@pytest.mark.parametrize("n,m,p", [(40, 300, 10), (25, 70, 30), (1, 2, 1), (3, 64, 63), (200, 1000, 3)])
def test_overfilled_and_tiny(ctx, pm, oracle, n, m, p):
    costs = oracle.random_costs(n + m, n, m, 1000)
    ctx.set_instance(costs, n, m, p)
    so, inc = oracle.build_ordering(n, m, p, costs)
    for count in (1, 31, 33, 97):
        pop = _overfilled(oracle, m, p, count, seed=count)
        rc, want, _, _ = oracle.evaluate(so, inc, m, pop)
        assert rc == 0
        for kind in (pm.EVAL_SCAN, pm.EVAL_GATHER, pm.EVAL_AUTO):
            ctx.set_eval_kernel(kind)
            assert (ctx.evaluate(pop) == want).all(), (kind, count)
        ctx.set_eval_kernel(pm.EVAL_AUTO)
        mcs = ctx.min_cost_sum(pop)
        assert all(mcs[r] == oracle.min_cost_sum(n, m, costs, pop[r])[1] for r in range(count))


def test_async_device_call_reports_later(ctx, pm, oracle):
    import torch
    n = m = 200
    p = 20
    ctx.set_instance(oracle.synth_euclid(n), n, m, p)
    pop = oracle.random_population(m, p, 64)
    pop[40] = 0
    w = torch.from_numpy(pop.view(np.int64)).cuda()
    out = torch.empty(64, dtype=torch.int64, device="cuda")
    ctx.evaluate_device(w, out, 64, words_per(m), check=False)  # returns without synchronising
    with pytest.raises(pm.ContractError) as ei:
        ctx.check_errors()
    assert ei.value.first_bad == 40
    ctx.check_errors()  # the error word was reset


def test_min_cost_sum_needs_an_open_site(ctx, pm, oracle):  # instance.cpp:37
    ctx.set_instance(oracle.random_costs(3, 4, 10, 9), 4, 10, 3)
    pop = np.zeros((3, 1), dtype=np.uint64)
    pop[0, 0] = 1
    pop[2, 0] = 4
    with pytest.raises(pm.ContractError, match="at least one site must be open") as ei:
        ctx.min_cost_sum(pop)
    assert ei.value.first_bad == 1
