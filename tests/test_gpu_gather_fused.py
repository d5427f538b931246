"""The fused gather (gather.cu k_gather_fused: one CTA per chromosome, lists in
shared memory, error word handed over by the last CTA) against the oracle.

Beyond the costs it checks the error handoff the fusion introduced: the lowest
failing chromosome of a call (ordering.cpp:50-52 runoff, instance.cpp:32-48
no open site), the context word re-armed for the next call, the sticky word of
the asynchronous device API, and the per-chunk slots of a pipelined host call.
"""
import numpy as np
import pytest

from oracle.oracle import open_to_words

pytestmark = pytest.mark.gpu


def _gather(ctx, pm, words):
    ctx.set_eval_kernel(pm.EVAL_GATHER)
    try:
        return ctx.evaluate(words)
    finally:
        ctx.set_eval_kernel(pm.EVAL_AUTO)


@pytest.fixture(params=[3000, 9500], ids=["one-slab", "two-slabs"])
def inst(ctx, oracle, request):
    n = request.param
    p = n // 100
    costs = oracle.synth_euclid(n, seed=77)
    ctx.set_instance(costs, n, n, p)
    so, inc = oracle.build_ordering(n, n, p, costs)
    return n, p, costs, so, inc


def test_costs_and_underfilled_chromosomes(ctx, pm, oracle, inst):
    n, p, costs, so, inc = inst
    pop = oracle.random_population(n, p, 900, seed=3)
    rng = np.random.default_rng(1)
    for r in rng.choice(900, 12, replace=False):  # over- and under-filled, none failing
        pop[r] = open_to_words(n, rng.choice(n, int(rng.integers(p - 5, 3 * p)), replace=False))
    keep = [r for r in range(900) if oracle.evaluate(so, inc, n, pop[r:r + 1])[0] == 0]
    pop = pop[keep]
    rc, want, _, _ = oracle.evaluate(so, inc, n, pop)
    assert rc == 0
    assert np.array_equal(_gather(ctx, pm, pop), want)
    # min_cost_sum: the gather without the scan-width contract (instance.cpp:32-48)
    for r in (0, 5, len(keep) - 1):
        assert ctx.min_cost_sum(pop[r:r + 1])[0] == oracle.min_cost_sum(n, n, costs, pop[r])[1]


def test_error_handoff_is_rearmed_between_calls(ctx, pm, oracle, inst):
    n, p, costs, so, inc = inst
    good = oracle.random_population(n, p, 1000, seed=4)
    bad = good.copy()
    bad[700] = 0
    bad[900] = 0
    with pytest.raises(pm.ContractError) as ei:
        _gather(ctx, pm, bad)
    assert ei.value.first_bad == 700
    want = oracle.evaluate(so, inc, n, good)[1]
    assert np.array_equal(_gather(ctx, pm, good), want)  # the word was re-armed
    with pytest.raises(pm.ContractError, match="at least one site must be open"):
        ctx.min_cost_sum(bad[695:705])
    assert np.array_equal(ctx.min_cost_sum(good[:50]),
                          [oracle.min_cost_sum(n, n, costs, w)[1] for w in good[:50]])


def test_device_api_sticky_error_word(ctx, pm, oracle, inst):
    import torch
    n, p, costs, so, inc = inst
    pop = oracle.random_population(n, p, 512, seed=5)
    wp = pop.shape[1]
    ctx.set_eval_kernel(pm.EVAL_GATHER)
    try:
        out = torch.empty(512, dtype=torch.int64, device="cuda")
        bad = pop.copy()
        bad[300] = 0
        dbad = torch.from_numpy(bad.view(np.int64)).cuda()
        dgood = torch.from_numpy(pop.view(np.int64)).cuda()
        ctx.evaluate_device(dbad, out, 512, wp, check=False)   # asynchronous: the error is kept
        ctx.evaluate_device(dgood, out, 512, wp, check=False)  # a clean call does not clear it
        with pytest.raises(pm.ContractError) as ei:
            ctx.check_errors()
        assert ei.value.first_bad == 300
        ctx.evaluate_device(dgood, out, 512, wp, check=True)
        assert np.array_equal(out.cpu().numpy(), oracle.evaluate(so, inc, n, pop)[1])
    finally:
        ctx.set_eval_kernel(pm.EVAL_AUTO)


def test_pipelined_host_call_slots(ctx, pm, oracle, monkeypatch):
    """A host call of >= 4 MB goes in two chunks (lead + rest), each with its own
    error slot written by the fused kernel's last CTA: the reported index is
    global, from whichever chunk fails first."""
    n, p = 4000, 40
    costs = oracle.synth_euclid(n, seed=8)
    ctx.set_instance(costs, n, n, p)
    so, inc = oracle.build_ordering(n, n, p, costs)
    count = 8448  # 8448 x 63 words x 8 B = 4.26 MB
    pop = oracle.random_population(n, p, count, seed=9)
    monkeypatch.setenv("PMB_H2D_LEAD", "4")
    want = oracle.evaluate(so, inc, n, pop)[1]
    assert np.array_equal(_gather(ctx, pm, pop), want)
    for at in (10, 5000):  # in the lead chunk, in the rest
        bad = pop.copy()
        bad[at] = 0
        bad[count - 1] = 0
        with pytest.raises(pm.ContractError) as ei:
            _gather(ctx, pm, bad)
        assert ei.value.first_bad == at
    assert np.array_equal(_gather(ctx, pm, pop), want)
