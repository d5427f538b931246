"""The scan's tail machinery (csrc/fitness.cu: shrinking client claims, the
segmented cooperative tail, column-pair appends) against the oracle.

Every knob setting -- the cooperative tail off, on from the first idle lane,
one client per pass or up to 32 side by side, claims always shrunk, pairs
forced on or off -- must give the sequential walk's costs (ordering.cpp:40-59),
its stopping depths (the roofline's sum of k*), and the lowest failing
chromosome when a walk runs off the scan width (ordering.cpp:50-52), also when
the failing walks are the long ones the cooperative tail takes over.
"""
import numpy as np
import pytest

from oracle.oracle import open_to_words

pytestmark = pytest.mark.gpu

SETTINGS = [
    {"PMB_SCAN_COOP": "0"},                                  # tail off
    {"PMB_SCAN_COOP": "32", "PMB_SCAN_COOPSEG": "5"},       # from the first idle lane, up to 32 lanes a client
    {"PMB_SCAN_COOP": "32", "PMB_SCAN_COOPSEG": "0"},       # one lane a client (the 16-column step, re-packed)
    {"PMB_SCAN_COOP": "8", "PMB_SCAN_COOPSEG": "2"},        # at most 4 lanes a client
    {"PMB_SCAN_TAILCLAIM": "1000000"},                      # claims always shrunk to the needy lanes
    {"PMB_SCAN_TAILCLAIM": "0", "PMB_SCAN_COOP": "1"},      # batches of 32 to the end
    {"PMB_SCAN_PAIR": "1", "PMB_SCAN_COOP": "32"},          # column pairs forced on
    {"PMB_SCAN_PAIR": "0"},                                  # and off
]
SHAPES = [(3000, 30, 1000), (900, 90, 3000), (2000, 200, 600), (1500, 3, 200)]


def _scan(ctx, pm, words):
    ctx.set_eval_kernel(pm.EVAL_SCAN)
    try:
        return ctx.evaluate(words)
    finally:
        ctx.set_eval_kernel(pm.EVAL_AUTO)


@pytest.mark.parametrize("npts,p,count", SHAPES)
def test_tail_settings_equal_the_sequential_walk(ctx, pm, oracle, monkeypatch, npts, p, count):
    import torch
    costs = oracle.synth_euclid(npts, seed=npts + p)
    ctx.set_instance(costs, npts, npts, p)
    so, inc = oracle.build_ordering(npts, npts, p, costs)
    pop = oracle.random_population(npts, p, count, seed=11)
    # chromosomes with more open sites than p walk short rows; fewer (but not
    # failing: the site nearest to every client is open) walk long ones
    rng = np.random.default_rng(npts)
    for r in rng.choice(count, 8, replace=False):
        picks = rng.choice(npts, int(rng.integers(1, 3 * p + 2)), replace=False)
        pop[r] = open_to_words(npts, picks)
    rc, want, _, sk = oracle.evaluate(so, inc, npts, pop, want_sum_k=True)
    ok = rc == 0
    if not ok:  # a drawn under-filled chromosome ran off: keep the others
        keep = [r for r in range(count) if oracle.evaluate(so, inc, npts, pop[r:r + 1])[0] == 0]
        pop = pop[keep]
        rc, want, _, sk = oracle.evaluate(so, inc, npts, pop, want_sum_k=True)
        assert rc == 0
    wp = pop.shape[1]
    dwords = torch.from_numpy(pop.view(np.int64)).cuda()
    depth = torch.zeros(pop.shape[0], dtype=torch.int64, device="cuda")
    for s in SETTINGS:
        with monkeypatch.context() as mp:
            for k, v in s.items():
                mp.setenv(k, v)
            got = _scan(ctx, pm, pop)
            ctx.scan_depths_device(dwords, depth, pop.shape[0], wp)
            torch.cuda.synchronize()
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (s, bad[:5])
        assert np.array_equal(depth.cpu().numpy().view(np.uint64), sk), s


@pytest.mark.parametrize("npts,p", [(3000, 30), (900, 90)])
def test_tail_settings_report_the_lowest_runoff(ctx, pm, oracle, monkeypatch, npts, p):
    """An all-closed chromosome walks every row to the end (the cooperative
    tail's runoff branch); one open far site runs off for some clients only."""
    costs = oracle.synth_euclid(npts, seed=5)
    ctx.set_instance(costs, npts, npts, p)
    so, inc = oracle.build_ordering(npts, npts, p, costs)
    count = 2000
    pop = oracle.random_population(npts, p, count, seed=12)
    far = int(np.argmax(costs.reshape(npts, npts).sum(axis=0)))  # the site farthest from everyone
    pop[1500] = open_to_words(npts, [far])
    pop[1700] = 0
    rc, _, fb, _ = oracle.evaluate(so, inc, npts, pop)
    assert rc != 0 and fb in (1500, 1700)
    for s in SETTINGS:
        with monkeypatch.context() as mp:
            for k, v in s.items():
                mp.setenv(k, v)
            with pytest.raises(pm.ContractError) as ei:
                _scan(ctx, pm, pop)
        assert ei.value.first_bad == fb, s
