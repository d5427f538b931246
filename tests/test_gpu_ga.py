"""GPU: the device GA against the reference's own GA (oracle/_ref, i.e. the
unmodified proj/src/ga.cpp + combinatorics.cpp) -- evolve_block bit for bit,
run_ga RunResult for RunResult -- and the reference's GA tests
(proj/tests/test_ga.cpp:224-454) restated."""
import numpy as np
import pytest

from oracle.oracle import bits_to_words, open_to_words, words_per

pytestmark = pytest.mark.gpu

E1 = [7, 10, 16, 11, 15, 17, 7, 7, 10, 4, 6, 6, 7, 11, 18, 12, 10, 22, 14, 8]


def _random_block(oracle, m, p, count, seed):
    return oracle.random_population(m, p, count, seed=seed)


@pytest.mark.parametrize("case", [
    # (n, m, p, nt, nb, seed, kernel, first_block, cx, mu, max_cost)
    (5, 4, 2, 4, 1, 11, 0, 0, -1, -1, None),
    (9, 9, 3, 8, 2, 99, 3, 1, -1, -1, 99),
    (30, 40, 6, 32, 3, 5, 2, 7, -1, -1, 99),
    (25, 130, 12, 16, 2, 8, 1, 0, 7, 5, 1000),   # crossover stride pattern restarts (ga.cpp:159)
    (20, 70, 1, 8, 2, 3, 0, 4, -1, -1, 50),      # p = 1: no crossover (ga.cpp:154)
    (40, 64, 63, 8, 1, 4, 6, 2, -1, -1, 30),     # p = m - 1
    (300, 300, 30, 64, 2, 21, 5, 9, -1, -1, None),
    (10, 20, 4, 8, 1, 2, 0, 0, 0, 0, 9),         # both cycles disabled
])
def test_evolve_block_matches_reference(ctx, pm, oracle, reflib, case):
    n, m, p, nt, nb, seed, kernel, fb, cx, mu, mx = case
    costs = np.array(E1) if mx is None and n == 5 else (
        oracle.synth_euclid(n) if mx is None else oracle.random_costs(seed * 31 + n, n, m, mx))
    ctx.set_instance(costs, n, m, p)
    ri = reflib.create(n, m, p, costs)
    blocks = _random_block(oracle, m, p, nb * nt, seed + 17)
    cfg = pm.ga_config(nb=nb, nt=nt, seed=seed, crossover_iters=None if cx < 0 else cx,
                       mutation_iters=None if mu < 0 else mu)
    got, bc, bt = ctx.evolve_blocks(blocks, cfg, kernel, fb)
    for b in range(nb):
        rc, want, wbest, wcost, wthread = ri.evolve_block(blocks[b * nt:(b + 1) * nt], nt, nb, seed, kernel,
                                                          fb + b, cx, mu)
        assert rc == 0, reflib.last_error()
        assert (got[b * nt:(b + 1) * nt] == want).all(), (case, b)
        assert bc[b] == wcost and bt[b] == wthread, (case, b)
        assert (got[b * nt + bt[b]] == wbest).all()


def test_evolve_block_keeps_optimum(ctx, pm):  # test_ga.cpp:224-244
    ctx.set_instance(np.array(E1), 5, 4, 2)
    block = np.stack([bits_to_words(b) for b in ("1001", "0110", "1100", "0101")])
    cfg = pm.ga_config(nb=1, nt=4, seed=11)
    out, bc, bt = ctx.evolve_blocks(block, cfg, 0, 0)
    assert bc[0] == 35 and (out[bt[0]] == bits_to_words("1001")).all()
    assert all(c >= 35 for c in ctx.evaluate(out))


def test_evolve_block_deterministic_and_kernel_sensitive(ctx, pm, oracle):  # test_ga.cpp:264-288
    costs = oracle.random_costs(7, 9, 9, 99)
    ctx.set_instance(costs, 9, 9, 3)
    blk = oracle.random_population(9, 3, 8, seed=5)
    cfg = pm.ga_config(nb=2, nt=8, seed=99)
    a = ctx.evolve_blocks(blk, cfg, 3, 1)
    b = ctx.evolve_blocks(blk, cfg, 3, 1)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and (a[2] == b[2]).all()
    c = ctx.evolve_blocks(blk, cfg, 4, 1)
    assert not (c[0] == a[0]).all()


def test_evolve_block_rejects_bad_shapes(ctx, pm):  # test_ga.cpp:290-320
    ctx.set_instance(np.array(E1), 5, 4, 2)
    with pytest.raises(pm.DomainError, match="nt must be a power of two"):
        ctx.evolve_blocks(np.zeros((3, 1), dtype=np.uint64), pm.ga_config(nb=1, nt=3), 0)
    for kw, msg in ((dict(nb=0), "nb must be >= 1"), (dict(evolve_limit=0), "evolve_limit"),
                    (dict(saturation=0), "saturation"), (dict(nb=16, nt=8, team=True), "team migration")):
        with pytest.raises(pm.DomainError, match=msg):
            ctx.run_ga(pm.ga_config(**dict(dict(nt=4), **kw)))


def test_evolve_block_checks_only_its_own_shape(ctx, pm, oracle, reflib):  # ga.cpp:136-141
    """evolve_block validates nt alone, as the reference does: run-level limits
    (evolve_limit, saturation, team migration) are run_ga's, so a config the
    reference's evolve_block accepts evolves the block identically here."""
    costs = oracle.random_costs(21, 9, 9, 50)
    ctx.set_instance(costs, 9, 9, 3)
    blk = oracle.random_population(9, 3, 8, seed=6)
    ri = reflib.create(9, 9, 3, costs)
    for cfg in (pm.ga_config(nb=1, nt=8, evolve_limit=0, saturation=0, seed=5),
                pm.ga_config(nb=16, nt=8, team=True, seed=5)):
        got, cost, thread = ctx.evolve_blocks(blk, cfg, 2, 0)
        rc, want, _, wcost, wthread = ri.evolve_block(blk, 8, 1, 5, 2, 0)
        assert rc == 0 and (got == want).all() and cost[0] == wcost and thread[0] == wthread


def _cmp_run(got, want):
    assert got["best_cost"] == want["best_cost"]
    assert (got["best"] == want["best"]).all()
    assert got["kernels_executed"] == want["kernels_executed"]
    assert got["kernel_of_best"] == want["kernel_of_best"]
    assert (got["per_kernel_best_costs"] == want["per_kernel_best_costs"]).all()


def test_run_ga_5x4_matches_reference_every_seed(ctx, pm, reflib):  # test_ga.cpp:322-336
    ctx.set_instance(np.array(E1), 5, 4, 2)
    ri = reflib.create(5, 4, 2, np.array(E1))
    for seed in range(1, 26):
        got = ctx.run_ga(pm.ga_config(nb=2, nt=4, evolve_limit=10, saturation=10, seed=seed))
        rc, want = ri.run_ga(2, 4, 10, 10, seed)
        assert rc == 0
        _cmp_run(got, want)
        assert got["best_cost"] == 35 and (got["best"] == bits_to_words("1001")).all()


def test_run_ga_12x12_matches_reference(ctx, pm, oracle, reflib):  # test_ga.cpp:338-354
    costs = oracle.random_costs(12345, 12, 12, 99)
    ctx.set_instance(costs, 12, 12, 4)
    ri = reflib.create(12, 12, 4, costs)
    rc, _, exact = ri.exact_optimum()
    for seed in range(1, 11):
        got = ctx.run_ga(pm.ga_config(nb=4, nt=32, evolve_limit=50, saturation=10, seed=seed))
        rc, want = ri.run_ga(4, 32, 50, 10, seed)
        _cmp_run(got, want)
        assert got["best_cost"] == exact


def test_run_ga_team_migration_and_overrides(ctx, pm, oracle, reflib):  # test_ga.cpp:420-454
    ctx.set_instance(np.array(E1), 5, 4, 2)
    ri = reflib.create(5, 4, 2, np.array(E1))
    for seed in range(1, 6):
        got = ctx.run_ga(pm.ga_config(nb=2, nt=4, evolve_limit=10, saturation=10, seed=seed, team=True))
        _cmp_run(got, ri.run_ga(2, 4, 10, 10, seed, team=True)[1])
    costs = oracle.random_costs(77, 10, 10, 99)
    ctx.set_instance(costs, 10, 10, 4)
    ri = reflib.create(10, 10, 4, costs)
    for cx, mu in ((7, 5), (0, 0)):
        got = ctx.run_ga(pm.ga_config(nb=2, nt=8, evolve_limit=6, saturation=6, seed=9, crossover_iters=cx,
                                      mutation_iters=mu))
        _cmp_run(got, ri.run_ga(2, 8, 6, 6, 9, cx, mu)[1])


def test_run_ga_saturation_and_monotone(ctx, pm, oracle):  # test_ga.cpp:356-399
    ctx.set_instance(np.array(E1), 5, 4, 2)
    r = ctx.run_ga(pm.ga_config(nb=2, nt=4, evolve_limit=50, saturation=3, seed=2))
    assert r["kernels_executed"] == r["kernel_of_best"] + 3
    r = ctx.run_ga(pm.ga_config(nb=1, nt=2, evolve_limit=1, saturation=1, seed=5))
    assert r["kernels_executed"] == 1 and r["kernel_of_best"] == 1
    for seed in range(1, 6):
        costs = oracle.random_costs(seed * 3, 8, 8, 99)
        ctx.set_instance(costs, 8, 8, 3)
        r = ctx.run_ga(pm.ga_config(nb=3, nt=8, evolve_limit=12, saturation=12, seed=seed))
        pk = r["per_kernel_best_costs"]
        assert (np.diff(pk) <= 0).all() and r["best_cost"] == pk[-1]


def test_run_ga_pmed40_shape_matches_reference(ctx, pm, oracle, reflib):
    """The paper's Table-1 GA shape (nb=60, nt=256) on a 900/90 Euclidean
    instance: identical RunResult to the reference over 2 generations."""
    costs = oracle.synth_euclid(900)
    ctx.set_instance(costs, 900, 900, 90)
    ri = reflib.create(900, 900, 90, costs)
    got = ctx.run_ga(pm.ga_config(nb=60, nt=256, evolve_limit=2, saturation=10, seed=1))
    rc, want = ri.run_ga(60, 256, 2, 10, 1, workers=16)
    assert rc == 0
    _cmp_run(got, want)


def test_run_ga_device_population(ctx, pm, oracle):
    costs = oracle.synth_euclid(200)
    ctx.set_instance(costs, 200, 200, 20)
    a = ctx.run_ga(pm.ga_config(nb=8, nt=32, evolve_limit=6, saturation=6, seed=3, population="device"))
    b = ctx.run_ga(pm.ga_config(nb=8, nt=32, evolve_limit=6, saturation=6, seed=3, population="device"))
    _cmp_run(a, b)
    assert sum(bin(int(x)).count("1") for x in a["best"]) == 20
    assert oracle.direct_cost(200, 200, 20, costs, a["best"]) == (0, a["best_cost"])


@pytest.mark.parametrize("npts,p,cap_mb", [(1500, 150, None), (2200, 330, None), (2600, 520, None),
                                           (2600, 520, "256")])
def test_run_ga_wide_ranks_match_reference(ctx, pm, oracle, reflib, npts, p, cap_mb, monkeypatch):
    """Population draws whose ranks need 12 / 22 / 31 limbs (the device
    unranking's 16- and 32-limb kernels) and, with the Pascal-table budget cut
    to 256 MB, the host unranking path -- against the reference's own draw."""
    if cap_mb:
        monkeypatch.setenv("PMB_PASCAL_MAX_MB", cap_mb)
    costs = oracle.synth_euclid(npts)
    ctx.set_instance(costs, npts, npts, p)
    ri = reflib.create(npts, npts, p, costs)
    got = ctx.run_ga(pm.ga_config(nb=2, nt=8, evolve_limit=2, saturation=5, seed=4))
    rc, want = ri.run_ga(2, 8, 2, 5, 4, workers=16)
    assert rc == 0
    _cmp_run(got, want)


def test_full_run_pmed1_shape_reaches_exhaustive_optimum(ctx, pm, reflib):
    """BASELINE config 1 on a synthetic pmed1-shaped instance (n=m=100, p=5; the
    OR-Library files are absent): the paper's Table-1 run (nb=60, nt=256,
    evolve_limit=100, saturation=10) gives the reference's RunResult and the
    optimum, found by evaluating all C(100, 5) = 75,287,520 subsets on the device."""
    import torch

    from paper_1610_10061_b200 import synth
    costs = synth.euclid_costs(100, 12345)
    ctx.set_instance(costs, 100, 100, 5)
    best = None
    for chunk in synth.all_subsets(100, 5):
        w = torch.from_numpy(chunk.view(np.int64)).cuda()
        out = torch.empty(chunk.shape[0], dtype=torch.int64, device="cuda")
        ctx.evaluate_device(w, out, chunk.shape[0], chunk.shape[1], check=True)
        v = int(out.min().item())
        best = v if best is None else min(best, v)
    got = ctx.run_ga(pm.ga_config(nb=60, nt=256, evolve_limit=100, saturation=10, seed=1))
    rc, want = reflib.create(100, 100, 5, costs).run_ga(60, 256, 100, 10, 1, workers=16)
    assert rc == 0
    _cmp_run(got, want)
    assert got["best_cost"] == best


def test_evolve_blocks_paper_shape_matches_reference(ctx, pm, oracle, reflib):
    """All 60 blocks of the paper's GA shape (nt=256: 8 crossover rounds, 8
    mutation attempts) at 900/90, block for block against the reference's
    evolve_block.  Guards the crossover kernel at scale: an earlier form of
    it produced children with the wrong popcount in some processes."""
    from paper_1610_10061_b200 import synth
    costs = synth.euclid_costs(900, 12345)
    ctx.set_instance(costs, 900, 900, 90)
    ri = reflib.create(900, 900, 90, costs)
    nb, nt = 60, 256
    blocks = synth.random_population(900, 90, nb * nt, seed=9)
    for kernel in (0, 3):
        got, bc, bt = ctx.evolve_blocks(blocks, pm.ga_config(nb=nb, nt=nt, seed=1), kernel)
        for b in range(nb):
            rc, want, _, wcost, wthread = ri.evolve_block(blocks[b * nt:(b + 1) * nt], nt, nb, 1, kernel, b, -1, -1)
            assert rc == 0
            assert (got[b * nt:(b + 1) * nt] == want).all(), (kernel, b)
            assert bc[b] == wcost and bt[b] == wthread, (kernel, b)


@pytest.mark.parametrize("npts,p,nb,nt", [(3000, 300, 4, 64), (6000, 60, 2, 128)])
def test_evolve_blocks_wide_chromosomes_match_reference(ctx, pm, reflib, npts, p, nb, nt):
    """Crossover and shift mutations over 47- and 94-word chromosomes (large
    exchange counts, multi-word rotations), block for block against the
    reference's evolve_block."""
    from paper_1610_10061_b200 import synth
    costs = synth.euclid_costs(npts, 12345)
    ctx.set_instance(costs, npts, npts, p)
    ri = reflib.create(npts, npts, p, costs)
    blocks = synth.random_population(npts, p, nb * nt, seed=5)
    got, bc, bt = ctx.evolve_blocks(blocks, pm.ga_config(nb=nb, nt=nt, seed=2), 1)
    for b in range(nb):
        rc, want, _, wcost, wthread = ri.evolve_block(blocks[b * nt:(b + 1) * nt], nt, nb, 2, 1, b, -1, -1)
        assert rc == 0
        assert (got[b * nt:(b + 1) * nt] == want).all(), b
        assert bc[b] == wcost and bt[b] == wthread, b
