"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's own golden vectors.  Bit-exact for every table entry and cost.

Mirrors the reference's formulation tests (proj/tests/test_formulation.cpp),
instance tests (test_instance.cpp) and acceptance criterion 2
(proj/tests/acceptance.cpp:86-116), then checks BASELINE-size populations
through size-independent properties (scan == gather, two independent
algorithms; sampled chromosomes against the oracle's gather-min).
"""
import itertools

import numpy as np
import pytest

from oracle.oracle import bits_to_words, open_to_words, words_per

pytestmark = pytest.mark.gpu

KINDS = [1, 2]  # EVAL_SCAN, EVAL_GATHER


def _eval(ctx, words, kind):
    ctx.set_eval_kernel(kind)
    return ctx.evaluate(words)


def test_example1_tables_and_fitness(ctx, pm, example1):  # test_formulation.cpp:18-39,187-192
    e = example1
    ctx.set_instance(np.array(e["costs"]), e["n"], e["m"], e["p"])
    so, inc = ctx.get_tables()
    assert so.tolist() == e["site_order"] and inc.tolist() == e["increments"]
    for kind in KINDS:
        for bits, want in e["all_pairs"].items():
            assert _eval(ctx, bits_to_words(bits)[None], kind)[0] == want, (kind, bits)
    assert pm.fitness(ctx, bits_to_words("1001")) == 35


def test_tie_break_and_single_row(ctx):  # test_formulation.cpp:41-61
    ctx.set_instance(np.array([4, 4, 4]), 1, 3, 1)
    so, inc = ctx.get_tables()
    assert so.tolist() == [[0, 1, 2]] and inc.tolist() == [[4, 0, 0]]
    ctx.set_instance(np.array([9, 1, 5]), 1, 3, 2)
    so, inc = ctx.get_tables()
    assert so.tolist() == [[1, 2]] and inc.tolist() == [[1, 4]]


@pytest.mark.parametrize("kind", KINDS)
def test_error_semantics(ctx, pm, kind):  # test_formulation.cpp:194-208
    ctx.set_instance(np.array([9, 1, 5]), 1, 3, 2)
    assert _eval(ctx, bits_to_words("010")[None], kind)[0] == 1
    assert _eval(ctx, bits_to_words("011")[None], kind)[0] == 1
    for bad in ("000", "100"):
        with pytest.raises(pm.ContractError) as ei:
            _eval(ctx, bits_to_words(bad)[None], kind)
        assert ei.value.first_bad == 0
        assert "no open site within the scan width" in str(ei.value)
    with pytest.raises(pm.StructuralError, match="chromosome length must equal the site count"):
        ctx.evaluate(np.zeros((1, 2), dtype=np.uint64))
    # the lowest failing chromosome is reported
    pop = np.stack([bits_to_words(b) for b in ("010", "011", "100", "000", "100")])
    with pytest.raises(pm.ContractError) as ei:
        _eval(ctx, pop, kind)
    assert ei.value.first_bad == 2


def test_instance_validation(ctx, pm):  # test_instance.cpp:520-530, instance.cpp:13-29
    with pytest.raises(pm.DomainError, match="p must be < m"):
        ctx.set_instance(np.array([1, 2]), 1, 2, 2)
    with pytest.raises(pm.DomainError, match="p must be >= 1"):
        ctx.set_instance(np.array([1, 2]), 1, 2, 0)
    with pytest.raises(pm.StructuralError):
        ctx.set_instance(np.array([1]), 1, 2, 1)
    with pytest.raises(pm.StructuralError, match="costs must be non-negative"):
        ctx.set_instance(np.array([1, -3]), 1, 2, 1)
    huge = np.iinfo(np.int64).max // 2 + 1
    with pytest.raises(pm.StructuralError, match="overflow"):
        ctx.set_instance(np.array([huge, 0, 0, 0]), 2, 2, 1)
    ctx.set_instance(np.array([huge, 0]), 1, 2, 1)
    assert ctx.evaluate(bits_to_words("10")[None])[0] == huge


def test_reference_golden_vectors(ctx, pm, ref_vectors):
    """Tables, fitness, runoff errors and min_cost_sum equal the reference's own outputs."""
    for name, c in ref_vectors.items():
        n, m, p = (int(x) for x in c["shape"])
        ctx.set_instance(c["costs"], n, m, p)
        so, inc = ctx.get_tables()
        assert (so == c["site_order"]).all(), name
        assert (inc == c["increments"]).all(), name
        for kind in KINDS:
            assert (_eval(ctx, c["pop"], kind) == c["fitness"]).all(), (name, kind)
            for r in range(c["under"].shape[0]):
                want = int(c["under_fitness"][r])
                if want < 0:
                    with pytest.raises(pm.ContractError):
                        _eval(ctx, c["under"][r:r + 1], kind)
                else:
                    assert _eval(ctx, c["under"][r:r + 1], kind)[0] == want, (name, kind, r)
            # batch of under-filled chromosomes: lowest failing index
            bad = np.nonzero(c["under_fitness"] < 0)[0]
            if bad.size:
                with pytest.raises(pm.ContractError) as ei:
                    _eval(ctx, c["under"], kind)
                assert ei.value.first_bad == bad[0], (name, kind)
        assert (ctx.min_cost_sum(c["pop"]) == c["min_cost_sum"]).all(), name


def test_acceptance_criterion2_exhaustive(ctx, oracle):  # acceptance.cpp:86-116
    st = oracle.stream(2024)
    for trial in range(50):
        n, m = 1 + st.below(8), 2 + st.below(9)  # m <= 10
        costs = oracle.random_costs(st.next(), n, m, 99)
        for p in range(1, m):
            ctx.set_instance(costs, n, m, p)
            pop = np.stack([open_to_words(m, pick) for pick in itertools.combinations(range(m), p)])
            want = np.array([oracle.direct_cost(n, m, p, costs, w)[1] for w in pop])
            for kind in KINDS:
                assert (_eval(ctx, pop, kind) == want).all(), (trial, p, kind)


@pytest.mark.parametrize("shape", [(130, 70, 9), (64, 200, 3), (257, 129, 40), (50, 1000, 100),
                                   (33, 70000, 9), (500, 2000, 1)])
def test_random_instances_vs_oracle(ctx, oracle, shape):
    """Covers u16/u32 site tables (m > 65535), ragged last word, partial groups, p = 1."""
    n, m, p = shape
    for mx in (5, 10**4, 3 * 10**9):
        costs = oracle.random_costs(n * 7 + m + mx, n, m, mx)
        ctx.set_instance(costs, n, m, p)
        so, inc = oracle.build_ordering(n, m, p, costs)
        so2, inc2 = ctx.get_tables()
        assert (so == so2).all() and (inc == inc2).all()
        pop = oracle.random_population(m, p, 70, seed=mx % 1000)
        rc, want, _, _ = oracle.evaluate(so, inc, m, pop)
        assert rc == 0
        for kind in KINDS:
            assert (_eval(ctx, pop, kind) == want).all(), (shape, mx, kind)


def test_empty_population_and_garbage_top_bits(ctx, oracle):
    n, m, p = 40, 100, 6
    costs = oracle.random_costs(5, n, m, 50)
    ctx.set_instance(costs, n, m, p)
    assert ctx.evaluate(np.zeros((0, words_per(m)), dtype=np.uint64)).shape == (0,)
    pop = oracle.random_population(m, p, 10)
    so, inc = oracle.build_ordering(n, m, p, costs)
    want = oracle.evaluate(so, inc, m, pop)[1]
    dirty = pop.copy()
    dirty[:, -1] |= np.uint64(0xFFFFFFF000000000)  # bits >= m: not sites (chromosome.hpp:11-12)
    for kind in KINDS:
        assert (_eval(ctx, dirty, kind) == want).all()


@pytest.mark.parametrize("npts,p,count", [(5000, 50, 1024), (20000, 200, 4096), (10000, 10, 512),
                                          (10000, 1000, 512), (900, 90, 15360)])
def test_baseline_sizes_scan_equals_gather(ctx, oracle, npts, p, count):
    """BASELINE configs syn5k / syn20k at full size: the two independent kernels
    agree on every chromosome, and sampled chromosomes equal the oracle's
    gather-min (instance.cpp:32-48)."""
    costs = oracle.synth_euclid(npts)
    ctx.set_instance(costs, npts, npts, p)
    pop = oracle.random_population(npts, p, count)
    a = _eval(ctx, pop, 1)
    b = _eval(ctx, pop, 2)
    assert (a == b).all()
    for r in range(0, count, count // 8):
        assert oracle.min_cost_sum(npts, npts, costs, pop[r]) == (0, a[r])


def test_device_buffers_and_stream(ctx, oracle):
    import torch
    n, m, p = 300, 300, 30
    costs = oracle.synth_euclid(n)
    dc = torch.from_numpy(costs).cuda()
    ctx.set_instance(dc, n, m, p)
    pop = oracle.random_population(m, p, 200)
    so, inc = oracle.build_ordering(n, m, p, costs)
    want = oracle.evaluate(so, inc, m, pop)[1]
    s = torch.cuda.Stream()
    ctx.set_stream(s)
    dw = torch.from_numpy(pop.view(np.int64)).cuda()
    out = torch.empty(pop.shape[0], dtype=torch.int64, device="cuda")
    before = ctx.kernel_launches
    ctx.evaluate_device(dw, out, pop.shape[0], pop.shape[1], check=False)
    s.synchronize()
    ctx.check_errors()
    assert ctx.kernel_launches > before
    assert (out.cpu().numpy() == want).all()
    ctx.set_stream(None)


def test_payload_key_path_huge_costs(ctx, oracle):
    """cost bits + site bits > 64: K1 sorts a u64 cost key with a separate site
    payload; D' is u64.  Ties are frequent (few distinct huge values)."""
    n, m, p = 7, 300, 11
    base = oracle.random_costs(9, n, m, 5)
    costs = (base.astype(np.int64) << np.int64(58)) // 7 + base  # ~2^60, many ties
    ctx.set_instance(costs, n, m, p)
    assert ctx.table_info().dist_bytes == 8
    so, inc = oracle.build_ordering(n, m, p, costs)
    so2, inc2 = ctx.get_tables()
    assert (so == so2).all() and (inc == inc2).all()
    pop = oracle.random_population(m, p, 100, seed=4)
    want = oracle.evaluate(so, inc, m, pop)[1]
    for kind in KINDS:
        assert (_eval(ctx, pop, kind) == want).all()


def test_pipelined_host_call_reports_global_first_bad(ctx, pm, oracle):
    """pm_evaluate splits large host batches into overlapped chunks; costs and the
    lowest failing index are still global."""
    npts, p, count = 20000, 200, 16384
    costs = oracle.synth_euclid(npts)
    ctx.set_instance(costs, npts, npts, p)
    pop = oracle.random_population(npts, p, count, seed=11)
    good = ctx.evaluate(pop)
    ctx.set_eval_kernel(pm.EVAL_GATHER)
    assert (ctx.evaluate(pop) == good).all()
    ctx.set_eval_kernel(pm.EVAL_AUTO)
    for r in range(0, count, count // 4):
        assert oracle.min_cost_sum(npts, npts, costs, pop[r]) == (0, good[r])
    bad = pop.copy()
    bad[12001] = 0
    bad[15000] = 0
    with pytest.raises(pm.ContractError) as ei:
        ctx.evaluate(bad)
    assert ei.value.first_bad == 12001
    # a 4096 batch (10 MB) goes as a lead chunk of 512 and the rest
    small = pop[:4096].copy()
    assert (ctx.evaluate(small) == good[:4096]).all()
    small[3000] = 0
    with pytest.raises(pm.ContractError) as ei:
        ctx.evaluate(small)
    assert ei.value.first_bad == 3000
    small[100] = 0
    with pytest.raises(pm.ContractError) as ei:
        ctx.evaluate(small)
    assert ei.value.first_bad == 100


def test_counting_sort_path_and_handback(ctx, oracle):
    """K1's counting-sort path (costs < 2^15, m >= 2^costbits / 2): ties put back
    into site order inside each bucket; a row with a bucket above 64 ties is
    handed to the radix kernel (ordering.cpp:25-28 order either way)."""
    n, m, p = 24, 9000, 90
    costs = oracle.random_costs(77, n, m, 10**4).reshape(n, m).copy()
    costs[3, :] = 4321                       # one bucket of m ties: handed back
    costs[7, :] = costs[7, :] % 3 + 9000     # three huge buckets
    costs[11, ::2] = 17                      # half the row tied at one cost
    costs = costs.reshape(-1)
    ctx.set_instance(costs, n, m, p)
    so, inc = oracle.build_ordering(n, m, p, costs)
    so2, inc2 = ctx.get_tables()
    assert (so == so2).all() and (inc == inc2).all()
    pop = oracle.random_population(m, p, 64, seed=5)
    want = oracle.evaluate(so, inc, m, pop)[1]
    for kind in KINDS:
        assert (_eval(ctx, pop, kind) == want).all()


@pytest.mark.parametrize("npts,p,count", [(20000, 200, 2048), (900, 90, 15360)])
def test_scan_shapes_agree(ctx, oracle, npts, p, count, monkeypatch):
    """The planner's 24-warp K2 variant (one 768-thread CTA per SM for long
    segments, 12 x 2-warp CTAs for short ones) and the 16-warp shapes it
    replaces (PMB_SCAN_WIDE=0) give identical costs."""
    costs = oracle.synth_euclid(npts)
    ctx.set_instance(costs, npts, npts, p)
    pop = oracle.random_population(npts, p, count, seed=3)
    wide = _eval(ctx, pop, 1)
    monkeypatch.setenv("PMB_SCAN_WIDE", "0")
    narrow = _eval(ctx, pop, 1)
    assert (wide == narrow).all()
    for r in range(0, count, count // 4):
        assert oracle.min_cost_sum(npts, npts, costs, pop[r]) == (0, wide[r])
