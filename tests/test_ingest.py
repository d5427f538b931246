"""Instance ingestion: OR-Library graph text (parse_orlib, proj/src/bench.cpp:106-168)
with the closure on the device, and the dense text format (parse_dense, :65-104).
Cases restate proj/tests/test_bench.cpp:40-135; results are compared with the
reference's own parsers (oracle/_ref) and the C restatement of the closure."""
import numpy as np
import pytest

SAMPLE_DENSE = "5 4 2\n7 10 16 11\n15 17 7 7\n10 4 6 6\n7 11 18 12\n10 22 14 8\n"


def random_graph(seed, n, extra, wmax=20, oracle=None):
    """test_bench.cpp:101-121: random spanning tree plus extra edges, as text."""
    st = oracle.stream(seed)
    body, edges = [], 0
    for v in range(2, n + 1):
        u = 1 + st.below(v - 1)
        body.append(f"{u} {v} {1 + st.below(wmax)}")
        edges += 1
    for _ in range(extra):
        u, v = 1 + st.below(n), 1 + st.below(n)
        if u == v:
            continue
        body.append(f"{u} {v} {1 + st.below(wmax)}")
        edges += 1
    return f"{n} {edges} 1\n" + "\n".join(body) + "\n"


def parse_edges(text):
    tok = text.split()
    n, e = int(tok[0]), int(tok[1])
    trip = np.array(tok[3:3 + 3 * e], dtype=np.int64).reshape(-1, 3)
    return n, trip[:, :2] - 1, trip[:, 2]


def test_oracle_closure_matches_reference(oracle, reflib):
    for seed in range(10):
        text = random_graph(61 + seed, 3 + seed * 4, 6, oracle=oracle)
        rc, n, m, p, want = reflib.parse(text)
        assert rc == 0
        nn, uv, w = parse_edges(text)
        rc2, got, _ = oracle.orlib_closure(nn, uv, w)
        assert rc2 == 0 and (got == want).all()
    rc, out, bad = oracle.orlib_closure(3, np.array([[0, 1]]), np.array([5]))
    assert rc == 1 and bad == 2  # vertices 1 and 3 (0-based pair (0, 2))


DIAGNOSTICS = [
    ("", None),
    ("3 1 1\n1 2 5\n", "graph format: disconnected graph, no path between vertices 1 and 3"),
    ("2 1 1\n1 3 5\n", "graph format: vertex index out of range in edge 1"),
    ("2 1 1\n1 2 -5\n", "graph format: negative cost on edge 1"),
    ("2 2 1\n1 2 5\n", "graph format: expected 2 'u v cost' triples, found 1 plus stray tokens"),
    ("x 1 1\n1 2 5\n", "could not parse vertex count: 'x'"),
]


@pytest.mark.gpu
def test_orlib_golden_cases(ctx, pm, reflib):  # test_bench.cpp:73-99
    n, p, c = ctx.orlib_closure("3 3 1\n1 2 3\n2 3 4\n1 3 10\n")
    assert (n, p) == (3, 1) and c.tolist() == [0, 3, 7, 3, 0, 4, 7, 4, 0]
    assert ctx.orlib_closure("2 1 1\n1 2 5\n")[2].tolist() == [0, 5, 5, 0]
    assert ctx.orlib_closure("2 2 1\n1 2 9\n2 1 4\n")[2].tolist() == [0, 4, 4, 0]
    for text, msg in DIAGNOSTICS:
        with pytest.raises(pm.StructuralError) as ei:
            ctx.orlib_closure(text)
        rc, *_ = reflib.parse(text)
        assert rc == 1
        if msg:
            assert str(ei.value) == msg
            assert reflib.last_error() == msg


@pytest.mark.gpu
@pytest.mark.parametrize("n,extra", [(5, 4), (12, 4), (33, 40), (100, 200), (257, 600), (900, 3000)])
def test_orlib_closure_matches_reference(ctx, oracle, reflib, n, extra):
    text = random_graph(1000 + n, n, extra, wmax=100, oracle=oracle)
    rc, nn, m, p, want = reflib.parse(text, cap=n * n)
    assert rc == 0
    got_n, got_p, got = ctx.orlib_closure(text)
    assert got_n == n and (got == want).all()


@pytest.mark.gpu
def test_orlib_instance_runs_like_reference(ctx, pm, oracle, reflib):
    """A pmed-shaped graph (n=100, ~200 edges) end to end: device closure -> K1
    tables -> run_ga, against the reference's parse_orlib + run_ga."""
    hdr = random_graph(7, 100, 110, wmax=100, oracle=oracle).split("\n", 1)
    e = int(hdr[0].split()[1])
    text = f"100 {e} 5\n" + hdr[1]
    ctx.set_instance_orlib(text)
    rc, n, m, p, costs = reflib.parse(text, cap=100 * 100)
    assert (n, m, p) == (100, 100, 5)
    so, inc = ctx.get_tables()
    so2, inc2 = oracle.build_ordering(n, m, p, costs)
    assert (so == so2).all() and (inc == inc2).all()
    ri = reflib.create(n, m, p, costs)
    got = ctx.run_ga(pm.ga_config(nb=4, nt=32, evolve_limit=8, saturation=8, seed=3))
    rc, want = ri.run_ga(4, 32, 8, 8, 3)
    assert got["best_cost"] == want["best_cost"] and (got["best"] == want["best"]).all()
    assert (got["per_kernel_best_costs"] == want["per_kernel_best_costs"]).all()
    ctx.set_instance_orlib(text, p=7)  # --p override (bench.cpp:241-243)
    assert ctx.table_info().open_count == 7


@pytest.mark.gpu
def test_dense_parser(ctx, pm, reflib):  # test_bench.cpp:40-70
    ctx.set_instance_dense(SAMPLE_DENSE)
    assert (ctx.n, ctx.m, ctx.p) == (5, 4, 2)
    so, inc = ctx.get_tables()
    assert so.tolist() == [[0, 1, 3], [2, 3, 0], [1, 2, 3], [0, 1, 3], [3, 0, 2]]
    ctx.set_instance_dense("  1   2 1 \n\n  0\t4 \n")
    assert (ctx.n, ctx.m) == (1, 2)
    for text, cls, msg in [
        ("", pm.StructuralError, "dense format: empty input"),
        ("1 2\n0 1\n", pm.StructuralError, "dense format: header must be 'n m p'"),
        ("2 2 1\n0 1\n", pm.StructuralError, "dense format: expected 2 cost rows, found 1"),
        ("1 3 1\n0 1\n", pm.StructuralError, "dense format: row 1 has 2 values, expected 3"),
        ("1 2 1\n0 -4\n", pm.StructuralError, "dense format: negative cost at row 1, column 2"),
        ("1 2 2\n0 4\n", pm.DomainError, "p must be < m"),
        ("1 2 x\n0 4\n", pm.StructuralError, None),
    ]:
        with pytest.raises(cls) as ei:
            ctx.set_instance_dense(text)
        if msg:
            assert str(ei.value) == msg
        assert reflib.parse(text, orlib=False)[0] == cls.status
