"""The benchmark CLI (paper_1610_10061_b200/pmedian_bench) against the reference
CLI's contract: proj/tests/CMakeLists.txt:21-36 smoke tests, and the reference's
own run_benchmark + emit_report (oracle/_ref) record for record."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1610_10061_b200", "pmedian_bench")


def _sample(tmp_path, example1):
    e = example1
    rows = [" ".join(str(v) for v in e["costs"][i * e["m"]:(i + 1) * e["m"]]) for i in range(e["n"])]
    path = tmp_path / "sample_5x4.dense"
    path.write_text(f"{e['n']} {e['m']} {e['p']}\n" + "\n".join(rows) + "\n")
    (tmp_path / "sample_5x4.opt").write_text(f"{e['optimum']['cost']}\n")
    return path


def _run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)


def test_cli_built():
    assert os.access(CLI, os.X_OK)


@pytest.mark.gpu
def test_cli_smoke_matches_reference_ctest(tmp_path, example1):  # tests/CMakeLists.txt:21-36
    inst = _sample(tmp_path, example1)
    common = ["--instance", inst, "--format", "dense", "--nb", 2, "--nt", 4, "--evolve-limit", 10,
              "--saturation", 5, "--seed", 7]
    r = _run(*common)
    assert r.returncode == 0 and "Optimal" in r.stdout, r.stderr
    r = _run(*common, "--report", "structured")
    assert r.returncode == 0 and '"best_cost":35' in r.stdout
    r = _run("--instance", inst, "--format", "dense", "--nt", 3)
    assert r.returncode != 0 and "nt must be a power of two" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--repeats", 3], ["--migration", "team"], ["--p", 3],
                                   ["--crossover-iters", 5, "--mutation-iters", 2]])
def test_cli_records_equal_reference(tmp_path, example1, reflib, oracle, extra):
    n = m = 40
    costs = oracle.random_costs(404, n, m, 99)
    path = tmp_path / "rand40.dense"
    path.write_text(f"{n} {m} 4\n" + "\n".join(" ".join(str(int(c)) for c in costs[i * m:(i + 1) * m])
                                                for i in range(n)) + "\n")
    (tmp_path / "rand40.opt").write_text("1234\n")
    cfg = dict(nb=4, nt=16, evolve_limit=6, saturation=6, seed=5)
    r = _run("--instance", path, "--nb", 4, "--nt", 16, "--evolve-limit", 6, "--saturation", 6,
             "--seed", 5, "--report", "structured", *extra)
    assert r.returncode == 0, r.stderr
    kw = dict(cfg)
    flags = dict(zip(extra[0::2], extra[1::2]))
    kw.update(repeats=flags.get("--repeats", 1), team=flags.get("--migration") == "team",
              p_override=flags.get("--p", 0), cx=flags.get("--crossover-iters", -1),
              mu=flags.get("--mutation-iters", -1), reference=1234)
    rc, want = reflib.run_benchmark(path, **kw)
    assert rc == 0, reflib.last_error()
    got, ref = json.loads(r.stdout), json.loads(want)
    assert list(got) == list(ref)  # same fields, same order
    for k in ref:
        if k != "wall_time":
            assert got[k] == ref[k], k
    # the table layout too, time column aside
    t = _run("--instance", path, "--nb", 4, "--nt", 16, "--evolve-limit", 6, "--saturation", 6,
             "--seed", 5, *extra).stdout.splitlines()
    rc, tw = reflib.run_benchmark(path, structured=False, **kw)
    tw = tw.splitlines()
    assert t[0] == tw[0]
    assert t[1][:-49] == tw[1][:-49] and t[1][-36:] == tw[1][-36:]
