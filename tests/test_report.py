"""Reporting: the compat emit_report /
parse_structured_report / to_scientific (include/compat/pmedian/bench.hpp)
against the reference's own (oracle/_ref, proj/src/bench.cpp:170-352), byte for
byte and in both directions: our structured report parsed and re-emitted by the
reference is unchanged, the reference's re-emission parsed and re-emitted by us
is unchanged, and malformed lines are rejected with StructuralError.  CPU only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("rr") / "test_report_roundtrip")
    lib = os.path.join(ROOT, "paper_1610_10061_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include", "compat"),
                    "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_report_roundtrip.cpp"), "-L", lib, "-lpmedian_b200",
                    f"-Wl,-rpath,{lib}", "-o", out], check=True)
    return out


def _run(exe, mode, stdin=""):
    return subprocess.run([exe, mode], input=stdin, capture_output=True, text=True, timeout=60)


def test_structured_report_round_trips_through_the_reference(exe, reflib):
    ours = _run(exe, "emit")
    assert ours.returncode == 0, ours.stderr
    rc, theirs, count = reflib.report_roundtrip(ours.stdout)
    assert rc == 0, reflib.last_error()
    assert count == 4 and theirs == ours.stdout
    back = _run(exe, "reparse", theirs)
    assert back.returncode == 0 and back.stdout == theirs


def test_table_report_equals_the_reference(exe, reflib):
    ours = _run(exe, "table")
    rc, theirs, _ = reflib.report_roundtrip(_run(exe, "emit").stdout, structured=False)
    assert rc == 0 and ours.stdout == theirs


@pytest.mark.parametrize("bad", ['{"n": 1}', "not json", '{"instance_code": 5, "n": 1}',
                                 '{"instance_code":"x","n":1,"m":1,"p":1,"search_space":"6x","best_cost":1,'
                                 '"kernel_calls":1,"wall_time":0.5,"seed":1}'])
def test_malformed_lines_are_structural_errors(exe, reflib, bad):
    assert _run(exe, "reject", bad).returncode == 0
    rc, _, _ = reflib.report_roundtrip(bad)
    assert rc != 0


def test_blank_report_is_empty(exe):
    r = _run(exe, "reparse", "\n\n")
    assert r.returncode == 0 and r.stdout == ""


def test_reference_combinatorics_unit_tests_on_the_compat_headers(tmp_path):
    """proj/tests/test_combinatorics.cpp (9 cases), unchanged, against the
    compat BigInt / binomial / unrank_combination / random_below (host code)."""
    src = "/root/reference/proj/tests/test_combinatorics.cpp"
    if not os.path.exists(src):
        pytest.skip("/root/reference absent")
    exe = str(tmp_path / "tc")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include", "compat"), "-I",
                    os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "tests", "cpp", "doctest_shim"),
                    os.path.join(ROOT, "tests", "cpp", "ref_tests_main.cpp"), src, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "9 test cases, 0 failed checks" in r.stdout, r.stdout + r.stderr


def test_compat_random_chromosome_equals_the_reference(tmp_path, reflib):
    """The compat host draw (BigInt binomial, rejection draw, unranking)
    consumes the keyed stream exactly as the reference's random_chromosome
    (combinatorics.cpp:54-75): identical chromosomes, including multi-word
    ranks (C(300, 40) ~ 2^163) and the paper's shapes."""
    import numpy as np
    exe = str(tmp_path / "draw")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include", "compat"), "-I",
                    os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "test_compat_draw.cpp"),
                    "-o", exe], check=True)
    cases = [(4, 2, 7, 50), (100, 5, 1, 40), (300, 40, 9, 20), (900, 90, 3, 8), (65, 64, 2, 5)]
    r = subprocess.run([exe], input="".join(f"{m} {p} {s} {c}\n" for m, p, s, c in cases), capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    at = 0
    for m, p, seed, count in cases:
        wp = (m + 63) // 64
        want = np.zeros(count * wp, dtype=np.uint64)
        assert reflib.L.ref_random_chromosome(m, p, seed, count, want) == 0
        got = np.array([[int(x) for x in ln.split()] for ln in lines[at:at + count]], dtype=np.uint64).reshape(-1)
        at += count
        assert (got == want).all(), (m, p, seed)
