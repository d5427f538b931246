"""Regenerates tests/golden/ref_vectors.npz from the REFERENCE ITSELF.

Runs in the build container only (it needs /root/reference, compiled into
oracle/_ref/libpmref.so by oracle/Makefile).  The committed .npz then travels
to the GPU box so GPU parity tests compare against the reference's own outputs
without /root/reference.  Instances use the reference test-suite generator
(proj/tests/test_support.hpp:22-30, restated as or_random_costs) and the
SURVEY.md 8(d) Euclidean generator; populations are uniform p-subsets plus
deliberately under-filled chromosomes that exercise the ContractError path
(proj/src/ordering.cpp:50-52).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, RefLib, words_per  # noqa: E402

CASES = [  # (name, kind, seed, n, m, p, max_cost)
    ("tie_heavy", "rand", 11, 40, 37, 5, 3),
    ("small_rand", "rand", 12, 25, 30, 7, 99),
    ("wide", "rand", 13, 9, 150, 4, 1000),
    ("tall", "rand", 14, 200, 20, 3, 50),
    ("p1", "rand", 15, 30, 70, 1, 99),
    ("p_m_minus_1", "rand", 16, 30, 70, 69, 99),
    ("m64", "rand", 17, 20, 64, 9, 500),
    ("m65", "rand", 18, 20, 65, 9, 500),
    ("big_cost_u32", "rand", 19, 30, 80, 6, 3_000_000_000),
    ("big_cost_u64", "rand", 20, 7, 40, 3, 900_000_000_000_000),
    ("euclid300", "euclid", 12345, 300, 300, 30, None),
]


def main():
    o, ref = Oracle(), RefLib()
    out = {}
    for name, kind, seed, n, m, p, mx in CASES:
        costs = o.random_costs(seed, n, m, mx) if kind == "rand" else o.synth_euclid(n, seed)
        ri = ref.create(n, m, p, costs)
        assert ri.rc == 0, ref.last_error()
        so, inc = ri.tables()
        pop = o.random_population(m, p, 96, seed=seed + 1000)
        rc, cs, fb = ri.evaluate(pop)
        assert rc == 0
        # under-filled chromosomes: 1..p-1 open sites (may or may not run off)
        st = o.stream(seed + 2000)
        under = np.zeros((32, words_per(m)), dtype=np.uint64)
        for r in range(32):
            k = 1 + st.below(max(1, p - 1)) if p > 1 else 1
            for _ in range(k):
                j = st.below(m)
                under[r, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
        ucost = np.full(32, -1, dtype=np.int64)
        for r in range(32):
            rcu, cu, _ = ri.evaluate(under[r:r + 1])
            ucost[r] = cu[0] if rcu == 0 else -1  # -1: ContractError
        mcs = np.array([ri.min_cost_sum(pop[r])[1] for r in range(pop.shape[0])], dtype=np.int64)
        out.update({f"{name}/shape": np.array([n, m, p], dtype=np.int64), f"{name}/costs": costs,
                    f"{name}/site_order": so, f"{name}/increments": inc, f"{name}/pop": pop,
                    f"{name}/fitness": cs, f"{name}/under": under, f"{name}/under_fitness": ucost,
                    f"{name}/min_cost_sum": mcs})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
