"""CPU: the vectorised benchmark input generator equals the oracle's sequential
restatement of the reference RandomStream (rng.hpp:22-55)."""
import numpy as np


def test_stream_matches_oracle(oracle):
    from paper_1610_10061_b200.synth import Stream
    for seed in (0, 1, 7, 12345, 2**63 + 5):
        s = Stream(seed)
        o = oracle.stream(seed)
        assert [s.next() for _ in range(50)] == [o.next() for _ in range(50)]
        bounds = [1, 2, 3, 10000, 2**63 + 1, 2**64 - 1, 17, 2**40]
        s2, o2 = Stream(seed), oracle.stream(seed)
        assert s2.below_many(np.array(bounds * 20, dtype=np.uint64)).tolist() == \
            [o2.below(b) for b in bounds * 20]


def test_rejection_path_exact(oracle):
    # bound 2^64-1: threshold 1 -> rejection only for v == 0; bound 2^63+1 rejects ~half
    from paper_1610_10061_b200.synth import Stream
    s, o = Stream(99), oracle.stream(99)
    b = np.full(200, 2**63 + 1, dtype=np.uint64)
    assert s.below_many(b).tolist() == [o.below(2**63 + 1) for _ in range(200)]
    assert s.next() == o.next()


def test_euclid_and_population_match_oracle(oracle):
    from paper_1610_10061_b200 import synth
    for n in (1, 50, 301):
        assert (synth.euclid_costs(n) == oracle.synth_euclid(n)).all()
    for m, p, cnt in ((100, 7, 10), (1000, 100, 5), (64, 63, 3), (130, 1, 4)):
        assert (synth.random_population(m, p, cnt, seed=3) == oracle.random_population(m, p, cnt, seed=3)).all()
