"""Regenerates tests/golden/baseline_golden.{json,npz} from the REFERENCE ITSELF
at every BASELINE.json size.

Runs in the build container only: it needs oracle/_ref/libpmref.so, the
reference's unmodified sources (/root/reference/proj/src) compiled by
oracle/Makefile.  For each shape it records

* the reference build_ordering tables (ordering.cpp:10-38) as SHA-256 digests
  of the exact bytes pm_get_tables returns (site_order u32 [n, W] and
  increments i64 [n, W], row-major), whole-table and per 2048-row slab;
* the reference fitness() (ordering.cpp:40-59) of EVERY chromosome of the
  benchmark population (seed 7), evaluated on the
  reference's own tables;
* two reference run_ga RunResults (ga.cpp:219-303): the paper's Table-1 run at
  the pmed40 shape (nb=60, nt=256, evolve_limit=100, saturation=10, seed 1;
  acceptance.cpp:323-328) and two generations of the syn20k island GA
  (nb=16, nt=256, seed 1) that bench.py times.

The GPU tests (tests/test_gpu_baseline.py) compare the device path against
these on the GPU box, where /root/reference does not exist.

    python tests/golden/make_baseline_golden.py [--only name,...]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, RefLib  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
JSON_OUT = os.path.join(HERE, "baseline_golden.json")
NPZ_OUT = os.path.join(HERE, "baseline_golden.npz")
SLAB = 2048

# (name, npts, p, population size) -- BASELINE.json configs 2-5
SHAPES = [("pmed40", 900, 90, 15360), ("syn5k", 5000, 50, 1024), ("syn20k", 20000, 200, 4096)] + [
    (f"sweep{p}", 10000, p, 4096) for p in (10, 20, 50, 100, 200, 500, 1000)]

GA_RUNS = {  # name: (npts, p, nb, nt, evolve_limit, saturation, seed)
    "table1_pmed40_shape": (900, 90, 60, 256, 100, 10, 1),
    "syn20k_islands_2gen": (20000, 200, 16, 256, 2, 3, 1),
    # the run bench.py times for the syn20k island GA figure (evolve_limit 20, saturation 21)
    "syn20k_islands_20gen": (20000, 200, 16, 256, 20, 21, 1),
}


def digests(a: np.ndarray):
    a = np.ascontiguousarray(a)
    slabs = [hashlib.sha256(a[r:r + SLAB].tobytes()).hexdigest() for r in range(0, a.shape[0], SLAB)]
    return hashlib.sha256(a.tobytes()).hexdigest(), slabs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    o, ref = Oracle(), RefLib()
    threads = len(os.sched_getaffinity(0))
    meta = json.load(open(JSON_OUT)) if os.path.exists(JSON_OUT) else {"shapes": {}, "ga": {}}
    arrays = dict(np.load(NPZ_OUT)) if os.path.exists(NPZ_OUT) else {}
    for name, npts, p, count in SHAPES:
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        costs = o.synth_euclid(npts)
        ri = ref.create(npts, npts, p, costs)
        assert ri.rc == 0, ref.last_error()
        tb = time.perf_counter() - t0
        so, inc = ri.tables()
        so_all, so_slabs = digests(so)
        inc_all, inc_slabs = digests(inc)
        del so, inc
        pop = o.random_population(npts, p, count, seed=7)
        t1 = time.perf_counter()
        rc, fit, _ = ri.evaluate(pop, threads)
        assert rc == 0
        te = time.perf_counter() - t1
        del ri
        meta["shapes"][name] = dict(n=npts, m=npts, p=p, count=count, instance_seed=12345, population_seed=7,
                                    width=npts - p + 1, slab_rows=SLAB, site_order_sha256=so_all,
                                    increments_sha256=inc_all, site_order_slabs=so_slabs,
                                    increments_slabs=inc_slabs,
                                    fitness_sum=int(fit.sum()), reference_build_ordering_s=round(tb, 2),
                                    reference_fitness_s=round(te, 2), reference_threads=threads)
        arrays[f"{name}/fitness"] = fit
        print(f"{name}: build_ordering {tb:.1f} s, fitness x{count} {te:.1f} s", flush=True)
    for name, (npts, p, nb, nt, lim, sat, seed) in GA_RUNS.items():
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        ri = ref.create(npts, npts, p, o.synth_euclid(npts))
        assert ri.rc == 0
        rc, r = ri.run_ga(nb, nt, lim, sat, seed, workers=threads)
        assert rc == 0, ref.last_error()
        meta["ga"][name] = dict(n=npts, m=npts, p=p, nb=nb, nt=nt, evolve_limit=lim, saturation=sat, seed=seed,
                                best_cost=int(r["best_cost"]), kernels_executed=int(r["kernels_executed"]),
                                kernel_of_best=int(r["kernel_of_best"]),
                                per_kernel_best_costs=[int(x) for x in r["per_kernel_best_costs"]],
                                best_words=[int(x) for x in r["best"]],
                                reference_wall_s=round(time.perf_counter() - t0, 1), reference_threads=threads)
        print(f"{name}: run_ga {time.perf_counter() - t0:.1f} s, best {r['best_cost']}, "
              f"{r['kernels_executed']} kernels", flush=True)
        del ri
    meta["generated_by"] = ("tests/golden/make_baseline_golden.py: oracle/_ref/libpmref.so = the reference's "
                            "unmodified proj/src (ordering, instance, chromosome, ga, combinatorics .cpp)")
    with open(JSON_OUT, "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(NPZ_OUT, **arrays)


if __name__ == "__main__":
    main()
