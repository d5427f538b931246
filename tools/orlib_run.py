"""OR-Library p-median runs (BASELINE.json configs 1-2; acceptance.cpp:294-340
criterion 7; bench.cpp:106-168 for the file format), idle until the files exist.

    python tools/orlib_run.py --orlib-dir DIR [--instances pmed1,pmed40] [--seeds 1]
                              [--reference] [--acceptance]

DIR holds the OR-Library graph files (pmed1 .. pmed40, optionally with .txt /
.dat extensions) and their optima, either as the OR-Library `pmedopt` table
("pmedN <optimum>" per line) or as `<name>.opt` sidecars (the reference CLI's
convention, tools/pmedian_bench.cpp:85-88).  For every instance it parses the
graph (the reference's parse_orlib diagnostics, the shortest-path closure on
the GPU), runs the paper's Table-1 GA (nb=60, nt=256, evolve_limit=100,
saturation=10) per seed through the library's run_ga, and
prints one JSON line: best vs optimum, ratio, kernel of best, gens/s.  With
--reference it times the reference's own run_ga (oracle/_ref) on the same file
for the CPU arm; with --acceptance it also runs the reference's acceptance gate
(tests/cpp/_ref/acceptance --orlib-dir DIR: criterion 7 on pmed1..pmed5).
Nothing is fabricated: a missing file is reported and skipped.
"""
import argparse
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def find_instance(d, name):
    for ext in ("", ".txt", ".dat"):
        p = os.path.join(d, name + ext)
        if os.path.exists(p):
            return p
    return None


def optima(d):
    """name -> optimum, from `pmedopt` (any "name value" lines) and `.opt` sidecars."""
    out = {}
    for cand in ("pmedopt", "pmedopt.txt"):
        p = os.path.join(d, cand)
        if os.path.exists(p):
            with open(p) as f:
                for line in f:
                    m = re.match(r"\s*(\S+)\s+(-?\d+)\s*$", line)
                    if m:
                        out[m.group(1)] = int(m.group(2))
    for fn in os.listdir(d):
        if fn.endswith(".opt"):
            with open(os.path.join(d, fn)) as f:
                tok = f.read().split()
            if tok:
                out.setdefault(fn[:-4], int(tok[0]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orlib-dir", required=True)
    ap.add_argument("--instances", default=",".join(f"pmed{i}" for i in range(1, 41)))
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--nb", type=int, default=60)
    ap.add_argument("--nt", type=int, default=256)
    ap.add_argument("--evolve-limit", type=int, default=100)
    ap.add_argument("--saturation", type=int, default=10)
    ap.add_argument("--reference", action="store_true", help="also time the reference run_ga (oracle/_ref)")
    ap.add_argument("--acceptance", action="store_true", help="also run the reference acceptance gate")
    args = ap.parse_args()
    d = args.orlib_dir
    if not os.path.isdir(d):
        print(json.dumps({"orlib": "unavailable", "reason": f"{d} is not a directory"}))
        return 0
    import paper_1610_10061_b200 as pm
    opt = optima(d)
    ctx = pm.Context(0)
    ran = 0
    for name in filter(None, args.instances.split(",")):
        path = find_instance(d, name)
        if path is None:
            print(json.dumps({"instance": name, "skipped": "file not found"}))
            continue
        with open(path) as f:
            text = f.read()
        t0 = time.perf_counter()
        ctx.set_instance_orlib(text)
        build_s = time.perf_counter() - t0
        rows = []
        for seed in range(1, args.seeds + 1):
            cfg = pm.ga_config(nb=args.nb, nt=args.nt, evolve_limit=args.evolve_limit,
                               saturation=args.saturation, seed=seed)
            r = ctx.run_ga(cfg)
            rows.append(r)
        best = min(r["best_cost"] for r in rows)
        line = {"instance": name, "n": ctx.n, "p": ctx.p, "seeds": args.seeds,
                "config": f"nb={args.nb}, nt={args.nt}, evolve_limit={args.evolve_limit}, "
                          f"saturation={args.saturation} (PAPER.md Table 1)",
                "best_cost": best, "optimum": opt.get(name),
                "ratio": (opt[name] / best) if name in opt and best else None,
                "optimal": (best == opt[name]) if name in opt else None,
                "kernel_of_best": [int(r["kernel_of_best"]) for r in rows],
                "gens_per_s": sum(r["kernels_executed"] for r in rows) / sum(r["wall_time"] for r in rows),
                "closure_and_build_s": round(build_s, 3)}
        if args.reference:
            from oracle.oracle import RefLib
            ref = RefLib()
            nv = int(text.split()[0])
            rc, n, m, p, costs = ref.parse(text, orlib=True, cap=nv * nv)
            ri = ref.create(n, m, p, costs)
            t0 = time.perf_counter()
            rc, rr = ri.run_ga(args.nb, args.nt, args.evolve_limit, args.saturation, 1,
                               workers=len(os.sched_getaffinity(0)))
            line["reference"] = {"best_cost": rr["best_cost"], "kernels": rr["kernels_executed"],
                                 "gens_per_s": rr["kernels_executed"] / max(rr["wall_time"], 1e-9),
                                 "same_run_as_gpu_seed1": rr["best_cost"] == rows[0]["best_cost"]
                                 and rr["kernels_executed"] == rows[0]["kernels_executed"],
                                 "wall_s": time.perf_counter() - t0}
        print(json.dumps(line), flush=True)
        ran += 1
    ctx.close()
    if args.acceptance:
        exe = os.path.join(ROOT, "tests", "cpp", "_ref", "acceptance")
        if os.path.exists(exe):
            r = subprocess.run([exe, "--orlib-dir", d], capture_output=True, text=True)
            crit7 = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion 7")]
            print(json.dumps({"acceptance_criterion_7": crit7[0] if crit7 else None, "rc": r.returncode}))
    if ran == 0:
        print(json.dumps({"orlib": "no instance files found", "dir": d}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
