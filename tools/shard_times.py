"""Per-GPU device time of one step of the strong split (BASELINE configs 3-4)
at N = 1, 2, 4, 8 ranks, measured on one GPU: rank 0's shard (the first
count/N chromosomes of the batch) evaluated alone, CUDA events, L2 flushed.
An upper bound on strong-scaling efficiency (no collective, no skew).
python tools/shard_times.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
print("| config | N | chromosomes per GPU | step ms (device) | evals/s per GPU | N x per-GPU / (1-GPU) |")
print("|---|---|---|---|---|---|")
for name in ("syn20k", "syn5k"):
    cfg = bench.config_for(name)
    n = m = cfg["npts"]
    p, count = cfg["p"], cfg["count"]
    wp = (m + 63) // 64
    ctx = pm.Context(0)
    s = torch.cuda.current_stream()
    ctx.set_stream(s)
    ctx.set_instance(synth.euclid_costs(n, 12345, device="cuda"), n, m, p)
    pop = synth.random_population(m, p, count, seed=7)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    base = None
    for N in (1, 2, 4, 8):
        lo, hi = bench.shard(count, N, 0)
        w = torch.from_numpy(np.ascontiguousarray(pop[lo:hi]).view(np.int64)).cuda()
        out = torch.empty(hi - lo, dtype=torch.int64, device="cuda")
        for _ in range(3):
            ctx.evaluate_device(w, out, hi - lo, wp, check=False)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record(s)
            ctx.evaluate_device(w, out, hi - lo, wp, check=False)
            b.record(s)
        torch.cuda.synchronize()
        ctx.check_errors()
        ms = sum(a.elapsed_time(b) for a, b in ev) / reps
        rate = (hi - lo) / (ms / 1e3)
        base = base or rate
        print(f"| {name} | {N} | {hi - lo} | {ms:.4f} | {rate:,.0f} | {N * rate / base:.2f} |", flush=True)
    ctx.close()
