"""Kernel timing experiments: python tools/time_eval.py config kind reps "shape1 shape2 ..." [rounds]
shape = "G,warps" (PMB_SCAN_SHAPE) or "auto"; interleaves shapes over rounds in one process."""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_10061_b200 as pm  # noqa: E402
from paper_1610_10061_b200 import synth  # noqa: E402

cfg = bench.config_for(sys.argv[1] if len(sys.argv) > 1 else "syn20k")
kind = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
shapes = (sys.argv[4] if len(sys.argv) > 4 else "auto").split()
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 2
n = m = cfg["npts"]
p, count = cfg["p"], int(os.environ.get("TE_COUNT") or cfg["count"])  # TE_COUNT: a shard-sized batch
wp = (m + 63) // 64
ctx = pm.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s)
if kind != "auto":
    ctx.set_eval_kernel({"scan": pm.EVAL_SCAN, "gather": pm.EVAL_GATHER}[kind])
costs = synth.euclid_costs(n, 12345, device="cuda")
torch.cuda.synchronize()
ctx.set_instance(costs, n, m, p)
del costs
pop = synth.random_population(m, p, count, seed=7)
words = torch.from_numpy(pop.view(np.int64)).cuda()
out = torch.empty(count, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def clock():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()


ref = None
for r in range(rounds):
    for sh in shapes:
        if sh == "auto":
            os.environ.pop("PMB_SCAN_SHAPE", None)
        else:
            os.environ["PMB_SCAN_SHAPE"] = sh
        with torch.cuda.stream(s):
            try:
                ctx.evaluate_device(words, out, count, wp, check=True)
            except pm.DomainError:
                print(f"{cfg['workload'][:6]} shape={sh} does not fit", flush=True)
                continue
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref)
            ctx.set_profiling(True)
            ctx.profile_read()
            for _ in range(reps):
                if not os.environ.get("TE_NOFLUSH"):
                    flush.zero_()
                ctx.evaluate_device(words, out, count, wp, check=False)
            ms, nl = ctx.profile_read()
            ctx.set_profiling(False)
        print(f"{cfg['workload'][:6]} kind={kind} shape={sh} kernel_ms={ms/nl:.3f} "
              f"evals/s={count/(ms/nl/1e3):.0f} sum={int(out.sum())} clk={clock()}", flush=True)
