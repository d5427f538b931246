"""bench.py's multi-rank path (torchrun, strong split of one batch with the
costs all-gathered, weak scaling, max-over-ranks timing, island GA allgather)
end to end.  Two ranks share the one GPU over gloo: the
collectives are host-side, so no kernel waits on another rank."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_two_ranks_gloo_one_gpu(scaling):
    env = dict(os.environ, PMB_DIST_BACKEND="gloo", PMB_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--config", "syn5k", "--no-cpu-baseline", "--scaling", scaling]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 prints one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    # strong: BASELINE config 3 -- one 1024-chromosome batch, 512 per GPU
    assert d["config"]["population"] == (1024 if scaling == "strong" else 2048)
    assert d["details"]["per_gpu_chromosomes"] == (512 if scaling == "strong" else 1024)
    assert d["ga"]["islands"]["generations"] >= 1
