"""tools/orlib_run.py (BASELINE configs 1-2 once the OR-Library files exist):
exercised on a synthetic graph written in the OR-Library format -- clearly
not a pmed file -- whose optimum is found exhaustively on the device."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _graph(seed, n, extra):
    from oracle.oracle import Oracle
    st = Oracle().stream(seed)
    edges = []
    for v in range(2, n + 1):  # spanning tree keeps it connected
        edges.append((1 + st.below(v - 1), v, 1 + st.below(50)))
    for _ in range(extra):
        u, v = 1 + st.below(n), 1 + st.below(n)
        if u != v:
            edges.append((u, v, 1 + st.below(50)))
    return edges


def test_runner_idles_without_files(tmp_path):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "orlib_run.py"), "--orlib-dir",
                        str(tmp_path / "absent")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "unavailable" in r.stdout


@pytest.mark.gpu
def test_runner_reaches_the_exhaustive_optimum_and_matches_the_reference(tmp_path, pm):
    n, p = 40, 3
    edges = _graph(77, n, 60)
    text = f"{n} {len(edges)} {p}\n" + "".join(f"{u} {v} {c}\n" for u, v, c in edges)
    (tmp_path / "synthA").write_text(text)
    import torch

    from paper_1610_10061_b200 import synth
    ctx = pm.Context(0)
    ctx.set_instance_orlib(text)
    best = None
    for chunk in synth.all_subsets(n, p):
        w = torch.from_numpy(chunk.view(np.int64)).cuda()
        out = torch.empty(chunk.shape[0], dtype=torch.int64, device="cuda")
        ctx.evaluate_device(w, out, chunk.shape[0], chunk.shape[1], check=True)
        v = int(out.min().item())
        best = v if best is None else min(best, v)
    ctx.close()
    (tmp_path / "pmedopt").write_text(f"synthA {best}\n")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "orlib_run.py"), "--orlib-dir", str(tmp_path),
                        "--instances", "synthA", "--nb", "4", "--nt", "32", "--reference"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.splitlines()[0])
    assert line["optimum"] == best and line["optimal"] is True
    assert line["reference"]["same_run_as_gpu_seed1"] is True
