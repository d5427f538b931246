import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle.oracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def example1():
    with open(os.path.join(GOLDEN, "example1.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref_vectors():
    z = np.load(os.path.join(GOLDEN, "ref_vectors.npz"))
    cases = {}
    for k in z.files:
        name, field = k.split("/")
        cases.setdefault(name, {})[field] = z[k]
    return cases


@pytest.fixture(scope="session")
def pm():
    import paper_1610_10061_b200 as pm
    return pm


@pytest.fixture()
def ctx(pm):
    c = pm.Context(0)
    yield c
    c.close()
