"""CPU: the C-ABI library loads, exports every symbol include/pmedian_b200.h
declares, and fails loudly (no CPU fallback) when there is no device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "pmedian_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(pm_[a-z_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol(pm):
    lib = ctypes.CDLL(pm.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(pm.C_ABI_SYMBOLS)


def test_library_is_sm100a(pm):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly(pm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(pm.PmError):
        pm.Context(0)


def test_error_taxonomy_matches_reference(pm):
    # errors.hpp:8-25: StructuralError(runtime), ContractError(logic), DomainError(invalid_argument)
    assert issubclass(pm.DomainError, ValueError)
    assert pm.StructuralError.status == 1 and pm.ContractError.status == 2
    assert pm.DomainError.status == 3 and pm.BudgetError.status == 4


def test_library_does_not_pin_nccl_before_torch(pm):
    """The library binds NCCL at run time (islands_nccl.cu): loading it before
    PyTorch must not pin the system libnccl.so.2 under torch's own NCCL."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", "import paper_1610_10061_b200, torch; print(torch.__version__)"],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    with open(pm.LIB_PATH, "rb") as f:
        assert b"libnccl.so.2\x00" in f.read()  # the dlopen name, not a DT_NEEDED entry
    needed = subprocess.run(["readelf", "-d", pm.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in needed
