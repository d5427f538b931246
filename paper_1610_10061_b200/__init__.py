"""B200-native HBP fitness path for arXiv 1610.10061 (pmedian).

Python view of the C ABI in ``include/pmedian_b200.h`` (libpmedian_b200.so,
built in-tree by ``make`` / ``__graft_entry__.build()``).  Names mirror the
reference's C++ API (/root/reference/proj/include/pmedian/): ``build_ordering``
(ordering.hpp:33), ``fitness`` (ordering.hpp:39), ``min_cost_sum``
(instance.hpp:39), and the reference's error types (errors.hpp:8-25).

There is no CPU path: every cost comes from a CUDA kernel, and importing the
module fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpmedian_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
        "(there is deliberately no CPU fallback)")

_lib = C.CDLL(LIB_PATH)
_sz = C.c_size_t
_vp = C.c_void_p

_lib.pm_create.argtypes = [C.c_int, C.POINTER(_vp)]
_lib.pm_destroy.argtypes = [_vp]
_lib.pm_last_error.restype = C.c_char_p
_lib.pm_last_error.argtypes = [_vp]
_lib.pm_set_stream.argtypes = [_vp, _vp]
_lib.pm_kernel_launches.restype = C.c_uint64
_lib.pm_kernel_launches.argtypes = [_vp]
_lib.pm_set_instance.argtypes = [_vp, _vp, _sz, _sz, _sz]
_lib.pm_set_instance_device.argtypes = [_vp, _vp, _sz, _sz, _sz]
_lib.pm_get_tables.argtypes = [_vp, _vp, _vp]
_lib.pm_evaluate.argtypes = [_vp, _vp, _sz, _sz, _vp, C.POINTER(_sz)]
_lib.pm_evaluate_device.argtypes = [_vp, _vp, _sz, _sz, _vp, C.POINTER(_sz)]
_lib.pm_check_errors.argtypes = [_vp, C.POINTER(_sz)]
_lib.pm_set_eval_kernel.argtypes = [_vp, C.c_int]
_lib.pm_auto_eval_kernel.argtypes = [_vp]
_lib.pm_min_cost_sum.argtypes = [_vp, _vp, _sz, _sz, _vp, C.POINTER(_sz)]
_lib.pm_scan_depths_device.argtypes = [_vp, _vp, _sz, _sz, _vp]
_lib.pm_set_profiling.argtypes = [_vp, C.c_int]
_lib.pm_profile_read.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]


class _TableInfo(C.Structure):
    _fields_ = [("clients", _sz), ("sites", _sz), ("open_count", _sz), ("width", _sz),
                ("row_stride", _sz), ("site_bytes", C.c_int), ("dist_bytes", C.c_int),
                ("max_cost", C.c_int64)]


_lib.pm_table_info_get.argtypes = [_vp, C.POINTER(_TableInfo)]

EVAL_AUTO, EVAL_SCAN, EVAL_GATHER = 0, 1, 2
C_ABI_SYMBOLS = (
    "pm_create", "pm_destroy", "pm_last_error", "pm_set_stream", "pm_kernel_launches",
    "pm_set_instance", "pm_set_instance_device", "pm_table_info_get", "pm_get_tables",
    "pm_evaluate", "pm_evaluate_device", "pm_check_errors", "pm_set_eval_kernel",
    "pm_auto_eval_kernel", "pm_min_cost_sum", "pm_scan_depths_device", "pm_set_profiling",
    "pm_profile_read",
)


# ---- errors: pmedian/errors.hpp:8-25 --------------------------------------------

class PmError(Exception):
    status = -1


class StructuralError(PmError):  # std::runtime_error in the reference
    status = 1


class ContractError(PmError):  # std::logic_error in the reference
    status = 2

    def __init__(self, msg, first_bad=None):
        super().__init__(msg)
        self.first_bad = first_bad


class DomainError(PmError, ValueError):  # std::invalid_argument in the reference
    status = 3


class BudgetError(PmError):
    status = 4


class CudaError(PmError):
    status = 5


class NcclError(PmError):
    status = 6


_BY_STATUS = {1: StructuralError, 2: ContractError, 3: DomainError, 4: BudgetError, 5: CudaError,
              6: NcclError}


def words_per(m: int) -> int:
    return (m + 63) // 64


@dataclass
class TableInfo:
    clients: int
    sites: int
    open_count: int
    width: int
    row_stride: int
    site_bytes: int
    dist_bytes: int
    max_cost: int


def _ptr(a) -> int:
    """Host numpy array or CUDA tensor -> raw address."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())


class Context:
    """One device, one stream, resident tables (the C ABI's pm_ctx)."""

    def __init__(self, device: int = 0):
        h = _vp()
        rc = _lib.pm_create(device, C.byref(h))
        if rc != 0:
            raise _BY_STATUS.get(rc, PmError)(f"pm_create(device={device}) failed with status {rc}")
        self._h = h
        self.device = device
        self.m = self.n = self.p = None

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pm_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --------------------------------------------------------------------------
    def _check(self, rc, first_bad=None):
        if rc == 0:
            return
        msg = _lib.pm_last_error(self._h).decode()
        cls = _BY_STATUS.get(rc, PmError)
        if cls is ContractError:
            raise ContractError(msg, first_bad)
        raise cls(msg)

    @property
    def kernel_launches(self) -> int:
        return int(_lib.pm_kernel_launches(self._h))

    def set_stream(self, stream) -> None:
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
        if stream is None:
            handle = None  # the context's own stream
        else:
            handle = int(getattr(stream, "cuda_stream", stream))
            if handle == 0:
                handle = 1  # torch's default stream is the legacy NULL stream: cudaStreamLegacy
        self._check(_lib.pm_set_stream(self._h, handle))

    def set_eval_kernel(self, kind: int) -> None:
        self._check(_lib.pm_set_eval_kernel(self._h, kind))

    def auto_eval_kernel(self) -> int:
        return int(_lib.pm_auto_eval_kernel(self._h))

    # ---- instance + K1 (Instance ctor instance.cpp:10-30, build_ordering ordering.cpp:10-38)
    def set_instance(self, costs, n: int, m: int, p: int) -> None:
        if isinstance(costs, np.ndarray) or isinstance(costs, (list, tuple)):
            a = np.ascontiguousarray(costs, dtype=np.int64)
            if a.size != n * m:
                raise StructuralError("cost matrix must be exactly n rows by m columns")
            self._check(_lib.pm_set_instance(self._h, a.ctypes.data if a.size else None, n, m, p))
        else:  # CUDA tensor of int64
            if costs.numel() != n * m:
                raise StructuralError("cost matrix must be exactly n rows by m columns")
            self._check(_lib.pm_set_instance_device(self._h, _ptr(costs), n, m, p))
        self.n, self.m, self.p = n, m, p

    def table_info(self) -> TableInfo:
        ti = _TableInfo()
        self._check(_lib.pm_table_info_get(self._h, C.byref(ti)))
        return TableInfo(ti.clients, ti.sites, ti.open_count, ti.width, ti.row_stride,
                         ti.site_bytes, ti.dist_bytes, ti.max_cost)

    def get_tables(self):
        """-> (site_order uint32 [n, W], increments int64 [n, W]) in the reference layout."""
        ti = self.table_info()
        so = np.empty((ti.clients, ti.width), dtype=np.uint32)
        inc = np.empty((ti.clients, ti.width), dtype=np.int64)
        self._check(_lib.pm_get_tables(self._h, so.ctypes.data, inc.ctypes.data))
        return so, inc

    # ---- K2 / K2b (fitness ordering.cpp:40-59) -------------------------------------
    def evaluate(self, words: np.ndarray) -> np.ndarray:
        """Host population [count, words_per] uint64 -> int64 costs (synchronous)."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        if w.ndim == 1:
            w = w[None, :]
        count, wp = w.shape
        out = np.zeros(count, dtype=np.int64)
        fb = _sz(0)
        rc = _lib.pm_evaluate(self._h, w.ctypes.data if w.size else None, count, wp,
                              out.ctypes.data if count else None, C.byref(fb))
        self._check(rc, fb.value)
        return out

    def evaluate_device(self, words, costs_out, count: int, wp: int, check: bool = True):
        """CUDA buffers (torch tensors): words int64/uint64 [count, wp], costs_out int64 [count].
        check=False keeps the call asynchronous (errors via check_errors())."""
        fb = _sz(0)
        rc = _lib.pm_evaluate_device(self._h, _ptr(words), count, wp, _ptr(costs_out),
                                     C.byref(fb) if check else None)
        self._check(rc, fb.value)

    def check_errors(self) -> None:
        fb = _sz(0)
        self._check(_lib.pm_check_errors(self._h, C.byref(fb)), fb.value)

    def scan_depths_device(self, words, sum_k_out, count: int, wp: int) -> None:
        """sum_k_out[c] = sum_i k*_i (1-based stopping columns) for chromosome c."""
        self._check(_lib.pm_scan_depths_device(self._h, _ptr(words), count, wp, _ptr(sum_k_out)))

    def set_profiling(self, on: bool) -> None:
        self._check(_lib.pm_set_profiling(self._h, int(on)))

    def profile_read(self):
        """-> (summed ms, launches) of the dominant kernel since the last read."""
        ms, n = C.c_double(0), C.c_uint64(0)
        self._check(_lib.pm_profile_read(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def min_cost_sum(self, words: np.ndarray) -> np.ndarray:
        """instance.cpp:32-48 per chromosome (gather-min, no scan-width contract)."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        if w.ndim == 1:
            w = w[None, :]
        count, wp = w.shape
        out = np.zeros(count, dtype=np.int64)
        fb = _sz(0)
        rc = _lib.pm_min_cost_sum(self._h, w.ctypes.data if w.size else None, count, wp,
                                  out.ctypes.data if count else None, C.byref(fb))
        self._check(rc, fb.value)
        return out


# ---- reference-named conveniences --------------------------------------------------

def build_ordering(costs, n: int, m: int, p: int, device: int = 0) -> Context:
    """pmedian::build_ordering: returns a Context holding the device tables."""
    ctx = Context(device)
    ctx.set_instance(costs, n, m, p)
    return ctx


def fitness(ctx: Context, words) -> int:
    """pmedian::fitness for one chromosome (ordering.hpp:39)."""
    return int(ctx.evaluate(np.asarray(words, dtype=np.uint64).reshape(1, -1))[0])


def evaluate_population(ctx: Context, words) -> np.ndarray:
    return ctx.evaluate(words)
