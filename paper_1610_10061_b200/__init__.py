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
# PMB_LIBRARY: an alternative in-tree build of the same library (A/B kernel
# experiments, tools/build_ab.sh); the default is the one `make` builds
LIB_PATH = os.environ.get("PMB_LIBRARY") or os.path.join(_HERE, "libpmedian_b200.so")

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
_lib.pm_scan_walks_device.argtypes = [_vp, _vp, _sz, _sz, _vp, _vp]
_lib.pm_set_profiling.argtypes = [_vp, C.c_int]
_lib.pm_profile_read.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]


class GaConfig(C.Structure):
    """pmedian::GaConfig (ga.hpp:24-38); crossover/mutation_iters < 0 mean lg(nt)."""
    _fields_ = [("nb", _sz), ("nt", _sz), ("evolve_limit", _sz), ("saturation", _sz),
                ("seed", C.c_uint64), ("crossover_iters", C.c_longlong),
                ("mutation_iters", C.c_longlong), ("migration", C.c_int), ("population", C.c_int)]


class _RunResult(C.Structure):
    _fields_ = [("best_cost", C.c_int64), ("kernels_executed", _sz), ("kernel_of_best", _sz),
                ("wall_time_s", C.c_double), ("evolve_time_s", C.c_double),
                ("evaluations", C.c_uint64), ("device_evaluations", C.c_uint64)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_lib.pm_evolve_blocks.argtypes = [_vp, _vp, _sz, _sz, C.POINTER(GaConfig), C.c_uint64, _sz, _vp, _vp]
_lib.pm_run_ga.argtypes = [_vp, C.POINTER(GaConfig), _vp, _vp, C.POINTER(_RunResult)]
_lib.pm_run_ga_islands.argtypes = [_vp, C.POINTER(GaConfig), C.c_int, C.c_int, ALLGATHER_FN, _vp, _vp,
                                   _vp, C.POINTER(_RunResult)]
ALLGATHER_DEVICE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p)
_lib.pm_run_ga_islands_device.argtypes = [_vp, C.POINTER(GaConfig), C.c_int, C.c_int, _vp, _vp, _vp, _vp,
                                          C.POINTER(_RunResult)]
_lib.pm_last_per_kernel_best.argtypes = [_vp, _vp, _sz, C.POINTER(_sz)]
_lib.pm_set_instance_orlib.argtypes = [_vp, C.c_char_p, _sz, _sz]
_lib.pm_set_instance_dense.argtypes = [_vp, C.c_char_p, _sz, _sz]
_lib.pm_orlib_closure.argtypes = [_vp, C.c_char_p, _sz, _vp, _sz, C.POINTER(_sz), C.POINTER(_sz)]
MIGRATE_BLOCK, MIGRATE_TEAM = 0, 1
POPULATION_REFERENCE, POPULATION_DEVICE = 0, 1


class _TableInfo(C.Structure):
    _fields_ = [("clients", _sz), ("sites", _sz), ("open_count", _sz), ("width", _sz),
                ("row_stride", _sz), ("site_bytes", C.c_int), ("dist_bytes", C.c_int),
                ("max_cost", C.c_int64)]


_lib.pm_table_info_get.argtypes = [_vp, C.POINTER(_TableInfo)]

EVAL_AUTO, EVAL_SCAN, EVAL_GATHER = 0, 1, 2
C_ABI_SYMBOLS = (
    "pm_warmup", "pm_create", "pm_destroy", "pm_last_error", "pm_set_stream", "pm_kernel_launches",
    "pm_set_instance", "pm_set_instance_device", "pm_table_info_get", "pm_get_tables",
    "pm_evaluate", "pm_evaluate_device", "pm_check_errors", "pm_set_eval_kernel",
    "pm_auto_eval_kernel", "pm_min_cost_sum", "pm_scan_depths_device", "pm_scan_walks_device", "pm_set_profiling",
    "pm_profile_read", "pm_evolve_blocks", "pm_run_ga", "pm_run_ga_islands", "pm_set_instance_orlib",
    "pm_orlib_closure", "pm_set_instance_dense", "pm_nccl_unique_id", "pm_nccl_create", "pm_nccl_destroy",
    "pm_nccl_allgather", "pm_nccl_allgather_device", "pm_nccl_rank", "pm_run_ga_islands_device",
    "pm_last_per_kernel_best", "pm_parse_dense",
)


def ga_config(nb=60, nt=256, evolve_limit=100, saturation=10, seed=1, crossover_iters=None,
              mutation_iters=None, team=False, population="reference") -> GaConfig:
    return GaConfig(nb, nt, evolve_limit, saturation, seed,
                    -1 if crossover_iters is None else crossover_iters,
                    -1 if mutation_iters is None else mutation_iters,
                    MIGRATE_TEAM if team else MIGRATE_BLOCK,
                    POPULATION_REFERENCE if population == "reference" else POPULATION_DEVICE)


_lib.pm_nccl_unique_id.argtypes = [C.c_char_p]
_lib.pm_nccl_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
_lib.pm_nccl_destroy.argtypes = [_vp]
_lib.pm_nccl_destroy.restype = None
_lib.pm_nccl_allgather.argtypes = [_vp, _sz, _vp, _vp]
_NCCL_ALLGATHER = ALLGATHER_FN(("pm_nccl_allgather", _lib))
# the device collective's address, passed straight back into the library (no Python in the loop)
_NCCL_ALLGATHER_DEVICE = C.cast(_lib.pm_nccl_allgather_device, _vp)
_lib.pm_nccl_rank.argtypes = [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """pm_nccl_unique_id: rank 0 creates it, the launcher hands it to every rank."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    if _lib.pm_nccl_unique_id(buf) != 0:
        raise NcclError("ncclGetUniqueId failed")
    return buf.raw


class NcclComm:
    """The library's native island communicator (pm_nccl_create); pass it as
    `allgather` to Context.run_ga."""

    def __init__(self, unique_id: bytes, rank: int, world: int, device: int = 0):
        h = _vp()
        rc = _lib.pm_nccl_create(C.create_string_buffer(unique_id, NCCL_ID_BYTES), rank, world, device,
                                 C.byref(h))
        if rc != 0:
            raise NcclError(f"pm_nccl_create failed ({rc})")
        self._h = h
        self.world = world

    def allgather(self, data: bytes) -> bytes:
        """One pm_nccl_allgather: every rank's `data` (equal sizes), in rank order."""
        send = C.create_string_buffer(data, len(data))
        recv = C.create_string_buffer(len(data) * self.world)
        rc = _lib.pm_nccl_allgather(send, len(data), recv, self._h)
        if rc != 0:
            raise NcclError(f"pm_nccl_allgather failed ({rc})")
        return recv.raw

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pm_nccl_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def torch_allgather(group=None, device=None):
    """An island allgather over torch.distributed (gloo on CPU tensors, NCCL on
    CUDA tensors) in the pm_allgather_fn shape."""
    import torch
    import torch.distributed as dist

    def fn(send, nbytes, recv, _user):
        try:
            world = dist.get_world_size(group)
            src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,))
            t = torch.from_numpy(src.copy())
            if device is not None:
                t = t.to(device)
            outs = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(outs, t, group=group)
            dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), shape=(nbytes * world,))
            dst[:] = torch.cat(outs).cpu().numpy()
            return 0
        except Exception:
            return 1

    return fn


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
        self._stream_handle = handle

    def _after_torch(self, *tensors) -> None:
        """Device buffers written by torch on its current stream must be complete
        before the context's stream reads them: nothing to do when the context
        runs on that same stream (set_stream), else wait for it on the host
        (the context's own stream is non-blocking, so it does not order against
        torch's default stream by itself)."""
        import torch
        for t in tensors:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                cur = torch.cuda.current_stream(t.device)
                h = cur.cuda_stream or 1
                if getattr(self, "_stream_handle", None) != h:
                    cur.synchronize()
                return

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
            self._after_torch(costs)
            self._check(_lib.pm_set_instance_device(self._h, _ptr(costs), n, m, p))
        self.n, self.m, self.p = n, m, p

    def set_instance_orlib(self, text: str, p: int = 0) -> None:
        """parse_orlib (bench.cpp:106-168) with the closure on the device."""
        b = text.encode()
        self._check(_lib.pm_set_instance_orlib(self._h, b, len(b), p))
        ti = self.table_info()
        self.n, self.m, self.p = ti.clients, ti.sites, ti.open_count

    def set_instance_dense(self, text: str, p: int = 0) -> None:
        """parse_dense (bench.cpp:65-104)."""
        b = text.encode()
        self._check(_lib.pm_set_instance_dense(self._h, b, len(b), p))
        ti = self.table_info()
        self.n, self.m, self.p = ti.clients, ti.sites, ti.open_count

    def orlib_closure(self, text: str):
        """-> (n, p, costs int64 [n*n]) -- the graph's shortest-path closure."""
        b = text.encode()
        n, p = _sz(0), _sz(0)
        self._check(_lib.pm_orlib_closure(self._h, b, len(b), None, 0, C.byref(n), C.byref(p)))
        out = np.zeros(n.value * n.value, dtype=np.int64)
        self._check(_lib.pm_orlib_closure(self._h, b, len(b), out.ctypes.data, out.size, C.byref(n),
                                          C.byref(p)))
        return n.value, p.value, out

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
        self._after_torch(words)
        rc = _lib.pm_evaluate_device(self._h, _ptr(words), count, wp, _ptr(costs_out),
                                     C.byref(fb) if check else None)
        self._check(rc, fb.value)

    def check_errors(self) -> None:
        fb = _sz(0)
        self._check(_lib.pm_check_errors(self._h, C.byref(fb)), fb.value)

    def scan_depths_device(self, words, sum_k_out, count: int, wp: int) -> None:
        """sum_k_out[c] = sum_i k*_i (1-based stopping columns) for chromosome c."""
        self._after_torch(words)
        self._check(_lib.pm_scan_depths_device(self._h, _ptr(words), count, wp, _ptr(sum_k_out)))

    def scan_walks_device(self, words, group_sum_out, client_max_out, count: int, wp: int) -> None:
        """group_sum_out[g] (int64, ceil(count/32)) = sum_i max_{c in group g} k*_ic;
        client_max_out[i] (int32, n) = max over groups (measurement only)."""
        self._after_torch(words)
        self._check(_lib.pm_scan_walks_device(self._h, _ptr(words), count, wp, _ptr(group_sum_out),
                                              _ptr(client_max_out)))

    def set_profiling(self, on: bool) -> None:
        self._check(_lib.pm_set_profiling(self._h, int(on)))

    def profile_read(self):
        """-> (summed ms, launches) of the dominant kernel since the last read."""
        ms, n = C.c_double(0), C.c_uint64(0)
        self._check(_lib.pm_profile_read(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # ---- GA (ga.cpp) ----------------------------------------------------------------
    def evolve_blocks(self, blocks, cfg: GaConfig, kernel_index: int, first_block: int = 0):
        """pmedian::evolve_block over nb = len(blocks)/cfg.nt consecutive blocks (in place on a
        copy).  -> (blocks_out [nb*nt, wp], best_cost[nb], best_thread[nb])"""
        b = np.ascontiguousarray(blocks, dtype=np.uint64).copy()
        if b.ndim == 1:
            b = b[None, :]
        nb = b.shape[0] // cfg.nt
        bc = np.zeros(max(nb, 1), dtype=np.int64)
        bt = np.zeros(max(nb, 1), dtype=np.uint64)
        self._check(_lib.pm_evolve_blocks(self._h, b.ctypes.data, nb, b.shape[1], C.byref(cfg), kernel_index,
                                          first_block, bc.ctypes.data, bt.ctypes.data))
        return b, bc[:nb], bt[:nb].astype(np.int64)

    def run_ga(self, cfg: GaConfig, rank: int = 0, world: int = 1, allgather=None, allgather_device=None):
        """pmedian::run_ga -> dict with the RunResult fields (ga.hpp:49-56) and work counters.
        allgather: None (one island), a NcclComm (the library's device NCCL exchange,
        records never leave the GPU) or a pm_allgather_fn-shaped host callable;
        allgather_device: a pm_allgather_device_fn-shaped callable
        (send_dev, bytes, recv_dev, stream, user) that gathers device buffers."""
        wp = words_per(self.m)
        best = np.zeros(wp, dtype=np.uint64)
        r = _RunResult()
        if allgather_device is not None:
            cb = ALLGATHER_DEVICE_FN(allgather_device)
            rc = _lib.pm_run_ga_islands_device(self._h, C.byref(cfg), rank, world, C.cast(cb, _vp), None,
                                               best.ctypes.data, None, C.byref(r))
        elif world == 1 and allgather is None:
            rc = _lib.pm_run_ga(self._h, C.byref(cfg), best.ctypes.data, None, C.byref(r))
        elif isinstance(allgather, NcclComm):  # the library's own NCCL exchange, no Python in the loop
            rc = _lib.pm_run_ga_islands_device(self._h, C.byref(cfg), rank, world, _NCCL_ALLGATHER_DEVICE,
                                               allgather._h, best.ctypes.data, None, C.byref(r))
        else:
            cb = ALLGATHER_FN(allgather)
            rc = _lib.pm_run_ga_islands(self._h, C.byref(cfg), rank, world, cb, None, best.ctypes.data,
                                        None, C.byref(r))
        self._check(rc)
        per = np.zeros(r.kernels_executed, dtype=np.int64)
        cnt = _sz(0)
        self._check(_lib.pm_last_per_kernel_best(self._h, per.ctypes.data if per.size else None, per.size,
                                                 C.byref(cnt)))
        return dict(best=best, best_cost=r.best_cost, kernels_executed=r.kernels_executed,
                    kernel_of_best=r.kernel_of_best, per_kernel_best_costs=per[:r.kernels_executed].copy(),
                    wall_time=r.wall_time_s, evolve_time=r.evolve_time_s, evaluations=r.evaluations,
                    device_evaluations=r.device_evaluations)

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
