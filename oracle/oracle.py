"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  The product path (paper_1610_10061_b200)
never does.

* ``Oracle`` wraps ``oracle/liboracle.so``: the C restatement in pmoracle.c.
* ``RefLib`` wraps ``oracle/_ref/libpmref.so``: the reference's own unmodified
  sources from /root/reference/proj/src, compiled by oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libpmref.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_sz = C.c_size_t

STATUS = {0: "ok", 1: "StructuralError", 2: "ContractError", 3: "DomainError", 4: "BudgetError", 9: "Error"}


def build() -> None:
    """Build liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def words_per(m: int) -> int:
    return (m + 63) // 64


def bits_to_words(bits: str) -> np.ndarray:
    """'1001' -> packed words (bit j = word j>>6 bit j&63, chromosome.hpp:24)."""
    w = np.zeros(words_per(len(bits)), dtype=np.uint64)
    for j, ch in enumerate(bits):
        if ch == "1":
            w[j >> 6] |= np.uint64(1) << np.uint64(j & 63)
    return w


def words_to_bits(w: np.ndarray, m: int) -> str:
    return "".join("1" if (int(w[j >> 6]) >> (j & 63)) & 1 else "0" for j in range(m))


def open_to_words(m: int, open_sites) -> np.ndarray:
    w = np.zeros(words_per(m), dtype=np.uint64)
    for j in open_sites:
        w[j >> 6] |= np.uint64(1) << np.uint64(j & 63)
    return w


class Oracle:
    """The C restatement (pmoracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            build()
        L = self.L = C.CDLL(path)
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_rs_derive.restype = C.c_uint64
        L.or_rs_derive.argtypes = [C.c_uint64, _u64p, _sz]
        L.or_rs_next.restype = C.c_uint64
        L.or_rs_next.argtypes = [C.POINTER(C.c_uint64)]
        L.or_rs_below.restype = C.c_uint64
        L.or_rs_below.argtypes = [C.POINTER(C.c_uint64), C.c_uint64]
        L.or_synth_euclid.argtypes = [C.c_uint64, _sz, _i64p]
        L.or_random_costs.argtypes = [C.c_uint64, _sz, _sz, C.c_int64, _i64p]
        L.or_random_population.argtypes = [C.c_uint64, _sz, _sz, _sz, _u64p]
        L.or_validate_instance.argtypes = [_sz, _sz, _sz, _i64p, _sz]
        L.or_build_ordering.argtypes = [_sz, _sz, _sz, _i64p, _u32p, _i64p]
        L.or_evaluate_population.argtypes = [_sz, _sz, _sz, _u32p, _i64p, _u64p, _sz, _sz, _i64p,
                                             _u64p, C.POINTER(_sz)]
        L.or_min_cost_sum.argtypes = [_sz, _sz, _i64p, _u64p, C.POINTER(C.c_int64)]
        L.or_direct_cost.argtypes = [_sz, _sz, _sz, _i64p, _u64p, C.POINTER(C.c_int64)]
        L.or_orlib_closure.argtypes = [_sz, _sz, _i64p, _i64p, _i64p, C.POINTER(_sz)]

    def orlib_closure(self, n, uv, w):
        """uv: 0-based endpoints [edges, 2]; -> (rc, closure n*n, first bad index)"""
        uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1)
        w = np.ascontiguousarray(w, dtype=np.int64)
        out = np.zeros(n * n, dtype=np.int64)
        bad = _sz(0)
        rc = self.L.or_orlib_closure(n, w.size, uv if uv.size else np.zeros(2, np.int64), w if w.size else np.zeros(1, np.int64), out, C.byref(bad))
        return rc, out, bad.value

    # rng.hpp
    def derive(self, master: int, key) -> int:
        k = np.ascontiguousarray(key, dtype=np.uint64)
        if k.size == 0:
            k = np.zeros(1, dtype=np.uint64)
            return self.L.or_rs_derive(master, k, 0)
        return self.L.or_rs_derive(master, k, k.size)

    def stream(self, seed: int):
        st = C.c_uint64(seed)
        L = self.L

        class _S:
            def next(self_):
                return L.or_rs_next(C.byref(st))

            def below(self_, b):
                return L.or_rs_below(C.byref(st), b)

            def coin(self_):
                return (L.or_rs_next(C.byref(st)) & 1) != 0

        return _S()

    # inputs
    def synth_euclid(self, npts: int, seed: int = 12345) -> np.ndarray:
        out = np.empty(npts * npts, dtype=np.int64)
        self.L.or_synth_euclid(seed, npts, out)
        return out

    def random_costs(self, seed: int, n: int, m: int, max_cost: int = 99) -> np.ndarray:
        out = np.empty(n * m, dtype=np.int64)
        self.L.or_random_costs(seed, n, m, max_cost, out)
        return out

    def random_population(self, m: int, p: int, count: int, seed: int = 7) -> np.ndarray:
        out = np.empty(count * words_per(m), dtype=np.uint64)
        self.L.or_random_population(seed, m, p, count, out)
        return out.reshape(count, words_per(m))

    # the path
    def validate_instance(self, n, m, p, costs) -> int:
        costs = np.ascontiguousarray(costs, dtype=np.int64)
        return self.L.or_validate_instance(n, m, p, costs, costs.size)

    def build_ordering(self, n, m, p, costs):
        W = m - p + 1
        so = np.empty(n * W, dtype=np.uint32)
        inc = np.empty(n * W, dtype=np.int64)
        self.L.or_build_ordering(n, m, p, np.ascontiguousarray(costs, dtype=np.int64), so, inc)
        return so.reshape(n, W), inc.reshape(n, W)

    def evaluate(self, site_order, increments, m, words, want_sum_k=False):
        """-> (status, costs, first_bad, sum_k)"""
        n, W = site_order.shape
        words = np.ascontiguousarray(words, dtype=np.uint64)
        count = words.shape[0] if words.ndim == 2 else 1
        wp = words.shape[-1]
        costs = np.zeros(count, dtype=np.int64)
        sk = np.zeros(count, dtype=np.uint64)
        fb = _sz(count)
        rc = self.L.or_evaluate_population(n, m, W, np.ascontiguousarray(site_order),
                                           np.ascontiguousarray(increments), words.reshape(-1), wp,
                                           count, costs, sk, C.byref(fb))
        return rc, costs, fb.value, (sk if want_sum_k else None)

    def min_cost_sum(self, n, m, costs, words):
        out = C.c_int64(0)
        rc = self.L.or_min_cost_sum(n, m, np.ascontiguousarray(costs, dtype=np.int64),
                                    np.ascontiguousarray(words, dtype=np.uint64), C.byref(out))
        return rc, out.value

    def direct_cost(self, n, m, p, costs, words):
        out = C.c_int64(0)
        rc = self.L.or_direct_cost(n, m, p, np.ascontiguousarray(costs, dtype=np.int64),
                                   np.ascontiguousarray(words, dtype=np.uint64), C.byref(out))
        return rc, out.value


class RefLib:
    """The reference's own sources (oracle/_ref/libpmref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(LIB_REF)

    def __init__(self, path: str = LIB_REF):
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_create.argtypes = [_sz, _sz, _sz, _i64p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_create_with_tables.argtypes = [_sz, _sz, _sz, _u32p, _i64p, C.POINTER(C.c_void_p)]
        L.ref_width.restype = _sz
        L.ref_width.argtypes = [C.c_void_p]
        L.ref_get_tables.argtypes = [C.c_void_p, _u32p, _i64p]
        L.ref_evaluate.argtypes = [C.c_void_p, _u64p, _sz, _sz, _i64p, C.POINTER(_sz), C.c_uint]
        L.ref_fitness_bits.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int64)]
        L.ref_min_cost_sum.argtypes = [C.c_void_p, _u64p, C.POINTER(C.c_int64)]
        L.ref_direct_cost.argtypes = [C.c_void_p, _u64p, C.POINTER(C.c_int64)]
        L.ref_exact_optimum.argtypes = [C.c_void_p, C.c_uint64, _u64p, C.POINTER(C.c_int64)]
        L.ref_format_polynomial.argtypes = [C.c_void_p, C.c_int, C.c_char_p, _sz]
        L.ref_evaluate_polynomial.argtypes = [C.c_void_p, C.c_int, _u64p, C.POINTER(C.c_int64)]
        L.ref_crossover.argtypes = [_u64p, _u64p, _sz, _sz, _sz, _u64p, C.POINTER(C.c_int)]
        L.ref_circular_shift.argtypes = [_u64p, _sz, _sz, C.c_int, _u64p]
        L.ref_block_shift.argtypes = [_u64p, _sz, _sz, _sz, _sz, C.c_int, _u64p]
        L.ref_random_shift_mutation.argtypes = [_u64p, _sz, C.POINTER(C.c_uint64), _u64p]
        L.ref_random_chromosome.argtypes = [_sz, _sz, C.c_uint64, _sz, _u64p]
        L.ref_evolve_block.argtypes = [C.c_void_p, _u64p, _sz, _sz, C.c_uint64, C.c_longlong,
                                       C.c_longlong, C.c_uint64, _sz, _u64p, C.POINTER(C.c_int64),
                                       C.POINTER(_sz)]
        L.ref_run_ga.argtypes = [C.c_void_p, _sz, _sz, _sz, _sz, C.c_uint64, C.c_longlong,
                                 C.c_longlong, C.c_int, C.c_uint, _u64p, C.POINTER(C.c_int64),
                                 C.POINTER(_sz), C.POINTER(_sz), _i64p, C.POINTER(C.c_double)]
        L.ref_validate_config.argtypes = [_sz, _sz, _sz, _sz, C.c_int]
        L.ref_parse.argtypes = [C.c_int, C.c_char_p, _i64p, _sz, C.POINTER(_sz), C.POINTER(_sz),
                                C.POINTER(_sz)]

    def run_benchmark(self, path, orlib=False, nb=60, nt=256, evolve_limit=100, saturation=10, seed=1,
                      cx=-1, mu=-1, team=False, repeats=1, p_override=0, reference=-1, structured=True):
        """The reference CLI pipeline (run_benchmark + emit_report) -> (rc, report text)."""
        self.L.ref_run_benchmark.argtypes = [C.c_char_p, C.c_int, _sz, _sz, _sz, _sz, C.c_uint64,
                                             C.c_longlong, C.c_longlong, C.c_int, _sz, _sz,
                                             C.c_longlong, C.c_int, C.c_char_p, _sz]
        buf = C.create_string_buffer(1 << 16)
        rc = self.L.ref_run_benchmark(str(path).encode(), int(orlib), nb, nt, evolve_limit, saturation,
                                      seed, cx, mu, int(team), repeats, p_override, reference,
                                      int(structured), buf, len(buf))
        return rc, buf.value.decode()

    def report_roundtrip(self, text: str, structured: bool = True):
        """The reference's parse_structured_report + emit_report -> (rc, text, records)."""
        self.L.ref_report_roundtrip.argtypes = [C.c_char_p, C.c_int, C.c_char_p, _sz, C.POINTER(_sz)]
        buf = C.create_string_buffer(1 << 20)
        cnt = _sz(0)
        rc = self.L.ref_report_roundtrip(text.encode(), int(structured), buf, len(buf), C.byref(cnt))
        return rc, buf.value.decode(), cnt.value

    def parse(self, text: str, orlib: bool = True, cap: int = 1 << 22):
        """parse_orlib / parse_dense -> (rc, n, m, p, costs)"""
        out = np.zeros(cap, dtype=np.int64)
        n, m, p = _sz(0), _sz(0), _sz(0)
        rc = self.L.ref_parse(int(orlib), text.encode(), out, cap, C.byref(n), C.byref(m), C.byref(p))
        return rc, n.value, m.value, p.value, out[: n.value * m.value].copy()

    def last_error(self) -> str:
        return self.L.ref_last_error().decode()

    def create(self, n, m, p, costs, build_tables=True):
        return RefInstance(self, n, m, p, costs, build_tables)

    def create_with_tables(self, n, m, p, site_order, increments):
        return RefInstance(self, n, m, p, None, tables=(site_order, increments))


class RefInstance:
    def __init__(self, lib: RefLib, n, m, p, costs, build_tables=True, tables=None):
        self.lib, self.n, self.m, self.p = lib, n, m, p
        self.h = C.c_void_p()
        if tables is not None:
            so = np.ascontiguousarray(tables[0], dtype=np.uint32).reshape(-1)
            inc = np.ascontiguousarray(tables[1], dtype=np.int64).reshape(-1)
            self.rc = lib.L.ref_create_with_tables(n, m, p, so, inc, C.byref(self.h))
        else:
            self.rc = lib.L.ref_create(n, m, p, np.ascontiguousarray(costs, dtype=np.int64),
                                       int(build_tables), C.byref(self.h))
        if self.rc != 0:
            self.h = None

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_destroy(self.h)
            self.h = None

    @property
    def width(self):
        return self.lib.L.ref_width(self.h)

    def tables(self):
        W = self.width
        so = np.empty(self.n * W, dtype=np.uint32)
        inc = np.empty(self.n * W, dtype=np.int64)
        self.lib.L.ref_get_tables(self.h, so, inc)
        return so.reshape(self.n, W), inc.reshape(self.n, W)

    def evaluate(self, words, nthreads=1):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        count = words.shape[0] if words.ndim == 2 else 1
        costs = np.zeros(count, dtype=np.int64)
        fb = _sz(count)
        rc = self.lib.L.ref_evaluate(self.h, words.reshape(-1), words.shape[-1], count, costs,
                                     C.byref(fb), nthreads)
        return rc, costs, fb.value

    def fitness_bits(self, bits: str):
        out = C.c_int64(0)
        rc = self.lib.L.ref_fitness_bits(self.h, bits.encode(), C.byref(out))
        return rc, out.value

    def min_cost_sum(self, words):
        out = C.c_int64(0)
        rc = self.lib.L.ref_min_cost_sum(self.h, np.ascontiguousarray(words, dtype=np.uint64),
                                         C.byref(out))
        return rc, out.value

    def direct_cost(self, words):
        out = C.c_int64(0)
        rc = self.lib.L.ref_direct_cost(self.h, np.ascontiguousarray(words, dtype=np.uint64),
                                        C.byref(out))
        return rc, out.value

    def exact_optimum(self, budget=10_000_000):
        w = np.zeros(words_per(self.m), dtype=np.uint64)
        cost = C.c_int64(0)
        rc = self.lib.L.ref_exact_optimum(self.h, budget, w, C.byref(cost))
        return rc, w, cost.value

    def format_polynomial(self, reduced=True) -> str:
        buf = C.create_string_buffer(1 << 20)
        self.lib.L.ref_format_polynomial(self.h, int(reduced), buf, len(buf))
        return buf.value.decode()

    def evolve_block(self, block_words, nt, nb, seed, kernel_index, block_index,
                     crossover_iters=-1, mutation_iters=-1):
        bw = np.ascontiguousarray(block_words, dtype=np.uint64).copy()
        best = np.zeros(words_per(self.m), dtype=np.uint64)
        cost, thread = C.c_int64(0), _sz(0)
        rc = self.lib.L.ref_evolve_block(self.h, bw.reshape(-1), nt, nb, seed, crossover_iters,
                                         mutation_iters, kernel_index, block_index, best,
                                         C.byref(cost), C.byref(thread))
        return rc, bw.reshape(nt, -1), best, cost.value, thread.value

    def run_ga(self, nb, nt, evolve_limit, saturation, seed, crossover_iters=-1,
               mutation_iters=-1, team=False, workers=1):
        best = np.zeros(words_per(self.m), dtype=np.uint64)
        cost, ke, kb = C.c_int64(0), _sz(0), _sz(0)
        per = np.zeros(evolve_limit, dtype=np.int64)
        wall = C.c_double(0)
        rc = self.lib.L.ref_run_ga(self.h, nb, nt, evolve_limit, saturation, seed, crossover_iters,
                                   mutation_iters, int(team), workers, best, C.byref(cost),
                                   C.byref(ke), C.byref(kb), per, C.byref(wall))
        return rc, dict(best=best, best_cost=cost.value, kernels_executed=ke.value,
                        kernel_of_best=kb.value, per_kernel_best_costs=per[:ke.value].copy(),
                        wall_time=wall.value)
