"""Seeded synthetic inputs for the benchmark, vectorised.

Bit-identical to the reference's RandomStream (proj/include/pmedian/rng.hpp:22-55):
the k-th draw of a splitmix64 stream is mix64(seed + k * gamma), so whole
blocks of draws are computed at once; rejection in below() (rng.hpp:41-49)
only triggers for draws under 2^64 mod bound, which is detected and redrawn
sequentially so the result stays exact.  tests/test_synth.py checks equality
with the oracle's sequential restatement.

* ``euclid_points``/``euclid_costs``: RandomStream(seed); x_i = below(10000),
  y_i = below(10000); d_ij = isqrt((x_i-x_j)^2 + (y_i-y_j)^2), n = m = npts.
* ``random_population``: RandomStream(seed); per chromosome a partial
  Fisher-Yates of p draws (j + below(m - j)) over the identity permutation.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class Stream:
    """Vectorised RandomStream: draws(k) returns the next k raw outputs."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed)

    def draws(self, k: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(1, k + 1, dtype=np.uint64)
            st = self.state + idx * GAMMA
            self.state = self.state + np.uint64(k) * GAMMA
        return mix64(st)

    def next(self) -> int:
        return int(self.draws(1)[0])

    def below_scalar(self, bound: int) -> int:
        if bound & (bound - 1) == 0:
            return self.next() & (bound - 1)
        thr = (1 << 64) % bound
        v = self.next()
        while v < thr:
            v = self.next()
        return v % bound

    def below_many(self, bounds: np.ndarray) -> np.ndarray:
        """Sequential below(bounds[0]), below(bounds[1]), ... (exact, vectorised)."""
        bounds = np.asarray(bounds, dtype=np.uint64)
        out = np.empty(bounds.shape[0], dtype=np.uint64)
        pos = 0
        while pos < bounds.shape[0]:
            b = bounds[pos:]
            v = self.draws(b.shape[0])
            pow2 = (b & (b - np.uint64(1))) == 0
            thr = np.where(pow2, np.uint64(0), (np.uint64(0) - b) % b)
            bad = np.nonzero(v < thr)[0]
            stop = b.shape[0] if bad.size == 0 else int(bad[0])
            res = np.where(pow2, v & (b - np.uint64(1)), v % b)
            out[pos:pos + stop] = res[:stop]
            if stop == b.shape[0]:
                break
            # rejection at `stop`: rewind the stream to just after draw `stop`, redo sequentially
            with np.errstate(over="ignore"):
                self.state = self.state - np.uint64(b.shape[0] - stop - 1) * GAMMA
            out[pos + stop] = self._finish_rejection(int(b[stop]))
            pos += stop + 1
        return out

    def _finish_rejection(self, bound: int) -> int:
        thr = (1 << 64) % bound
        v = self.next()
        while v < thr:
            v = self.next()
        return v % bound


def euclid_points(npts: int, seed: int = 12345):
    s = Stream(seed)
    xy = s.below_many(np.full(2 * npts, 10000, dtype=np.uint64)).astype(np.int64)
    return xy[0::2], xy[1::2]


def isqrt_exact(v):
    """floor(sqrt(v)) for int64 arrays (numpy or torch), exact."""
    try:
        import torch
        if isinstance(v, torch.Tensor):
            r = torch.sqrt(v.to(torch.float64)).to(torch.int64)
            r = r - (r * r > v).to(torch.int64)
            r = r + ((r + 1) * (r + 1) <= v).to(torch.int64)
            return r
    except ImportError:
        pass
    r = np.sqrt(v.astype(np.float64)).astype(np.int64)
    r -= (r * r > v)
    r += ((r + 1) * (r + 1) <= v)
    return r


def euclid_costs(npts: int, seed: int = 12345, device=None):
    """n x m int64 cost matrix (row-major).  device=None -> numpy; else a torch
    device on which the matrix is computed directly (no host copy)."""
    x, y = euclid_points(npts, seed)
    if device is None:
        out = np.empty((npts, npts), dtype=np.int64)
        step = max(1, (1 << 24) // npts)
        for i0 in range(0, npts, step):
            dx = x[i0:i0 + step, None] - x[None, :]
            dy = y[i0:i0 + step, None] - y[None, :]
            out[i0:i0 + step] = isqrt_exact(dx * dx + dy * dy)
        return out.reshape(-1)
    import torch
    tx = torch.from_numpy(x).to(device)
    ty = torch.from_numpy(y).to(device)
    out = torch.empty((npts, npts), dtype=torch.int64, device=device)
    step = max(1, (1 << 26) // npts)
    for i0 in range(0, npts, step):
        dx = tx[i0:i0 + step, None] - tx[None, :]
        dy = ty[i0:i0 + step, None] - ty[None, :]
        out[i0:i0 + step] = isqrt_exact(dx * dx + dy * dy)
    return out.reshape(-1)


def random_population(m: int, p: int, count: int, seed: int = 7) -> np.ndarray:
    """count x ceil(m/64) uint64 words, each row a uniform p-subset."""
    wp = (m + 63) // 64
    s = Stream(seed)
    bounds = np.tile(np.arange(m, m - p, -1, dtype=np.uint64), count)
    r = s.below_many(bounds).reshape(count, p).astype(np.int64) + np.arange(p, dtype=np.int64)
    words = np.zeros((count, wp), dtype=np.uint64)
    for c in range(count):
        perm = {}
        rc = r[c]
        for j in range(p):
            t = int(rc[j])
            pj = perm.get(j, j)
            pt = perm.get(t, t)
            perm[j], perm[t] = pt, pj
        sites = np.fromiter((perm.get(j, j) for j in range(p)), dtype=np.int64, count=p)
        np.bitwise_or.at(words[c], sites >> 6, np.left_shift(np.uint64(1), (sites & 63).astype(np.uint64)))
    return words


def _subsets(m: int, k: int):
    """All k-subsets of range(m) as (words [N, wp] u64, min, max); k small."""
    import itertools
    wp = (m + 63) // 64
    comb = np.array(list(itertools.combinations(range(m), k)), dtype=np.int64).reshape(-1, k)
    words = np.zeros((comb.shape[0], wp), dtype=np.uint64)
    for c in range(k):
        np.bitwise_or.at(words, (np.arange(comb.shape[0]), comb[:, c] >> 6),
                         np.left_shift(np.uint64(1), (comb[:, c] & 63).astype(np.uint64)))
    lo = comb[:, 0] if k else np.full(1, m, dtype=np.int64)
    hi = comb[:, -1] if k else np.full(1, -1, dtype=np.int64)
    return words, lo, hi


def all_subsets(m: int, p: int, chunk: int = 1 << 22):
    """Every p-subset of range(m) exactly once, as chunks of chromosome words
    (exhaustive optima for small instances, e.g. the pmed1 shape C(100, 5)).
    A p-subset = a (p//2)-subset followed by a (p - p//2)-subset whose
    minimum exceeds the first part's maximum."""
    a_words, _, a_hi = _subsets(m, p // 2)
    b_words, b_lo, _ = _subsets(m, p - p // 2)
    order = np.argsort(b_lo, kind="stable")
    b_words, b_lo = b_words[order], b_lo[order]
    buf, size = [], 0
    for i in range(a_words.shape[0]):
        j = int(np.searchsorted(b_lo, a_hi[i] + 1))
        if j == b_words.shape[0]:
            continue
        part = b_words[j:] | a_words[i]
        buf.append(part)
        size += part.shape[0]
        if size >= chunk:
            yield np.concatenate(buf)
            buf, size = [], 0
    if buf:
        yield np.concatenate(buf)
