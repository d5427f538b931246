/*
 * pmoracle.c -- CPU restatement of the reference's HBP fitness path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1610_10061_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * reference's own golden vectors (proj/tests/test_formulation.cpp:18-83,187-208,
 * proj/tests/test_instance.cpp:21-23) and, where /root/reference is present,
 * against oracle/_ref (the reference's unmodified sources compiled by
 * oracle/Makefile) on random instances.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pmoracle.h"

/* ---- RNG: include/pmedian/rng.hpp:11-51 (splitmix64) ------------------- */

uint64_t or_mix64(uint64_t z) { /* rng.hpp:11-15 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t or_rs_derive(uint64_t master, const uint64_t* key, size_t nkey) { /* rng.hpp:26-32 */
  uint64_t s = or_mix64(master ^ 0x6a09e667f3bcc909ULL);
  for (size_t i = 0; i < nkey; ++i) s = or_mix64(s ^ or_mix64(key[i] + 0x9e3779b97f4a7c15ULL));
  return s;
}

uint64_t or_rs_next(uint64_t* state) { /* rng.hpp:34-37 */
  *state += 0x9e3779b97f4a7c15ULL;
  return or_mix64(*state);
}

uint64_t or_rs_below(uint64_t* state, uint64_t bound) { /* rng.hpp:41-49 */
  if ((bound & (bound - 1)) == 0) return or_rs_next(state) & (bound - 1);
  const uint64_t threshold = (0 - bound) % bound;
  uint64_t v = or_rs_next(state);
  while (v < threshold) v = or_rs_next(state);
  return v % bound;
}

int or_rs_coin(uint64_t* state) { return (or_rs_next(state) & 1) != 0; } /* rng.hpp:51 */

/* ---- synthetic inputs (not reference code) ------------- */

static uint64_t isqrt_u64(uint64_t v) {
  uint64_t r = 0, bit = (uint64_t)1 << 62;
  while (bit > v) bit >>= 2;
  while (bit) {
    if (v >= r + bit) {
      v -= r + bit;
      r = (r >> 1) + bit;
    } else {
      r >>= 1;
    }
    bit >>= 2;
  }
  return r;
}

/* Euclidean instance: RandomStream(seed); x_i = below(10000), y_i = below(10000);
 * d_ij = floor(sqrt((x_i-x_j)^2 + (y_i-y_j)^2)).  n = m = npts. */
void or_synth_euclid(uint64_t seed, size_t npts, int64_t* costs) {
  uint64_t st = seed;
  int64_t* xs = (int64_t*)malloc(npts * sizeof(int64_t));
  int64_t* ys = (int64_t*)malloc(npts * sizeof(int64_t));
  for (size_t i = 0; i < npts; ++i) {
    xs[i] = (int64_t)or_rs_below(&st, 10000);
    ys[i] = (int64_t)or_rs_below(&st, 10000);
  }
  for (size_t i = 0; i < npts; ++i)
    for (size_t j = 0; j < npts; ++j) {
      const int64_t dx = xs[i] - xs[j], dy = ys[i] - ys[j];
      costs[i * npts + j] = (int64_t)isqrt_u64((uint64_t)(dx * dx + dy * dy));
    }
  free(xs);
  free(ys);
}

/* Uniform random costs as tests/test_support.hpp:22-30 (random_instance):
 * RandomStream(seed), every cell below(max_cost + 1). */
void or_random_costs(uint64_t seed, size_t n, size_t m, int64_t max_cost, int64_t* costs) {
  uint64_t st = seed;
  for (size_t i = 0; i < n * m; ++i) costs[i] = (int64_t)or_rs_below(&st, (uint64_t)max_cost + 1);
}

/* Uniform p-subsets: one RandomStream(seed) for the whole population; per
 * chromosome a partial Fisher-Yates of p draws (j + below(m - j)) over the
 * identity permutation.  words: count x ceil(m/64), bit j = word j>>6 bit j&63
 * (include/pmedian/chromosome.hpp:24). */
void or_random_population(uint64_t seed, size_t m, size_t p, size_t count, uint64_t* words) {
  const size_t wp = (m + 63) / 64;
  uint64_t st = seed;
  uint32_t* perm = (uint32_t*)malloc(m * sizeof(uint32_t));
  for (size_t j = 0; j < m; ++j) perm[j] = (uint32_t)j;
  size_t* swaps = (size_t*)malloc((p ? p : 1) * sizeof(size_t));
  memset(words, 0, count * wp * sizeof(uint64_t));
  for (size_t c = 0; c < count; ++c) {
    uint64_t* w = words + c * wp;
    for (size_t j = 0; j < p; ++j) {
      const size_t r = j + (size_t)or_rs_below(&st, m - j);
      swaps[j] = r;
      const uint32_t t = perm[j];
      perm[j] = perm[r];
      perm[r] = t;
      w[perm[j] >> 6] |= (uint64_t)1 << (perm[j] & 63);
    }
    for (size_t j = p; j-- > 0;) { /* undo: back to the identity */
      const size_t r = swaps[j];
      const uint32_t t = perm[j];
      perm[j] = perm[r];
      perm[r] = t;
    }
  }
  free(swaps);
  free(perm);
}

/* ---- Instance validation: src/instance.cpp:10-30 ----------------------- */

int or_validate_instance(size_t n, size_t m, size_t p, const int64_t* costs, size_t ncosts) {
  if (n == 0) return OR_STRUCTURAL;                 /* instance.cpp:13 */
  if (m == 0) return OR_STRUCTURAL;                 /* instance.cpp:14 */
  if (p < 1) return OR_DOMAIN;                      /* instance.cpp:15 */
  if (p >= m) return OR_DOMAIN;                     /* instance.cpp:16 */
  if (ncosts != n * m) return OR_STRUCTURAL;        /* instance.cpp:17-19 */
  int64_t mx = 0;
  for (size_t i = 0; i < ncosts; ++i) {
    if (costs[i] < 0) return OR_STRUCTURAL;         /* instance.cpp:22 */
    if (costs[i] > mx) mx = costs[i];
  }
  if (mx > 0 && mx > INT64_MAX / (int64_t)n) return OR_STRUCTURAL; /* instance.cpp:26-29 */
  return OR_OK;
}

/* ---- build_ordering: src/ordering.cpp:10-38 ---------------------------- */

static const int64_t* g_row; /* qsort has no context argument */
static int cmp_site(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  if (g_row[a] != g_row[b]) return g_row[a] < g_row[b] ? -1 : 1; /* ordering.cpp:26 */
  return a < b ? -1 : (a > b);                                  /* ordering.cpp:27 */
}

void or_build_ordering(size_t n, size_t m, size_t p, const int64_t* costs, uint32_t* site_order,
                       int64_t* increments) {
  const size_t width = m - p + 1; /* ordering.cpp:17 */
  uint32_t* order = (uint32_t*)malloc(m * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) {
    const int64_t* row = costs + i * m;
    for (size_t j = 0; j < m; ++j) order[j] = (uint32_t)j; /* ordering.cpp:24 */
    g_row = row;
    qsort(order, m, sizeof(uint32_t), cmp_site); /* ordering.cpp:25-28 */
    int64_t prev = 0;
    for (size_t k = 0; k < width; ++k) { /* ordering.cpp:29-35 */
      const uint32_t site = order[k];
      site_order[i * width + k] = site;
      increments[i * width + k] = row[site] - prev;
      prev = row[site];
    }
  }
  free(order);
}

/* ---- fitness: src/ordering.cpp:40-59 ----------------------------------- */

static int test_bit(const uint64_t* w, size_t j) { return (int)((w[j >> 6] >> (j & 63)) & 1); }

int or_fitness(size_t n, size_t width, const uint32_t* site_order, const int64_t* increments,
               const uint64_t* words, int64_t* out) {
  int64_t total = 0;
  for (size_t i = 0; i < n; ++i) { /* ordering.cpp:45 */
    const uint32_t* order = site_order + i * width;
    const int64_t* inc = increments + i * width;
    int64_t acc = 0;
    for (size_t k = 0;; ++k) {
      if (k == width) return OR_CONTRACT; /* ordering.cpp:50-52 */
      acc += inc[k];                      /* ordering.cpp:53 */
      if (test_bit(words, order[k])) break; /* ordering.cpp:54 */
    }
    total += acc; /* ordering.cpp:56 */
  }
  *out = total;
  return OR_OK;
}

/* Batch form: the loop a caller of fitness() runs (src/ga.cpp:147).  Stops at
 * the first failing chromosome, as a sequential loop of throwing calls would;
 * *first_bad receives its index.  Also reports sum_k = sum_i k*_i (1-based
 * stopping column) per chromosome, the quantity SURVEY.md 8(d)'s B_eval uses. */
int or_evaluate_population(size_t n, size_t m, size_t width, const uint32_t* site_order,
                           const int64_t* increments, const uint64_t* words, size_t words_per,
                           size_t count, int64_t* costs_out, uint64_t* sum_k_out,
                           size_t* first_bad) {
  if (words_per != (m + 63) / 64) return OR_STRUCTURAL; /* ordering.cpp:41-43 */
  for (size_t c = 0; c < count; ++c) {
    const uint64_t* w = words + c * words_per;
    if (sum_k_out) {
      uint64_t sk = 0;
      for (size_t i = 0; i < n; ++i) {
        size_t k = 0;
        while (k < width && !test_bit(w, site_order[i * width + k])) ++k;
        sk += (uint64_t)(k + 1);
      }
      sum_k_out[c] = sk;
    }
    const int rc = or_fitness(n, width, site_order, increments, w, &costs_out[c]);
    if (rc != OR_OK) {
      if (first_bad) *first_bad = c;
      return rc;
    }
  }
  return OR_OK;
}

/* ---- min_cost_sum / direct_cost: src/instance.cpp:32-58 ---------------- */

int or_min_cost_sum(size_t n, size_t m, const int64_t* costs, const uint64_t* words,
                    int64_t* out) {
  size_t* open = (size_t*)malloc((m ? m : 1) * sizeof(size_t)); /* instance.cpp:36 open_indices */
  size_t np = 0;
  for (size_t j = 0; j < m; ++j)
    if (test_bit(words, j)) open[np++] = j;
  if (np == 0) { /* instance.cpp:37 */
    free(open);
    return OR_CONTRACT;
  }
  int64_t total = 0;
  for (size_t i = 0; i < n; ++i) { /* instance.cpp:39-46 */
    const int64_t* row = costs + i * m;
    int64_t best = row[open[0]];
    for (size_t k = 1; k < np; ++k)
      if (row[open[k]] < best) best = row[open[k]];
    total += best;
  }
  free(open);
  *out = total;
  return OR_OK;
}

int or_direct_cost(size_t n, size_t m, size_t p, const int64_t* costs, const uint64_t* words,
                   int64_t* out) {
  size_t pc = 0; /* instance.cpp:54-56 */
  for (size_t j = 0; j < m; ++j) pc += (size_t)test_bit(words, j);
  if (pc != p) return OR_CONTRACT;
  return or_min_cost_sum(n, m, costs, words, out);
}

/* ---- parse_orlib closure: src/bench.cpp:121-166 -------------------------
 * uv: 2*edges 0-based endpoints, w: edge costs (already validated).  out: n*n.
 * Returns OR_STRUCTURAL and the first unreachable pair (row-major) in *bad. */
int or_orlib_closure(size_t n, size_t edges, const int64_t* uv, const int64_t* w, int64_t* out,
                     size_t* bad) {
  const int64_t kUnreachable = INT64_MAX / 4; /* bench.cpp:123 */
  for (size_t x = 0; x < n * n; ++x) out[x] = kUnreachable;
  for (size_t i = 0; i < n; ++i) out[i * n + i] = 0;
  for (size_t e = 0; e < edges; ++e) { /* bench.cpp:141-143: cheapest parallel edge */
    const size_t a = (size_t)uv[2 * e], b = (size_t)uv[2 * e + 1];
    if (w[e] < out[a * n + b]) out[a * n + b] = w[e];
    if (w[e] < out[b * n + a]) out[b * n + a] = w[e];
  }
  for (size_t k = 0; k < n; ++k) /* bench.cpp:146-157 */
    for (size_t i = 0; i < n; ++i) {
      const int64_t dik = out[i * n + k];
      if (dik == kUnreachable) continue;
      for (size_t j = 0; j < n; ++j) {
        const int64_t t = dik + out[k * n + j];
        if (t < out[i * n + j]) out[i * n + j] = t;
      }
    }
  for (size_t x = 0; x < n * n; ++x) /* bench.cpp:159-166 */
    if (out[x] >= kUnreachable) {
      if (bad) *bad = x;
      return OR_STRUCTURAL;
    }
  return OR_OK;
}
