// K3: the GA's evolve_block on the device, batched over every block, plus the
// run_ga generation loop (K4 islands: blocks sharded over processes/GPUs,
// one allgather of block bests per generation).
//
// Reference semantics (proj/src/ga.cpp) reproduced exactly:
//  * evolve_block (:136-194): fitness of the block; `rounds` crossover rounds
//    over the snapshot `before`, couples t ^ (nt >> (round % lg nt + 1)),
//    both partners drawing (start, exchanges) from derive(seed, {2, kernel,
//    block, round, min(t, couple)}); strict-improvement replacement; then
//    `attempts` shift mutations per thread from derive(seed, {3, kernel, block,
//    t}) stopping at the first strict improvement; min-reduce, ties to the
//    lower thread.
//  * run_ga (:219-303): per generation evolve all blocks, draw the next
//    population, global best by strict < (lowest block wins ties), stale
//    counter, stop rule, migration only when continuing.
// The mutation attempts of a thread all mutate the same parent (the parent
// only changes on success, and success ends the attempts), and the RNG stream
// advances identically whether or not an attempt succeeds -- so all attempts
// are generated and evaluated as one batch and the first improving one is
// taken.  This evaluates attempts the reference would skip; they are counted
// separately (device_evaluations) and never reported as reference work.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "combinatorics.h"
#include "ctx.h"
#include "common.cuh"
#include "ga_ops.cuh"

namespace pmb {

// ---- kernels ----------------------------------------------------------------------

__global__ void k_crossover_children(const uint64_t* __restrict__ before, uint64_t* __restrict__ child,
                                     uint8_t* __restrict__ ok, int nbl, int nt, int wp, int m, int p,
                                     uint64_t seed, uint64_t kernel, uint64_t block0, uint64_t round,
                                     int cycle) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nbl * nt) return;
  const int b = idx / nt, t = idx % nt;
  const uint32_t couple = crossover_couple((uint32_t)t, (uint32_t)(round % cycle), (uint32_t)nt);
  const uint64_t key[5] = {kCoupleTag, kernel, block0 + b, round, (uint64_t)min((uint32_t)t, couple)};
  Stream rng = Stream::derive(seed, key, 5);
  const int start = (int)rng.below((uint64_t)m);
  const int exchanges = 2 * (1 + (int)rng.below((uint64_t)(p / 2)));
  PMB_CHECK(couple < (uint32_t)nt && start >= 0 && start < m && exchanges <= p);
  const uint64_t* a = before + (size_t)idx * wp;
  const uint64_t* bb = before + ((size_t)b * nt + couple) * wp;
  uint64_t* c = child + (size_t)idx * wp;
  const bool success = crossover(a, bb, c, m, start, exchanges);
  if (!success)  // keep the parent (ga.cpp:165)
    for (int w = 0; w < wp; ++w) c[w] = a[w];
  ok[idx] = success;
}

// Accept into the other population buffer: nxt = child where it improved,
// else the parent (ga.cpp:165-167), so the next round reads nxt as its
// snapshot `before` and no copy of the population is needed between rounds.
__global__ void k_crossover_accept_pp(const uint64_t* __restrict__ cur, uint64_t* __restrict__ nxt,
                                      int64_t* __restrict__ cost, const uint64_t* __restrict__ child,
                                      const int64_t* __restrict__ ccost, const uint8_t* __restrict__ ok, int count,
                                      int wp, unsigned long long* __restrict__ evals) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned e = 0;
  if (idx < count) {
    const bool success = ok[idx];
    e = success;  // the reference evaluates every successful child (ga.cpp:166)
    const bool take = success && ccost[idx] < cost[idx];
    const uint64_t* src = (take ? child : cur) + (size_t)idx * wp;
    for (int w = 0; w < wp; ++w) nxt[(size_t)idx * wp + w] = src[w];
    if (take) cost[idx] = ccost[idx];
  }
  e = __reduce_add_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0 && e) atomicAdd(evals, (unsigned long long)e);
}

__global__ void k_mutation_children(const uint64_t* __restrict__ pop, uint64_t* __restrict__ child,
                                    int nbl, int nt, int wp, int m, uint64_t seed, uint64_t kernel,
                                    uint64_t block0, int attempts) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nbl * nt) return;
  const int b = idx / nt, t = idx % nt;
  const uint64_t key[4] = {kMutationTag, kernel, block0 + b, (uint64_t)t};
  Stream rng = Stream::derive(seed, key, 4);
  const uint64_t* parent = pop + (size_t)idx * wp;
  for (int a = 0; a < attempts; ++a)
    random_shift_mutation(parent, child + ((size_t)idx * attempts + a) * wp, m, rng);
}

// 32 chromosomes per 256-thread block: warp 0 draws every attempt's shift
// (one keyed stream per chromosome, consumed in the reference's order), then
// the whole block builds the children word by word -- attempts x words
// independent outputs per chromosome, written coalesced.  (One thread per
// chromosome left the kernel latency-bound: 15,360 threads at the paper's
// shape is ~3 warps per SM.)
__global__ void __launch_bounds__(256) k_mutation_children_wide(const uint64_t* __restrict__ pop,
                                                                uint64_t* __restrict__ child, int nbl, int nt,
                                                                int wp, int m, uint64_t seed, uint64_t kernel,
                                                                uint64_t block0, int attempts) {
  extern __shared__ ShiftDraw sd[];  // [32][attempts]
  __shared__ int redo[32];           // a rejection shifted the stream: redraw sequentially
  const int count = nbl * nt;
  const int c0 = blockIdx.x * 32;
  if (threadIdx.x < 32) redo[threadIdx.x] = 0;
  __syncthreads();
  // Every (chromosome, attempt) draws in parallel.  An attempt consumes 2 coins
  // plus 1 (whole rotation) or 3 (sub-range) bounded draws, one output each
  // unless a draw rejects (probability < 2^-47 per draw at these bounds), so a
  // task finds its attempt's stream position from the earlier attempts' first
  // coins alone; a task whose own draw rejected flags its chromosome, which
  // is then redrawn sequentially -- exact in every case.
  constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
  for (int task = threadIdx.x; task < 32 * attempts; task += blockDim.x) {
    const int cl = task / attempts, a = task - cl * attempts;
    const int idx = c0 + cl;
    if (idx >= count) continue;
    const int b = idx / nt, t = idx % nt;
    const uint64_t key[4] = {kMutationTag, kernel, block0 + b, (uint64_t)t};
    Stream rng = Stream::derive(seed, key, 4);
    for (int q = 0; q < a; ++q) {
      const bool whole = rng.coin();
      rng.state += (whole ? 2 : 4) * kGamma;  // direction coin + 1 or 3 draws
    }
    const uint64_t before = rng.state;
    const bool whole = (mix64(before + kGamma) & 1) != 0;  // this attempt's first coin
    sd[cl * attempts + a] = draw_shift(m, rng);
    if (rng.state != before + (whole ? 3 : 5) * kGamma) redo[cl] = 1;  // a draw rejected
  }
  __syncthreads();
  if (threadIdx.x < 32 && redo[threadIdx.x]) {
    const int idx = c0 + threadIdx.x;
    const int b = idx / nt, t = idx % nt;
    const uint64_t key[4] = {kMutationTag, kernel, block0 + b, (uint64_t)t};
    Stream rng = Stream::derive(seed, key, 4);
    for (int a = 0; a < attempts; ++a) sd[threadIdx.x * attempts + a] = draw_shift(m, rng);
  }
  __syncthreads();
  const int nc = min(32, count - c0);
  const int per = attempts * wp;
  const int total = nc * per;
  const uint64_t* base = pop + (size_t)c0 * wp;
  uint64_t* out = child + (size_t)c0 * per;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int cl = e / per, r = e - cl * per;
    const int a = r / wp, wi = r - a * wp;
    const ShiftDraw d = sd[cl * attempts + a];
    out[e] = rotate_word(base + (size_t)cl * wp, d.lo, d.len, d.offset, wi);
  }
}

__global__ void k_mutation_accept(uint64_t* __restrict__ pop, int64_t* __restrict__ cost,
                                  const uint64_t* __restrict__ child, const int64_t* __restrict__ ccost,
                                  int count, int attempts, int wp, unsigned long long* __restrict__ evals) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned e = 0;
  if (idx < count) {
    e = attempts;
    for (int a = 0; a < attempts; ++a) {
      const size_t ci = (size_t)idx * attempts + a;
      if (ccost[ci] < cost[idx]) {  // first strict improvement wins (ga.cpp:184-187)
        for (int w = 0; w < wp; ++w) pop[(size_t)idx * wp + w] = child[ci * wp + w];
        cost[idx] = ccost[ci];
        e = a + 1;
        break;
      }
    }
  }
  e = __reduce_add_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0 && e) atomicAdd(evals, (unsigned long long)e);
}

// block_min_reduce (ga.cpp:113-134): lexicographic (cost, thread) minimum.
// Writes block b's record {cost, thread, words[wp]} at rec + b * (2 + wp): the
// layout the islands exchange, copied to the host in one transfer.
__global__ void k_block_min(const int64_t* __restrict__ cost, const uint64_t* __restrict__ pop, int nt,
                            int wp, uint64_t* __restrict__ rec) {
  __shared__ int64_t sc[32];
  __shared__ int st[32];
  const int b = blockIdx.x;
  int64_t best = INT64_MAX;
  int bt = INT32_MAX;
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    const int64_t c = cost[(size_t)b * nt + t];
    if (c < best || (c == best && t < bt)) {
      best = c;
      bt = t;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t c = __shfl_xor_sync(0xffffffffu, best, o);
    const int t = __shfl_xor_sync(0xffffffffu, bt, o);
    if (c < best || (c == best && t < bt)) {
      best = c;
      bt = t;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sc[warp] = best;
    st[warp] = bt;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sc[lane] : INT64_MAX;
    bt = lane < nw ? st[lane] : INT32_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t c = __shfl_xor_sync(0xffffffffu, best, o);
      const int t = __shfl_xor_sync(0xffffffffu, bt, o);
      if (c < best || (c == best && t < bt)) {
        best = c;
        bt = t;
      }
    }
    if (lane == 0) {
      sc[0] = best;
      st[0] = bt;
      rec[(size_t)b * (2 + wp)] = (uint64_t)best;
      rec[(size_t)b * (2 + wp) + 1] = (uint64_t)bt;
    }
  }
  __syncthreads();
  const int t = st[0];
  for (int w = threadIdx.x; w < wp; w += blockDim.x)
    rec[(size_t)b * (2 + wp) + 2 + w] = pop[((size_t)b * nt + t) * wp + w];
}

// run_ga's per-generation step (ga.cpp:279-297) on the device, after the
// island exchange: every rank runs it on the same gathered records grec
// (nb x {cost, thread, words[wp]}) and so reaches the same decision.
//  * global best: strict <, lowest block wins ties (ga.cpp:279-282);
//  * per-kernel best, best-so-far, kernel_of_best (1-based), stale counter,
//    stop when stale >= saturation or kernel + 1 >= evolve_limit (:285-296);
//  * migration only when continuing (:293-297) into the freshly drawn next
//    population: block b's best to slot 0 of block b, or (team) every block's
//    best to slots 0..nb-1 of block 0 (:204-215) -- local blocks only.
// gstate: [0] best cost, [1] kernel_of_best, [2] stale, [3] kernels executed,
// [4] stop, [5] reference-semantics evaluations at the stop, [8..8+wp) best words.
constexpr int kStateWords = 8;
__global__ void __launch_bounds__(256) k_generation_step(const uint64_t* __restrict__ grec, int nb, int wp,
                                                         uint64_t kernel, uint64_t saturation, uint64_t limit,
                                                         uint64_t* __restrict__ gstate, int64_t* __restrict__ perk,
                                                         uint64_t* __restrict__ next, int nt, int team, int block0,
                                                         int nbl, const unsigned long long* __restrict__ evals) {
  __shared__ int64_t sc[8];
  __shared__ int sb[8];
  __shared__ int s_best, s_improved, s_stop;
  const size_t rec = 2 + (size_t)wp;
  int64_t best = INT64_MAX;
  int bb = INT32_MAX;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int64_t c = (int64_t)grec[(size_t)b * rec];
    if (c < best || (c == best && b < bb)) {
      best = c;
      bb = b;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t c = __shfl_xor_sync(0xffffffffu, best, o);
    const int b = __shfl_xor_sync(0xffffffffu, bb, o);
    if (c < best || (c == best && b < bb)) {
      best = c;
      bb = b;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sc[warp] = best;
    sb[warp] = bb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sc[w] < best || (sc[w] == best && sb[w] < bb)) {
        best = sc[w];
        bb = sb[w];
      }
    perk[kernel] = best;
    const bool improved = best < (int64_t)gstate[0];
    if (improved) {
      gstate[0] = (uint64_t)best;
      gstate[1] = kernel + 1;
      gstate[2] = 0;
    } else {
      gstate[2] += 1;
    }
    const bool stop = gstate[2] >= saturation || kernel + 1 >= limit;
    gstate[3] = kernel + 1;
    gstate[4] = stop;
    gstate[5] = *evals;
    s_best = bb;
    s_improved = improved;
    s_stop = stop;
  }
  __syncthreads();
  const int b = s_best;
  if (s_improved)
    for (int w = threadIdx.x; w < wp; w += blockDim.x) gstate[kStateWords + w] = grec[(size_t)b * rec + 2 + w];
  if (s_stop) return;
  if (!team) {
    for (int x = threadIdx.x; x < nbl * wp; x += blockDim.x) {
      const int lb = x / wp, w = x - lb * wp;
      next[(size_t)lb * nt * wp + w] = grec[(size_t)(block0 + lb) * rec + 2 + w];
    }
  } else if (block0 == 0) {
    for (int x = threadIdx.x; x < nb * wp; x += blockDim.x) {
      const int gb = x / wp, w = x - gb * wp;
      next[(size_t)gb * wp + w] = grec[(size_t)gb * rec + 2 + w];
    }
  }
}

// Device-native population draw: uniform p-subsets by Floyd's algorithm from a
// keyed splitmix stream derive(seed, {4, generation, global chromosome}).
// (Not the reference's BigInt unranking -- see population mode in pmedian_b200.h.)
__global__ void k_draw_population(uint64_t* __restrict__ pop, int count, int wp, int m, int p,
                                  uint64_t seed, uint64_t generation, uint64_t index0) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  uint64_t* w = pop + (size_t)idx * wp;
  for (int i = 0; i < wp; ++i) w[i] = 0;
  const uint64_t key[3] = {4, generation, index0 + idx};
  Stream rng = Stream::derive(seed, key, 3);
  for (int j = m - p; j < m; ++j) {
    const int r = (int)rng.below((uint64_t)j + 1);
    const uint64_t bit = 1ull << (r & 63);
    if (w[r >> 6] & bit) w[j >> 6] |= 1ull << (j & 63);
    else w[r >> 6] |= bit;
  }
}

__global__ void k_popcount_check(const uint64_t* __restrict__ pop, int count, int wp, int m, int p,
                                 unsigned long long* __restrict__ bad) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  int pc = 0;
  for (int w = 0; w < wp; ++w) {
    uint64_t x = pop[(size_t)idx * wp + w];
    if (w == wp - 1 && (m & 63)) x &= (1ull << (m & 63)) - 1;
    pc += __popcll(x);
  }
  if (pc != p) atomicMin(bad, (unsigned long long)idx);
}

// Reference-exact unranking on the device (combinatorics.cpp:20-52): the
// rank-th p-subset of {0..m-1} in lexicographic order.  The reference walks
// the candidates one by one (take candidate when C(a, k) > r, else
// r -= C(a, k)); a run of skips telescopes (hockey stick:
// sum_{t<j} C(a-t, k) = C(a+1, k+1) - C(a-j+1, k+1)), so with X = C(a+1, k+1) - r
// the next taken candidate is the first j with C(a-j, k+1) < X, after which
// X -= C(a-j, k+1), a -= j+1, k -= 1.  One warp per chromosome tests 32
// consecutive candidates per probe (one contiguous table run), so a draw costs
// ~p dependent probes instead of ~m.  The table is limb-major ([y][limb][x]),
// so each limb load of a probe is one contiguous 256-byte run.  Same subsets as the reference's walk,
// bit for bit (tests/test_gpu_ga.py).
// One probe of S consecutive candidates per chromosome with kN-limb
// arithmetic (X and the probed binomials fit in kN limbs at this step).  The
// warp holds 32/S chromosomes, one S-lane group each; every lane of the warp
// runs the probe (`live` false for a finished group), so the warp stays
// converged.  On a hit the group's X -= C(a-j, k+1) and `jl` is the lane (in
// the group) of the taken candidate.
template <int kN, int kL, int S>
__device__ __forceinline__ bool unrank_probe(const uint64_t* __restrict__ table, int m, int L, int k, int x,
                                             bool live, int gbase, uint64_t (&X)[kL], int& jl) {
  uint64_t cv[kN];
  int cmp = 1;  // sign of C(x, k+1) - X; C(x, .) = 0 for x < 0
  if (live) {
    cmp = -1;
    if (x >= 0) {
      const uint64_t* cp = table + (size_t)(k + 1) * L * m + x;  // limb i at cp[i * m]
#pragma unroll
      for (int i = 0; i < kN; ++i) cv[i] = i < L ? __ldg(cp + (size_t)i * m) : 0;  // bucket may exceed L
      cmp = 0;
#pragma unroll
      for (int i = kN - 1; i >= 0; --i)
        if (cmp == 0) cmp = cv[i] < X[i] ? -1 : (cv[i] > X[i] ? 1 : 0);
    } else {
#pragma unroll
      for (int i = 0; i < kN; ++i) cv[i] = 0;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kN; ++i) cv[i] = 0;
  }
  const unsigned bal = __ballot_sync(kFull, cmp < 0);
  const unsigned hit = S == 32 ? bal : (bal >> gbase) & ((1u << S) - 1);
  jl = hit ? __ffs(hit) - 1 : 0;
  const bool take = live && hit != 0;
  uint64_t borrow = 0;
#pragma unroll
  for (int i = 0; i < kN; ++i) {
    const uint64_t v = __shfl_sync(kFull, cv[i], gbase + jl);
    const uint64_t d = X[i] - v - borrow;
    const uint64_t nb = (X[i] < v) || (X[i] - v < borrow);
    if (take) {
      X[i] = d;
      borrow = nb;
    }
  }
  return take;
}

// Dispatch on the step's limb count (warp-uniform: the largest over the
// warp's groups): the smallest instantiated width that holds it.
template <int kL, int S>
__device__ __forceinline__ bool unrank_probe_n(int lim, const uint64_t* __restrict__ table, int m, int L, int k,
                                               int x, bool live, int gbase, uint64_t (&X)[kL], int& jl) {
  if (lim <= 1) return unrank_probe<1, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  if (lim <= 2) return unrank_probe<2, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  if constexpr (kL >= 4) {
    if (lim <= 3) return unrank_probe<3, kL, S>(table, m, L, k, x, live, gbase, X, jl);
    if (lim <= 4) return unrank_probe<4, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  }
  if constexpr (kL >= 8) {
    if (lim <= 6) return unrank_probe<6, kL, S>(table, m, L, k, x, live, gbase, X, jl);
    if (lim <= 8) return unrank_probe<8, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  }
  if constexpr (kL >= 16) {
    if (lim <= 12) return unrank_probe<12, kL, S>(table, m, L, k, x, live, gbase, X, jl);
    if (lim <= 16) return unrank_probe<16, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  }
  if constexpr (kL >= 32) {
    if (lim <= 24) return unrank_probe<24, kL, S>(table, m, L, k, x, live, gbase, X, jl);
  }
  return unrank_probe<kL, kL, S>(table, m, L, k, x, live, gbase, X, jl);
}

// Reference-exact unranking on the device (combinatorics.cpp:20-52): the
// rank-th p-subset of {0..m-1} in lexicographic order.  The reference walks
// the candidates one by one (take candidate when C(a, k) > r, else
// r -= C(a, k)); a run of skips telescopes (hockey stick:
// sum_{t<j} C(a-t, k) = C(a+1, k+1) - C(a-j+1, k+1)), so with X = C(a+1, k+1) - r
// the next taken candidate is the first j with C(a-j, k+1) < X, after which
// X -= C(a-j, k+1), a -= j+1, k -= 1.  A group of S lanes per chromosome tests
// S consecutive candidates per probe (one contiguous table run per limb), so
// a draw costs ~p * E[probes per gap] dependent probes instead of ~m, each
// with only the limbs the step's values need (X < C(m, k+1) shrinks as k
// falls).  S is picked from the gap density p/m (pick_unrank_group): 32 lanes
// on one chromosome waste most of a probe when the mean gap m/p is ~10.
// Same subsets as the reference's walk, bit for bit (tests/test_gpu_ga.py).
template <int kL, int S>
__global__ void __launch_bounds__(256) k_unrank(const uint64_t* __restrict__ ranks,
                                                const uint64_t* __restrict__ table, int m, int p, int L, int wp,
                                                int count, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int gbase = S == 32 ? 0 : lane / S * S, gl = lane - gbase;
  const int idx = (int)(((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5) * (32 / S) + lane / S);
  const bool active = idx < count;
  if (__ballot_sync(kFull, active) == 0) return;  // warp-uniform
  const uint64_t* bound = table + (size_t)(p + 1) * L * m;
  const uint64_t* lims = bound + L;  // limbs of C(m, k + 1), k < p
  uint64_t X[kL];  // X = C(m, p) - r (every lane of the group holds the same value)
  {
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      if (active && i < L) {
        const uint64_t b = __ldg(bound + i), r = __ldg(ranks + (size_t)idx * L + i);
        X[i] = b - r - borrow;
        borrow = (b < r) || (b - r < borrow);
      } else {
        X[i] = 0;
      }
    }
  }
  uint64_t* w = out + (size_t)idx * wp;
  if (active)
    for (int i = gl; i < wp; i += S) w[i] = 0;
  __syncwarp();
  int a = m - 1, k = active ? p - 1 : -1, base = 0;
  int word_idx = 0;
  uint64_t word = 0;  // the output word being filled (candidates increase)
  int lim = k >= 0 ? (int)__ldg(lims + k) : 0;
  while (true) {
    const bool live = k >= 0;
    if (__ballot_sync(kFull, live) == 0) break;
    const int limw = __reduce_max_sync(kFull, live ? lim : 0);
    int jl;
    const bool take = unrank_probe_n<kL, S>(limw, table, m, L, k, a - base - gl, live, gbase, X, jl);
    if (live) {
      if (!take) {
        base += S;
      } else {
        const int j = base + jl;
        const int cand = m - 1 - a + j;
        if ((cand >> 6) != word_idx) {
          if (gl == 0 && word) w[word_idx] = word;
          word_idx = cand >> 6;
          word = 0;
        }
        word |= 1ull << (cand & 63);
        a -= j + 1;
        --k;
        base = 0;
        if (k >= 0) lim = (int)__ldg(lims + k);
      }
    }
  }
  if (active && gl == 0 && word) w[word_idx] = word;
}

// Reference-exact unranking, one thread per chromosome, guided by logarithms:
// the next taken candidate is the smallest j with C(a-j, k+1) < X, and
// ln C(x, y) = ln x! - ln y! - ln (x-y)! is monotone in j, so a binary search
// over a table of ln x! (doubles) lands on j or next to it; two exact
// multi-limb comparisons against the Pascal table (C(a-j, k+1) < X and, for
// j > 0, C(a-j+1, k+1) >= X) confirm it or step it by one.  The doubles only
// guide; every decision is exact, so the subsets are the reference's bit for
// bit.  ~p exact probes of one entry each instead of ~p * E[gap]/S probes of S
// entries: far less work than the lane-group probe (k_unrank).
template <int kL>
__device__ __forceinline__ void load_entry(const uint64_t* __restrict__ table, int m, int L, int y, int x, int lim,
                                           uint64_t (&cv)[kL]) {
  // C(x, y) as kL limbs (the top ones beyond this step's lim are zero); 0 for x < y
  const uint64_t* cp = table + (size_t)y * L * m + (x < y ? 0 : x);
#pragma unroll
  for (int i = 0; i < kL; ++i) cv[i] = (i < lim && x >= y) ? __ldg(cp + (size_t)i * m) : 0;
}

template <int kL>
__device__ __forceinline__ int cmp_limbs(const uint64_t (&cv)[kL], const uint64_t (&X)[kL]) {
  int cmp = 0;  // sign of cv - X
#pragma unroll
  for (int i = kL - 1; i >= 0; --i)
    if (cmp == 0) cmp = cv[i] < X[i] ? -1 : (cv[i] > X[i] ? 1 : 0);
  return cmp;
}

// Reference-exact unranking, one thread per chromosome, guided by logarithms:
// the next taken candidate is the smallest j with C(a-j, k+1) < X, and
// ln C(x, y) = ln x! - ln y! - ln (x-y)! is monotone in j, so a binary search
// over a table of ln x! (doubles, in shared memory) lands on j or next to it;
// exact multi-limb comparisons against the Pascal table (C(a-j, k+1) < X and,
// for j > 0, C(a-j+1, k+1) >= X; both entries loaded together) confirm it or
// step it by one.  The doubles only guide; every decision is exact, so the
// subsets are the reference's bit for bit.  One L2 round trip per taken
// element instead of ~E[gap]/S probes of S entries (k_unrank).
template <int kL>
__global__ void __launch_bounds__(128) k_unrank_log(const uint64_t* __restrict__ ranks,
                                                    const uint64_t* __restrict__ table,
                                                    const double* __restrict__ lf_g, int m, int p, int L, int wp,
                                                    int count, uint64_t* __restrict__ out) {
  extern __shared__ double lf_s[];  // m + 2 entries when they fit (see launch), else unused
  const bool in_smem = lf_s != nullptr && (size_t)(m + 2) * 8 <= 48 * 1024;
  if (in_smem)
    for (int x = threadIdx.x; x < m + 2; x += blockDim.x) lf_s[x] = lf_g[x];
  __syncthreads();
  const double* lf = in_smem ? lf_s : lf_g;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const uint64_t* bound = table + (size_t)(p + 1) * L * m;
  const uint64_t* lims = bound + L;  // limbs of C(m, k + 1), k < p
  uint64_t X[kL];                    // X = C(m, p) - r
  {
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      if (i < L) {
        const uint64_t b = __ldg(bound + i), r = __ldg(ranks + (size_t)idx * L + i);
        X[i] = b - r - borrow;
        borrow = (b < r) || (b - r < borrow);
      } else {
        X[i] = 0;
      }
    }
  }
  uint64_t* w = out + (size_t)idx * wp;
  for (int i = 0; i < wp; ++i) w[i] = 0;
  int a = m - 1, k = p - 1;
  int word_idx = 0;
  uint64_t word = 0;
  uint64_t cv[kL], cw[kL];
  while (k >= 0) {
    const int lim = (int)__ldg(lims + k);
    // ln X from its top two limbs
    double lX = 0.0;
    {
      bool found = false;
#pragma unroll
      for (int i = kL - 1; i >= 0; --i) {
        if (!found && X[i] != 0) {
          found = true;
          const double lo = i > 0 ? (double)X[i - 1] * 5.421010862427522e-20 : 0.0;  // 2^-64
          lX = log((double)X[i] + lo) + (double)i * 44.3614195558365;              // 64 ln 2
        }
      }
    }
    // smallest j in [0, a-k] with ln C(a-j, k+1) < ln X (C(k, k+1) = 0 at j = a-k)
    const double lk = lf[k + 1];
    int lo = 0, hi = a - k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1, x = a - mid;
      const double lc = lf[x] - lk - lf[x - k - 1];
      if (lc < lX) hi = mid;
      else lo = mid + 1;
    }
    int j = lo;
    // exact confirmation (both entries in flight together), stepping by one
    // when the estimate is off
    load_entry<kL>(table, m, L, k + 1, a - j, lim, cv);
    if (j > 0) load_entry<kL>(table, m, L, k + 1, a - j + 1, lim, cw);
    while (true) {
      if (cmp_limbs<kL>(cv, X) >= 0) {  // C(a-j, k+1) >= X: the taken one is further
        ++j;
#pragma unroll
        for (int i = 0; i < kL; ++i) cw[i] = cv[i];
        load_entry<kL>(table, m, L, k + 1, a - j, lim, cv);
        continue;
      }
      if (j > 0 && cmp_limbs<kL>(cw, X) < 0) {  // C(a-j+1, k+1) < X too: it is earlier
        --j;
#pragma unroll
        for (int i = 0; i < kL; ++i) cv[i] = cw[i];
        if (j > 0) load_entry<kL>(table, m, L, k + 1, a - j + 1, lim, cw);
        continue;
      }
      break;
    }
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      const uint64_t d = X[i] - cv[i] - borrow;
      borrow = (X[i] < cv[i]) || (X[i] - cv[i] < borrow);
      X[i] = d;
    }
    const int cand = m - 1 - a + j;
    if ((cand >> 6) != word_idx) {
      if (word) w[word_idx] = word;
      word_idx = cand >> 6;
      word = 0;
    }
    word |= 1ull << (cand & 63);
    a -= j + 1;
    --k;
  }
  if (word) w[word_idx] = word;
}

// Lanes per chromosome for k_unrank: the width S minimising the expected warp
// work per draw, (S/32) * E[probes per gap] = (S/32) / (1 - (1 - p/m)^S)
// (PMB_UNRANK_S overrides, for tuning).
static int pick_unrank_group(int m, int p) {
  if (const char* e = getenv("PMB_UNRANK_S")) {
    const int s = atoi(e);
    if (s == 8 || s == 16 || s == 32) return s;
  }
  const double q = (double)p / m;
  int best = 32;
  double bc = 1e300;
  for (int s : {8, 16, 32}) {
    const double c = s / 32.0 / (1.0 - std::pow(1.0 - q, s));
    if (c < bc) {
      bc = c;
      best = s;
    }
  }
  return best;
}

template <int kL>
static void launch_unrank(int S, const uint64_t* ranks, const uint64_t* table, int m, int p, int L, int wp,
                          int count, uint64_t* out, cudaStream_t st) {
  const unsigned g = (unsigned)(((size_t)count * S + 255) / 256);
  if (S == 8) k_unrank<kL, 8><<<g, 256, 0, st>>>(ranks, table, m, p, L, wp, count, out);
  else if (S == 16) k_unrank<kL, 16><<<g, 256, 0, st>>>(ranks, table, m, p, L, wp, count, out);
  else k_unrank<kL, 32><<<g, 256, 0, st>>>(ranks, table, m, p, L, wp, count, out);
}

// Reference-exact rank draws on the device.  The reference draws every rank of
// a generation's population from one sequential host stream (ga.cpp:226-235)
// with random_below(C(m, p)) (combinatorics.cpp:54-70): an attempt consumes
// `words` outputs (the first one masked to the top limb's bits, then shifted
// in below) and is accepted when the value is below the bound.  Splitmix
// outputs are random-access -- output i is mix64(state0 + (i+1) * gamma) -- so
// every attempt of a generation is tested at once and the accepted ones are
// compacted in stream order; the stream position lives on the device
// (rstate), so no host work and no synchronisation are involved.
__device__ __forceinline__ void attempt_value(uint64_t state0, uint64_t first, int words, uint64_t top_mask,
                                              uint64_t* v /* little-endian, words limbs */) {
  for (int w = 0; w < words; ++w) {
    uint64_t x = mix64(state0 + (first + (uint64_t)w + 1) * 0x9e3779b97f4a7c15ULL);
    if (w == 0) x &= top_mask;
    v[words - 1 - w] = x;
  }
}

// rstate: {stream position for even generations, for odd ones, shortfall
// flag}; generation g reads slot g&1 and writes slot (g+1)&1, so the blocks of
// one compaction never see a position updated under them.
__global__ void __launch_bounds__(256) k_rank_flags(uint64_t state0, const unsigned long long* __restrict__ rstate,
                                                    int slot, int words, uint64_t top_mask,
                                                    const uint64_t* __restrict__ bound, int L, int A,
                                                    uint32_t* __restrict__ flags, uint32_t* __restrict__ blockcnt) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  int cmp = 1;
  if (a < A) {
    uint64_t v[32];
    attempt_value(state0, rstate[slot] + (uint64_t)a * words, words, top_mask, v);
    cmp = 0;  // sign of v - bound, most significant limb first
    for (int i = L - 1; i >= 0 && cmp == 0; --i) {
      const uint64_t x = i < words ? v[i] : 0, b = bound[i];
      cmp = x < b ? -1 : (x > b ? 1 : 0);
    }
    flags[a] = cmp < 0;
  }
  const int c = __syncthreads_count(cmp < 0);
  if (threadIdx.x == 0) blockcnt[blockIdx.x] = (uint32_t)c;
}

// Stream-order compaction of the accepted attempts, one thread per attempt:
// ranks [lo, hi) of the population are written (islands keep their own
// slice), and the next generation's stream position is the one just past the
// total-th accepted attempt.
__global__ void __launch_bounds__(256) k_rank_compact(uint64_t state0, unsigned long long* __restrict__ rstate,
                                                      int slot, int words, uint64_t top_mask, int L, int A,
                                                      const uint32_t* __restrict__ flags,
                                                      const uint32_t* __restrict__ blockcnt, int total, int lo,
                                                      int hi, uint64_t* __restrict__ ranks) {
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {  // accepted attempts in the blocks before this one
    uint32_t sacc = 0;
    for (int b = lane; b < (int)blockIdx.x; b += 32) sacc += blockcnt[b];
    sacc = warp_sum(sacc);
    if (lane == 0) base = sacc;
  }
  const int a = blockIdx.x * blockDim.x + tid;
  const uint32_t f = a < A ? flags[a] : 0u;
  const unsigned bal = __ballot_sync(kFull, f);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  uint32_t k = base + __popc(bal & lanemask_lt());
  for (int w = 0; w < warp; ++w) k += wsum[w];
  const uint64_t pos = rstate[slot];
  if (f && (int)k < total) {
    if ((int)k >= lo && (int)k < hi) {
      uint64_t v[32];
      attempt_value(state0, pos + (uint64_t)a * words, words, top_mask, v);
      uint64_t* dst = ranks + (size_t)(k - lo) * L;
      for (int i = 0; i < L; ++i) dst[i] = i < words ? v[i] : 0;
    }
    if ((int)k == total - 1) rstate[slot ^ 1] = pos + (uint64_t)(a + 1) * words;
  }
  if (blockIdx.x == gridDim.x - 1 && tid == 0) {  // window exhausted (checked by the host)
    uint32_t all = base;
    for (int w = 0; w < 8; ++w) all += wsum[w];
    if (all < (uint32_t)total) rstate[2] = 1;
  }
}

static unsigned cdiv(size_t a, unsigned b) { return (unsigned)((a + b - 1) / b); }

// ---- GA engine ---------------------------------------------------------------------


struct GaShape {
  int nbl = 0, nt = 0, wp = 0, m = 0, p = 0, rounds = 0, attempts = 0, cycle = 0;
  uint64_t seed = 0;
  size_t block0 = 0;
};

static int lg2(size_t v) {
  int r = 0;
  while ((size_t{1} << r) < v) ++r;
  return r;
}

// One evolve_block over every local block (kernel index `kernel`).
static int evolve_all(pm_ctx* c, GaBuffers& B, const GaShape& s, uint64_t kernel) {
  const size_t count = (size_t)s.nbl * s.nt;
  // one thread per chromosome; 64-thread blocks spread the 15,360 threads of
  // the paper's shape over all SMs (256-thread blocks left 88 SMs idle)
  const unsigned tb = 64;
  uint64_t* pop = B.pop.as<uint64_t>();
  int64_t* cost = B.cost.as<int64_t>();
  unsigned long long* evals = B.evals.as<unsigned long long>();
  int rc = evaluate_core(c, pop, count, cost, 0);  // ga.cpp:146-147
  if (rc) return rc;
  if (s.p >= 2) {  // ga.cpp:154
    // ping-pong between pop and before: a round reads its snapshot `cur` and
    // the accept writes the next round's population into `nxt`
    uint64_t* cur = pop;
    uint64_t* nxt = B.before.as<uint64_t>();
    for (int r = 0; r < s.rounds; ++r) {
      k_crossover_children<<<cdiv(count, tb), tb, 0, c->stream>>>(
          cur, B.child.as<uint64_t>(), B.ok.as<uint8_t>(), s.nbl, s.nt, s.wp, s.m, s.p, s.seed, kernel, s.block0,
          (uint64_t)r, s.cycle);
      PM_CUDA_TRY(c, cudaGetLastError());
      rc = evaluate_core(c, B.child.as<uint64_t>(), count, B.ccost.as<int64_t>(), 0);
      if (rc) return rc;
      k_crossover_accept_pp<<<cdiv(count, tb), tb, 0, c->stream>>>(cur, nxt, cost, B.child.as<uint64_t>(),
                                                                    B.ccost.as<int64_t>(), B.ok.as<uint8_t>(),
                                                                    (int)count, s.wp, evals);
      PM_CUDA_TRY(c, cudaGetLastError());
      c->launches += 2;
      std::swap(cur, nxt);
    }
    if (cur != pop) {  // an odd round count left the population in `before`
      std::swap(B.pop, B.before);
      pop = B.pop.as<uint64_t>();
    }
  }
  if (s.attempts > 0) {
    const size_t sd_bytes = (size_t)32 * s.attempts * sizeof(ShiftDraw);
    if (sd_bytes <= 48 * 1024 && (size_t)s.attempts * s.wp * 32 < (size_t)INT32_MAX) {
      k_mutation_children_wide<<<cdiv(count, 32), 256, sd_bytes, c->stream>>>(
          pop, B.child.as<uint64_t>(), s.nbl, s.nt, s.wp, s.m, s.seed, kernel, s.block0, s.attempts);
    } else {
      k_mutation_children<<<cdiv(count, tb), tb, 0, c->stream>>>(pop, B.child.as<uint64_t>(), s.nbl, s.nt,
                                                                  s.wp, s.m, s.seed, kernel, s.block0,
                                                                  s.attempts);
    }
    PM_CUDA_TRY(c, cudaGetLastError());
    rc = evaluate_core(c, B.child.as<uint64_t>(), count * s.attempts, B.ccost.as<int64_t>(), 0);
    if (rc) return rc;
    k_mutation_accept<<<cdiv(count, tb), tb, 0, c->stream>>>(pop, cost, B.child.as<uint64_t>(),
                                                              B.ccost.as<int64_t>(), (int)count, s.attempts,
                                                              s.wp, evals);
    PM_CUDA_TRY(c, cudaGetLastError());
    c->launches += 2;
  }
  k_block_min<<<s.nbl, 256, 0, c->stream>>>(cost, pop, s.nt, s.wp, B.brec.as<uint64_t>());
  PM_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return PM_OK;
}

static int ga_alloc(pm_ctx* c, GaBuffers& B, const GaShape& s) {
  const size_t count = (size_t)s.nbl * s.nt;
  const size_t kids = count * std::max(1, s.attempts);
  PM_CUDA_TRY(c, B.pop.ensure(count * s.wp * 8));
  PM_CUDA_TRY(c, B.next.ensure(count * s.wp * 8));
  PM_CUDA_TRY(c, B.cost.ensure(count * 8));
  PM_CUDA_TRY(c, B.before.ensure(count * s.wp * 8));
  PM_CUDA_TRY(c, B.child.ensure(kids * s.wp * 8));
  PM_CUDA_TRY(c, B.ccost.ensure(kids * 8));
  PM_CUDA_TRY(c, B.ok.ensure(count));
  PM_CUDA_TRY(c, B.brec.ensure((size_t)s.nbl * (2 + s.wp) * 8));
  PM_CUDA_TRY(c, B.evals.ensure(16));
  PM_CUDA_TRY(c, B.tmp.ensure(16));
  return PM_OK;
}


// GaConfig::validate (ga.cpp:25-33), same texts.
static int validate_config(pm_ctx* c, const pm_ga_config* cfg) {
  if (!cfg) return c->fail(PM_STRUCTURAL, "null config");
  if (cfg->nb < 1) return c->fail(PM_DOMAIN, "nb must be >= 1");
  if (cfg->nt < 2 || (cfg->nt & (cfg->nt - 1)) != 0) return c->fail(PM_DOMAIN, "nt must be a power of two >= 2");
  if (cfg->evolve_limit < 1) return c->fail(PM_DOMAIN, "evolve_limit must be >= 1");
  if (cfg->saturation < 1) return c->fail(PM_DOMAIN, "saturation must be >= 1");
  if (cfg->migration == PM_MIGRATE_TEAM && cfg->nb > cfg->nt) return c->fail(PM_DOMAIN, "team migration needs nb <= nt");
  if (cfg->population != PM_POPULATION_REFERENCE && cfg->population != PM_POPULATION_DEVICE)
    return c->fail(PM_DOMAIN, "unknown population mode");
  return PM_OK;
}

// evolve_block's own checks only (ga.cpp:139-140): the run-level limits
// (evolve_limit, saturation, team migration) belong to run_ga.
static int validate_evolve_config(pm_ctx* c, const pm_ga_config* cfg) {
  if (!cfg) return c->fail(PM_STRUCTURAL, "null config");
  if (cfg->nt < 2 || (cfg->nt & (cfg->nt - 1)) != 0) return c->fail(PM_DOMAIN, "nt must be a power of two >= 2");
  return PM_OK;
}

static GaShape make_shape(pm_ctx* c, const pm_ga_config* cfg, size_t nbl, size_t block0) {
  GaShape s;
  s.nbl = (int)nbl;
  s.nt = (int)cfg->nt;
  s.m = c->t.m;
  s.p = c->t.p;
  s.wp = (s.m + 63) / 64;
  s.cycle = lg2(cfg->nt);
  s.rounds = cfg->crossover_iters >= 0 ? (int)cfg->crossover_iters : s.cycle;
  s.attempts = cfg->mutation_iters >= 0 ? (int)cfg->mutation_iters : s.cycle;
  s.seed = cfg->seed;
  s.block0 = block0;
  return s;
}

// Reference-exact population (ga.cpp:226-235): one host stream derive(seed,
// {1}) drawing nb*nt ranks in order; this rank unranks its own blocks
// (the draws of other ranks' blocks are consumed to stay in step).
struct HostDraw {
  Stream stream;
  UBig bound;
  size_t m = 0, p = 0;
  size_t L = 0;                // limbs of the device table / ranks (0: host draw and unranking)
  int words = 0;           // 64-bit outputs per random_below attempt
  uint64_t top_mask = 0;   // mask of the first (most significant) output
  double accept = 1.0;     // P(attempt accepted) = bound / 2^bits
  void init(uint64_t seed, size_t m_, size_t p_) {
    const uint64_t key[1] = {kHostTag};
    stream = Stream::derive(seed, key, 1);
    m = m_;
    p = p_;
    bound = binomial(m, p);
    UBig bm1 = bound;
    bm1.dec();
    const size_t bits = bm1.bit_length();
    words = (int)((bits + 63) / 64);
    const size_t top = bits - 64 * (words - 1);
    top_mask = top == 64 ? ~0ull : ((1ull << top) - 1);
    accept = bound.div_pow2(bits);
    // table entries C(x, y), x < m, y <= p, are at most C(m-1, min(p, (m-1)/2));
    // ranks are < C(m, p)
    const size_t L0 = std::max(binomial(m - 1, std::min(p, (m - 1) / 2)).limbs(), bound.limbs()) + 1;
    // device unranking while the Pascal table fits the budget (default 2 GiB of
    // the 180 GB: syn20k's 20000 x 201 x 27 limbs take 0.87 GB); PMB_PASCAL_MAX_MB
    // lowers it (tests force the host unranking path with it)
    const char* cap_env = std::getenv("PMB_PASCAL_MAX_MB");
    const size_t cap = (cap_env ? (size_t)std::atoll(cap_env) : (size_t)2048) << 20;
    if (L0 <= 32 && (m * (p + 1) + 1) * L0 * 8 <= cap) L = L0;
  }
  void draw(size_t total, size_t lo, size_t hi, uint64_t* out /* (hi-lo) x wp */) {
    std::vector<UBig> ranks;
    ranks.reserve(hi - lo);
    for (size_t i = 0; i < total; ++i) {
      UBig r = random_below(bound, stream);
      if (i >= lo && i < hi) ranks.push_back(std::move(r));
    }
    const size_t wp = (m + 63) / 64, n = ranks.size();
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const unsigned workers = (unsigned)std::min<size_t>(hw, std::max<size_t>(1, n / 64));
    auto work = [&](unsigned w) {
      for (size_t i = n * w / workers; i < n * (w + 1) / workers; ++i) unrank_combination(m, p, ranks[i], out + i * wp);
    };
    if (workers <= 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (unsigned w = 0; w < workers; ++w) pool.emplace_back(work, w);
      for (auto& th : pool) th.join();
    }
  }
};

}  // namespace pmb

using namespace pmb;

extern "C" {

int pm_evolve_blocks(pm_ctx* c, uint64_t* blocks, size_t nb, size_t words_per, const pm_ga_config* cfg,
                     uint64_t kernel_index, size_t first_block, int64_t* best_cost, size_t* best_thread) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  int rc = validate_evolve_config(c, cfg);
  if (rc) return rc;
  if (words_per != (size_t)(c->t.m + 63) / 64) return c->fail(PM_STRUCTURAL, kMsgLength);
  if (nb == 0) return PM_OK;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  GaBuffers& B = c->ga;  // grow-only, kept across calls
  const GaShape s = make_shape(c, cfg, nb, first_block);
  rc = ga_alloc(c, B, s);
  if (rc) return rc;
  const size_t count = nb * cfg->nt;
  PM_CUDA_TRY(c, cudaMemcpyAsync(B.pop.p, blocks, count * s.wp * 8, cudaMemcpyHostToDevice, c->stream));
  // every chromosome must open exactly p sites (the GA's invariant; see pmedian_b200.h)
  unsigned long long bad = ~0ull;
  PM_CUDA_TRY(c, cudaMemcpyAsync(B.tmp.p, &bad, 8, cudaMemcpyHostToDevice, c->stream));
  k_popcount_check<<<cdiv(count, 256), 256, 0, c->stream>>>(B.pop.as<uint64_t>(), (int)count, s.wp, s.m, s.p,
                                                             B.tmp.as<unsigned long long>());
  PM_CUDA_TRY(c, cudaMemcpyAsync(&bad, B.tmp.p, 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (bad != ~0ull) {
    return c->fail(PM_DOMAIN, "every chromosome of an evolved block must open exactly p sites");
  }
  PM_CUDA_TRY(c, cudaMemsetAsync(c->errw.p, 0xff, 8, c->stream));
  PM_CUDA_TRY(c, cudaMemsetAsync(B.evals.p, 0, 8, c->stream));
  rc = evolve_all(c, B, s, kernel_index);
  if (rc) {
    return rc;
  }
  const size_t rec = 2 + (size_t)s.wp;
  std::vector<uint64_t> hr(nb * rec);
  PM_CUDA_TRY(c, cudaMemcpyAsync(blocks, B.pop.p, count * s.wp * 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaMemcpyAsync(hr.data(), B.brec.p, nb * rec * 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  size_t fb = 0;
  rc = pm_check_errors(c, &fb);
  if (rc) return rc;
  for (size_t b = 0; b < nb; ++b) {
    if (best_cost) best_cost[b] = (int64_t)hr[b * rec];
    if (best_thread) best_thread[b] = (size_t)hr[b * rec + 1];
  }
  return PM_OK;
}

}  // extern "C"

namespace pmb {

// run_ga over islands.  The block records never leave the device: k_block_min
// writes them, the exchange (dev_fn: a device collective enqueued on the
// context stream, e.g. NCCL; host_fn: a host callback through pinned staging)
// gathers every island's records, and k_generation_step makes the global
// decision and migrates on the device.  The host only reads the stop word.
static int run_ga_impl(pm_ctx* c, const pm_ga_config* cfg, int rank, int world, pm_allgather_fn host_fn,
                       pm_allgather_device_fn dev_fn, void* user, uint64_t* best_words, int64_t* per_kernel_best,
                       pm_run_result* res) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  int rc = validate_config(c, cfg);
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !host_fn && !dev_fn))
    return c->fail(PM_DOMAIN, "invalid island layout");
  if (cfg->nb % (size_t)world != 0) return c->fail(PM_DOMAIN, "nb must be a multiple of the number of islands");
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  const auto t0 = std::chrono::steady_clock::now();
  const size_t nb = cfg->nb, nt = cfg->nt, nbl = nb / world, block0 = nbl * rank;
  GaBuffers& B = c->ga;  // grow-only, kept across calls
  const GaShape s = make_shape(c, cfg, nbl, block0);
  rc = ga_alloc(c, B, s);
  if (rc) return rc;
  const size_t count = nbl * nt, wp = s.wp;
  const bool ref_draw = cfg->population == PM_POPULATION_REFERENCE;
  HostDraw hd;
  std::vector<uint64_t> host_pop;
  if (ref_draw) {
    hd.init(cfg->seed, s.m, s.p);
    host_pop.resize(count * wp);
  }
  if (ref_draw && hd.L && !(B.tab_m == (size_t)s.m && B.tab_p == (size_t)s.p && B.tab_L == hd.L)) {
    // the Pascal table for device unranking: built and uploaded once per
    // (m, p, limbs), kept across runs
    B.tab_m = B.tab_p = B.tab_L = 0;
    const std::vector<uint64_t> tab = binomial_table(s.m, s.p, hd.L);
    PM_CUDA_TRY(c, B.table.ensure(tab.size() * 8));
    std::vector<double> lfact((size_t)s.m + 2);  // ln x!, the search guide of k_unrank_log
    for (size_t x = 0; x < lfact.size(); ++x) lfact[x] = std::lgamma((double)x + 1.0);
    PM_CUDA_TRY(c, B.lfact.ensure(lfact.size() * 8));
    PM_CUDA_TRY(c, cudaMemcpyAsync(B.lfact.p, lfact.data(), lfact.size() * 8, cudaMemcpyHostToDevice, c->stream));
    // stream-ordered upload: a plain cudaMemcpy runs on the legacy stream, which
    // does not order against the context's non-blocking streams (the first
    // draw could read a partly written table)
    PM_CUDA_TRY(c, cudaMemcpyAsync(B.table.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, c->stream));
    PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // `tab` is freed at the end of this block
    B.tab_m = (size_t)s.m;
    B.tab_p = (size_t)s.p;
    B.tab_L = hd.L;
  }
  if (ref_draw && hd.L) {
    PM_CUDA_TRY(c, B.ranks.ensure(count * hd.L * 8));
    PM_CUDA_TRY(c, B.rstate.ensure(24));  // {position (even gen), position (odd gen), shortfall}
    PM_CUDA_TRY(c, cudaMemsetAsync(B.rstate.p, 0, 24, c->stream));
  }
  // Draws run on their own stream: the population of generation g+1 does not
  // depend on generation g (ga.cpp:274), so its draw overlaps g's evolution;
  // the main stream waits for it only before migrating into it.
  cudaStream_t ds = c->draw_stream;
  auto draw = [&](DevBuf& dst, uint64_t generation) -> int {
    if (ref_draw && hd.L) {
      const int L = (int)hd.L, total = (int)(nb * nt);
      // attempts window: the accepted count falls short of `total` with
      // probability < 1e-30 (12 sigma); a shortfall is reported, never ignored
      const int A = (int)std::ceil((total + 12.0 * std::sqrt((double)total) + 64.0) / hd.accept);
      const unsigned G = cdiv(A, 256);
      PM_CUDA_TRY(c, B.rflags.ensure(((size_t)A + G) * 4));
      uint32_t* flags = B.rflags.as<uint32_t>();
      uint32_t* blockcnt = flags + A;
      const int slot = (int)(generation & 1);
      const uint64_t* bound = B.table.as<uint64_t>() + (size_t)(s.p + 1) * s.m * L;
      k_rank_flags<<<G, 256, 0, ds>>>(hd.stream.state, B.rstate.as<unsigned long long>(), slot, hd.words,
                                             hd.top_mask, bound, L, A, flags, blockcnt);
      k_rank_compact<<<G, 256, 0, ds>>>(hd.stream.state, B.rstate.as<unsigned long long>(), slot, hd.words,
                                               hd.top_mask, L, A, flags, blockcnt, total, (int)(block0 * nt),
                                               (int)((block0 + nbl) * nt), B.ranks.as<uint64_t>());
      PM_CUDA_TRY(c, cudaGetLastError());
      c->launches += 2;
      const int S = pick_unrank_group(s.m, s.p);
      const char* ue = getenv("PMB_UNRANK");
      if (!(ue && std::string(ue) == "probe")) {  // log-guided search (default)
        const unsigned gl = cdiv(count, 128);
        const double* lf = B.lfact.as<double>();
        uint64_t* o = dst.as<uint64_t>();
        const size_t lsm = (size_t)(s.m + 2) * 8 <= 48 * 1024 ? (size_t)(s.m + 2) * 8 : 0;
        if (L <= 8) k_unrank_log<8><<<gl, 128, lsm, ds>>>(B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), lf, s.m, s.p, L, (int)wp, (int)count, o);
        else if (L <= 16) k_unrank_log<16><<<gl, 128, lsm, ds>>>(B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), lf, s.m, s.p, L, (int)wp, (int)count, o);
        else k_unrank_log<32><<<gl, 128, lsm, ds>>>(B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), lf, s.m, s.p, L, (int)wp, (int)count, o);
      } else if (L <= 8) launch_unrank<8>(S, B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), s.m, s.p, L, (int)wp, (int)count, dst.as<uint64_t>(), ds);
      else if (L <= 16) launch_unrank<16>(S, B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), s.m, s.p, L, (int)wp, (int)count, dst.as<uint64_t>(), ds);
      else launch_unrank<32>(S, B.ranks.as<uint64_t>(), B.table.as<uint64_t>(), s.m, s.p, L, (int)wp, (int)count, dst.as<uint64_t>(), ds);
      PM_CUDA_TRY(c, cudaGetLastError());
      c->launches += 1;
    } else if (ref_draw) {
      hd.draw(nb * nt, block0 * nt, (block0 + nbl) * nt, host_pop.data());
      PM_CUDA_TRY(c, cudaMemcpyAsync(dst.p, host_pop.data(), count * wp * 8, cudaMemcpyHostToDevice, ds));
    } else {
      k_draw_population<<<cdiv(count, 64), 64, 0, ds>>>(dst.as<uint64_t>(), (int)count, (int)wp, s.m,
                                                                  s.p, cfg->seed, generation, block0 * nt);
      PM_CUDA_TRY(c, cudaGetLastError());
      c->launches += 1;
    }
    return PM_OK;
  };
  PM_CUDA_TRY(c, cudaMemsetAsync(c->errw.p, 0xff, 8, c->stream));
  PM_CUDA_TRY(c, cudaMemsetAsync(B.evals.p, 0, 8, c->stream));
  PM_CUDA_TRY(c, cudaEventRecord(c->draw_ev, c->stream));  // table / rstate uploads above
  PM_CUDA_TRY(c, cudaStreamWaitEvent(ds, c->draw_ev, 0));
  rc = draw(B.pop, 0);
  if (rc) return rc;
  PM_CUDA_TRY(c, cudaEventRecord(c->draw_ev, ds));
  PM_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->draw_ev, 0));

  // per-block record exchanged between islands: {cost, thread, words[wp]}
  const size_t rec = 2 + wp;
  const size_t bytes = nbl * rec * 8;
  PM_CUDA_TRY(c, B.grec.ensure(nb * rec * 8));
  PM_CUDA_TRY(c, B.gstate.ensure((kStateWords + wp) * 8));
  PM_CUDA_TRY(c, B.hflag.ensure(64));
  if (host_fn && world > 1) {
    PM_CUDA_TRY(c, B.hrec.ensure(bytes));
    PM_CUDA_TRY(c, B.hglob.ensure(nb * rec * 8));
  }
  {
    std::vector<uint64_t> st(kStateWords + wp, 0);
    st[0] = (uint64_t)std::numeric_limits<int64_t>::max();  // ga.cpp:241: kernel 0 always improves
    PM_CUDA_TRY(c, cudaMemcpyAsync(B.gstate.p, st.data(), st.size() * 8, cudaMemcpyHostToDevice, c->stream));
    PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // `st` is a host temporary
  }
  const uint64_t* grec = world > 1 ? B.grec.as<uint64_t>() : B.brec.as<uint64_t>();
  uint64_t* flag = B.hflag.as<uint64_t>();
  size_t kernels = 0;
  uint64_t device_evals = 0;
  double evolve_s = 0;
  const size_t kids_per_gen = count * (1 + (s.p >= 2 ? s.rounds : 0) + s.attempts);
  for (uint64_t kernel = 0;; ++kernel) {
    const auto g0 = std::chrono::steady_clock::now();
    if (kernel >= B.perk_cap) {  // per-kernel bests: grown on demand, never sized by evolve_limit
      const size_t cap = std::max<size_t>(64, 2 * B.perk_cap);
      DevBuf grown;
      PM_CUDA_TRY(c, grown.ensure(cap * 8));
      if (kernel) PM_CUDA_TRY(c, cudaMemcpyAsync(grown.p, B.perk.p, kernel * 8, cudaMemcpyDeviceToDevice, c->stream));
      PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      B.perk.release();
      B.perk = grown;
      grown.p = nullptr;
      B.perk_cap = cap;
    }
    rc = evolve_all(c, B, s, kernel);
    if (rc) return rc;
    device_evals += kids_per_gen;
    // draw the next population while the device evolves (ga.cpp:274)
    rc = draw(B.next, kernel + 1);
    if (rc) return rc;
    if (world > 1 && dev_fn) {  // device collective on the context stream (NVLink / NVSwitch)
      if (dev_fn(B.brec.p, bytes, B.grec.p, (void*)c->stream, user) != 0)
        return c->fail(PM_NCCL, "island allgather failed");
    } else if (world > 1) {  // host callback: pinned staging
      PM_CUDA_TRY(c, cudaMemcpyAsync(B.hrec.p, B.brec.p, bytes, cudaMemcpyDeviceToHost, c->stream));
      PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (host_fn(B.hrec.p, bytes, B.hglob.p, user) != 0) return c->fail(PM_NCCL, "island allgather failed");
      PM_CUDA_TRY(c, cudaMemcpyAsync(B.grec.p, B.hglob.p, nb * rec * 8, cudaMemcpyHostToDevice, c->stream));
    }
    // the step migrates into the next population: after its draw
    PM_CUDA_TRY(c, cudaEventRecord(c->draw_ev, ds));
    PM_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->draw_ev, 0));
    k_generation_step<<<1, 256, 0, c->stream>>>(grec, (int)nb, (int)wp, kernel, cfg->saturation, cfg->evolve_limit,
                                                B.gstate.as<uint64_t>(), B.perk.as<int64_t>(), B.next.as<uint64_t>(),
                                                (int)nt, cfg->migration == PM_MIGRATE_TEAM, (int)block0, (int)nbl,
                                                B.evals.as<unsigned long long>());
    PM_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
    PM_CUDA_TRY(c, cudaMemcpyAsync(flag, B.gstate.as<uint64_t>() + 4, 8, cudaMemcpyDeviceToHost, c->stream));
    PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    evolve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - g0).count();
    if (*flag) {
      kernels = (size_t)kernel + 1;
      break;
    }
    std::swap(B.pop, B.next);
  }
  PM_CUDA_TRY(c, cudaStreamSynchronize(ds));  // the last (unused) draw
  std::vector<uint64_t> st(kStateWords + wp);
  c->per_kernel_best.assign(kernels, 0);
  unsigned long long rstate[3] = {0, 0, 0};
  PM_CUDA_TRY(c, cudaMemcpyAsync(st.data(), B.gstate.p, st.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaMemcpyAsync(c->per_kernel_best.data(), B.perk.p, kernels * 8, cudaMemcpyDeviceToHost,
                                 c->stream));
  if (ref_draw && hd.L)
    PM_CUDA_TRY(c, cudaMemcpyAsync(rstate, B.rstate.p, 24, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (rstate[2]) return c->fail(PM_CUDA, "population draw: attempt window exhausted");
  size_t fb = 0;
  rc = pm_check_errors(c, &fb);
  if (rc) return rc;
  if (best_words) std::memcpy(best_words, &st[kStateWords], wp * 8);
  if (per_kernel_best) std::memcpy(per_kernel_best, c->per_kernel_best.data(), kernels * 8);
  if (res) {
    res->best_cost = (int64_t)st[0];
    res->kernels_executed = kernels;
    res->kernel_of_best = (size_t)st[1];
    res->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    res->evolve_time_s = evolve_s;
    res->evaluations = st[5] + (uint64_t)kernels * count;  // + the initial evaluation of each generation
    res->device_evaluations = device_evals;
  }
  return PM_OK;
}

}  // namespace pmb

extern "C" {

int pm_run_ga_islands(pm_ctx* c, const pm_ga_config* cfg, int rank, int world, pm_allgather_fn allgather,
                      void* user, uint64_t* best_words, int64_t* per_kernel_best, pm_run_result* res) {
  return pmb::run_ga_impl(c, cfg, rank, world, allgather, nullptr, user, best_words, per_kernel_best, res);
}

int pm_run_ga_islands_device(pm_ctx* c, const pm_ga_config* cfg, int rank, int world,
                             pm_allgather_device_fn allgather, void* user, uint64_t* best_words,
                             int64_t* per_kernel_best, pm_run_result* res) {
  return pmb::run_ga_impl(c, cfg, rank, world, nullptr, allgather, user, best_words, per_kernel_best, res);
}

int pm_last_per_kernel_best(pm_ctx* c, int64_t* out, size_t capacity, size_t* count) {
  if (!c) return PM_STRUCTURAL;
  const size_t k = c->per_kernel_best.size();
  if (count) *count = k;
  if (out) std::memcpy(out, c->per_kernel_best.data(), std::min(k, capacity) * 8);
  return PM_OK;
}

int pm_run_ga(pm_ctx* c, const pm_ga_config* cfg, uint64_t* best_words, int64_t* per_kernel_best,
              pm_run_result* res) {
  return pm_run_ga_islands(c, cfg, 0, 1, nullptr, nullptr, best_words, per_kernel_best, res);
}

}  // extern "C"
