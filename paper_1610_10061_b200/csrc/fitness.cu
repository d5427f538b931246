// K2 / K2b: population fitness on the device.
//
// Replaces the per-chromosome loop of pmedian::fitness
// (/root/reference/proj/src/ordering.cpp:40-59) as evolve_block calls it
// (ga.cpp:147,166,183).  Per chromosome c and client i the reference scans
// client i's ordered sites until the first open one (k*_i) and adds the
// increments up to and including it; that prefix sum is dist[i][k*_i].
//
// K2 ("scan", bit-sliced).  32 (or 64) chromosomes form a group.  The group's
// open sets are transposed into T[s] (bit c = chromosome c has site s open),
// staged in shared memory.  Each lane owns one client at a time and walks its
// row once for the whole group: alive &= ~T[pi_ik], and every bit leaving
// `alive` at column k is a (chromosome, client) pair whose cost is dist[i][k].
// One row walk of length max_c k*_ic serves the whole group, so a row prefix
// is read from L2/HBM once per group instead of once per chromosome; lanes
// claim clients dynamically so a short row does not wait for a long one.  Hits
// are accumulated into per-lane private shared-memory counters (no atomics) and
// reduced once per CTA segment.
//
// K2b ("gather", gather-min, gather.cu).  fitness = sum_i min_{j open} cost(i, j)
// (instance.cpp:32-48, equal to the scan by acceptance.cpp:86-116).  A thread
// owns 16 bytes of consecutive clients (8 at u16 costs); each open site j of a
// chromosome is one 16-byte read of the site-major row dT[j][i0..] and a packed
// min.  Wins when p is small (the scan reads ~m/p columns per client, the
// gather p): AUTO picks the scan iff p >= 1.1 sqrt(m), measured.  The reference's scan-width contract
// (ordering.cpp:50-52) is enforced exactly: with popcount >= p it cannot fail
// (W = m-p+1 columns always contain one of p distinct sites); with fewer open
// sites the (cost, site)-smallest open site must not sort after column W-1.
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace pmb {

// ---- K2t: population -> transposed group masks ------------------------------

size_t scan_t_stride(int m) { return ((size_t)m + 1 + 1) / 2 * 2; }

// 32 x 32 bit-matrix transpose across a warp: lane L holds row L (bit b =
// element (L, b)); on return lane L holds column L (bit b = element (b, L)).
__device__ __forceinline__ uint32_t transpose32(int lane, uint32_t x) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int j = 16 >> i;
    const uint32_t m = masks[i];
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

__global__ void __launch_bounds__(256) k_transpose_population(const uint64_t* __restrict__ words,
                                                              size_t count, int wp, int m,
                                                              uint64_t* __restrict__ T,
                                                              size_t Ts,
                                                              unsigned long long* __restrict__ costs,
                                                              unsigned long long* __restrict__ err_init) {
  const int lane = threadIdx.x & 31;
  const int wi = blockIdx.x * 8 + (threadIdx.x >> 5);
  const size_t groups = (count + 63) / 64;
  // the call's error word starts at "none" (replaces a memset; the scan runs after)
  if (err_init && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *err_init = ~0ull;
  // groups stride over gridDim.y (<= 65535) so any population size launches
  for (size_t g = blockIdx.y; g < groups; g += gridDim.y) {
    uint64_t* Tg = T + g * Ts;
    if (blockIdx.x == 0 && threadIdx.x < 32) {
      for (size_t s = (size_t)m + lane; s < Ts; s += 32) Tg[s] = 0;  // sentinel site m
    }
    // the scan accumulates into costs: zero the group's 64 (replaces a memset launch)
    if (blockIdx.x == 0 && threadIdx.x >= 64 && threadIdx.x < 128 && g * 64 + threadIdx.x - 64 < count)
      costs[g * 64 + threadIdx.x - 64] = 0;
    if (wi >= wp) continue;  // warp-uniform
    const size_t c0 = g * 64 + lane, c1 = c0 + 32;
    const uint64_t x = c0 < count ? words[c0 * wp + wi] : 0;
    const uint64_t y = c1 < count ? words[c1 * wp + wi] : 0;
    // four 32 x 32 bit transposes (butterfly over the lanes: 5 shuffle stages
    // each): lane L ends with bit c = chromosome c opens site 64 wi + L (+ 32)
    const uint64_t t0 =
        (uint64_t)transpose32(lane, (uint32_t)x) | ((uint64_t)transpose32(lane, (uint32_t)y) << 32);
    const uint64_t t1 = (uint64_t)transpose32(lane, (uint32_t)(x >> 32)) |
                        ((uint64_t)transpose32(lane, (uint32_t)(y >> 32)) << 32);
    const int s0 = wi * 64 + lane, s1 = s0 + 32;
    if (s0 < m) Tg[s0] = t0;
    if (s1 < m) Tg[s1] = t1;
  }
}

cudaError_t launch_transpose_population(const uint64_t* words, size_t count, int words_per, int m,
                                        uint64_t* T, unsigned long long* costs, unsigned long long* err_init,
                                        cudaStream_t st) {
  const size_t groups = (count + 63) / 64;
  dim3 grid((words_per + 7) / 8, (unsigned)std::min<size_t>(groups, 65535));
  k_transpose_population<<<grid, 256, 0, st>>>(words, count, words_per, m, T, scan_t_stride(m), costs, err_init);
  return cudaGetLastError();
}

// ---- K2: bit-sliced scan -------------------------------------------------------

constexpr int kChunk = 16;  // columns per lane step (32 B of u16 sites)
// A/B switches for K2 variants (tools/build_variant.sh); defaults are the
// measured choice (profiles/r02_k2_ab.md: every switch on is slower at syn20k)
#ifndef PMB_X_SPLITQ
#define PMB_X_SPLITQ 0
#endif
#ifndef PMB_X_BFIND
#define PMB_X_BFIND 0
#endif
#ifndef PMB_X_NOSENT
#define PMB_X_NOSENT 0
#endif
#ifndef PMB_X_RED
#define PMB_X_RED 0
#endif
// ... and for the short-segment shapes of the many-warp variant only (2- and
// 4-warp CTAs: pmed40-size instances, the GA's evaluation batches), where the
// split records and the FLO-indexed drain measured faster (0.072 -> 0.069 ms)
#ifndef PMB_X_SHORT
#define PMB_X_SHORT 1
#endif
constexpr int kWideWarps = 24, kWideQueue = 256;  // the many-warp K2 variant (plan_scan)
#ifndef PMB_PAIRQ
#define PMB_PAIRQ 192
#endif
constexpr int kPairQueue = PMB_PAIRQ;  // its column-pair CTA: 192 records (syn20k -1.2 % vs 256)
constexpr int kCoop = 16;          // clients per warp at which the cooperative tail starts
constexpr int kTailClaim = 32;     // clients left per warp below which claims shrink (tools/env_ab.sh)
#ifndef PMB_QCHECK
#define PMB_QCHECK 2
#endif
constexpr int kQCheck = PMB_QCHECK;  // columns between queue-overflow checks (many-warp variant)
static_assert(16 % kQCheck == 0 && kWideQueue > 32 * kQCheck, "queue check stride");
static_assert(kPairQueue % 2 == 0 && kPairQueue >= 64 && kPairQueue <= kWideQueue, "pair queue: whole pairs");

template <class OrdT, class DistT>
struct Chunk {
  static constexpr int kO = kChunk * sizeof(OrdT) / 16;   // uint4s of sites
  static constexpr int kD = kChunk * sizeof(DistT) / 16;  // uint4s of costs
  uint4 o[kO];
  uint4 d[kD];

  // 32-byte loads (LDG.256): one full sector per lane per instruction; rows
  // are 32-byte aligned (Wp is a multiple of 16 elements, k of kChunk).
  __device__ __forceinline__ void load(const OrdT* orow, const DistT* drow, int k) {
#pragma unroll
    for (int x = 0; x < kO; x += 2) ldg_stream32(reinterpret_cast<const uint4*>(orow + k) + x, o[x], o[x + 1]);
#pragma unroll
    for (int x = 0; x < kD; x += 2) ldg_stream32(reinterpret_cast<const uint4*>(drow + k) + x, d[x], d[x + 1]);
  }
  // Every site of the chunk becomes `s` (the never-open sentinel site m).
  __device__ __forceinline__ void set_sentinel(uint32_t s) {
    const uint32_t w = sizeof(OrdT) == 2 ? (s | (s << 16)) : s;
#pragma unroll
    for (int x = 0; x < kO; ++x) o[x] = make_uint4(w, w, w, w);
  }
  __device__ __forceinline__ uint32_t site(int j) const {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(o);
    if constexpr (sizeof(OrdT) == 2) return (w[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
    else return w[j];
  }
  // u16 costs: the 32-bit word holding column j's cost in its low 16 bits
  // (the high half is the next column's cost for even j)
  __device__ __forceinline__ uint32_t cost_raw(int j) const {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(d);
    return (j & 1) ? (w[j >> 1] >> 16) : w[j >> 1];
  }
  __device__ __forceinline__ uint64_t cost(int j) const {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(d);
    if constexpr (sizeof(DistT) == 2) return (w[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
    else if constexpr (sizeof(DistT) == 4) return w[j];
    else return (uint64_t)w[2 * j] | ((uint64_t)w[2 * j + 1] << 32);
  }
};

// Group width: MaskT = uint64_t (64 chromosomes per row walk) or uint32_t (32).
// Wider groups amortise a row walk over more evaluations (E[max k*] grows only
// like H_G) but need twice the shared memory per site and per lane counter;
// plan_scan picks the width that keeps enough warps resident.
template <class MaskT>
struct MaskOps {
  static constexpr int kG = 8 * sizeof(MaskT);
  template <bool kFlo>
  __device__ __forceinline__ static int pop_high(MaskT& h) {  // index of the top set bit, cleared
    if constexpr (sizeof(MaskT) == 4) {
      int c;
      if constexpr (kFlo) asm("bfind.u32 %0, %1;" : "=r"(c) : "r"(h));  // FLO: the top bit's position directly
      else c = 31 - __clz(h);
      h ^= 1u << c;
      return c;
    } else {
      const int c = 63 - __clzll((long long)h);
      h ^= 1ull << c;
      return c;
    }
  }
  __device__ __forceinline__ static int low_index(MaskT h) {
    return sizeof(MaskT) == 4 ? __ffs((int)h) - 1 : __ffsll((long long)h) - 1;
  }
};

// kTSmem: the group's masks T live in shared memory; otherwise they are read
// from global memory through L1/L2 (any m).
//
// Per chunk of 16 columns a lane (1) looks up the 16 masks, (2) walks them to
// update `alive`, appending each column's newly-dead chromosomes h_j and the
// column's cost to the warp's shared-memory queue (ballot + popc position, no
// loops), and (3) the warp drains the queue lane-parallel into per-lane
// private counters acc[c][lane] (no atomics, no bank conflicts).  The drain
// loop runs the largest record's bit count, so one lane's burst of hits at a
// client start no longer stalls the warp.
// kW > 0: the many-warp variant -- kW warps per SM in CTAs of kCtaW warps
// (registers capped at 64K / (32 kW)), a kWQ-record queue, two row chunks.
template <class OrdT, class DistT, class AccT, class MaskT, bool kTSmem, bool kDepth, int kW = 0, int kWQ = 128,
          int kCtaW = kW, bool kPairCols = false>
__global__ void __launch_bounds__(kW ? kCtaW * 32 : 512, kW ? kW / (kCtaW ? kCtaW : 1) : 1)
    k_scan(const OrdT* __restrict__ ord, const DistT* __restrict__ dist, int n, int Wp,
           const uint64_t* __restrict__ T, size_t Ts, size_t count, int groups,
           unsigned long long* __restrict__ costs, unsigned long long* __restrict__ err, int coop,
           int tail_claim) {
  using Ops = MaskOps<MaskT>;
  constexpr int kG = Ops::kG;
  // row chunks in registers: 3 (two in flight while one is consumed) when the
  // table types are narrow, else 2 to stay within the register budget
  constexpr int kBufs = (kW == 0 && sizeof(OrdT) + sizeof(DistT) <= 4) ? 3 : 2;
  // queue records per warp: a whole chunk's worth, or (kW: many warps per SM,
  // less shared memory per warp) kQ with a mid-chunk drain when it could overflow
  constexpr int kQ = kW ? kWQ : kChunk * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const int nwarps = blockDim.x >> 5;
  MaskT* Tsm = reinterpret_cast<MaskT*>(smem);
  const size_t tbytes = kTSmem ? (Ts * sizeof(MaskT) + 15) / 16 * 16 : 0;
  AccT* acc = reinterpret_cast<AccT*>(smem + tbytes);                              // [warp][c][lane]
  MaskT* hbuf = reinterpret_cast<MaskT*>(acc + (size_t)nwarps * kG * 32);           // [warp][kQ]
  AccT* dbuf = reinterpret_cast<AccT*>(hbuf + (size_t)nwarps * kQ);                // [warp][kQ]
  int* next_client = reinterpret_cast<int*>(dbuf + (size_t)nwarps * kQ);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = lanemask_lt();
  AccT* myacc = acc + (size_t)warp * kG * 32 + lane;
  // the warp's queue of hit columns (at most kChunk * 32 per chunk).  32-bit
  // masks and costs: one [mask x kQ | cost x kQ] region per warp, so both
  // stores of a record share one address register (immediate offset kQ * 4)
  // and need no register pair; otherwise separate [warp][kQ] arrays.
  constexpr bool kPacked = sizeof(MaskT) == 4 && sizeof(AccT) == 4;
  MaskT* wqh = kPacked ? hbuf + (size_t)warp * 2 * kQ : hbuf + (size_t)warp * kQ;
  AccT* wqd = kPacked ? reinterpret_cast<AccT*>(wqh + kQ) : dbuf + (size_t)warp * kQ;
  uint64_t* wq = reinterpret_cast<uint64_t*>(hbuf) + (size_t)warp * kQ;  // one 8-byte record (!kSplitQ)
  (void)wq;
  // u16 sorted distances: a record of an even column stores the raw 32-bit
  // word holding the column's cost in its low half (no extraction in the
  // column loop); the drain masks it
  constexpr bool kShortCta = kW > 0 && kCtaW < kW;
  constexpr bool kSplitQ = kPacked && (PMB_X_SPLITQ || (PMB_X_SHORT && kShortCta));
  constexpr bool kFlo = PMB_X_BFIND || (PMB_X_SHORT && kShortCta);
  constexpr bool kRawCost = kSplitQ && !kDepth && sizeof(DistT) == 2 && sizeof(AccT) == 4;
  // column pairs (plan_scan: long walks only): one ballot per two columns
  constexpr bool kPair = kPairCols && kPacked && !kSplitQ && kW > 0 && !kShortCta && !kDepth;

  const long long U = (long long)groups * n;
  long long u = U * blockIdx.x / gridDim.x;
  const long long uend = U * (blockIdx.x + 1) / gridDim.x;
  while (u < uend) {
    const int g = (int)(u / n);
    const int c0 = (int)(u % n);
    const int c1 = (int)min((long long)n, c0 + (uend - u));
    u += c1 - c0;
    // T is stored as 64-chromosome words; a 32-wide group is one half of one
    const uint64_t* Tg = T + (size_t)(g * kG / 64) * Ts;
    const int half = (kG == 32) ? (g & 1) * 32 : 0;

    {  // stage the group's masks, clear the counters
      if constexpr (kTSmem) {
        if constexpr (kG == 64) {
          const uint4* src = reinterpret_cast<const uint4*>(Tg);
          uint4* dstT = reinterpret_cast<uint4*>(Tsm);
          for (size_t x = tid; x < Ts / 2; x += blockDim.x) dstT[x] = src[x];
        } else {
          // 8 independent loads in flight per thread: small CTAs (2 warps at
          // pmed40's shape) would otherwise pay one L2 round trip per 64 masks
          constexpr int kU = 8;
          for (size_t x0 = tid; x0 < Ts; x0 += (size_t)blockDim.x * kU) {
            uint64_t v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const size_t x = x0 + (size_t)u * blockDim.x;
              v[u] = x < Ts ? __ldg(Tg + x) : 0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const size_t x = x0 + (size_t)u * blockDim.x;
              if (x < Ts) Tsm[x] = (MaskT)(v[u] >> half);
            }
          }
        }
      }
      for (int x = tid; x < nwarps * kG * 32; x += blockDim.x) acc[x] = 0;
      if (tid == 0) *next_client = c0;
    }
    __syncthreads();
    const size_t nvalid = min((size_t)kG, count - (size_t)g * kG);
    const MaskT vmask = nvalid == (size_t)kG ? (MaskT)~(MaskT)0 : (MaskT)((((MaskT)1) << nvalid) - 1);

    int i = -1, k = 0;
    MaskT alive = 0;
    const OrdT* orow = nullptr;
    const DistT* drow = nullptr;
    Chunk<OrdT, DistT> ca, cb, cc;
    // T[Ts-1] is a zero mask (k_transpose_population clears [m, Ts)): idle
    // lanes look it up and never hit
    const uint32_t sentinel = (uint32_t)(Ts - 1);
    ca.set_sentinel(sentinel);
    cb.set_sentinel(sentinel);
    cc.set_sentinel(sentinel);
    int wb_next = 0, wb_end = 0;
    bool exhausted = false;

    // drain: lane r applies queue records r, r+32, ... -- the loop runs the
    // largest record's bit count, not the busiest lane's hit count
    auto drain = [&](uint32_t qn) {
      __syncwarp();  // queue writes visible to the draining lanes
      for (uint32_t base = 0; base < qn; base += 32) {
        MaskT h = 0;
        AccT dv = 0;
        if (base + lane < qn) {
          if constexpr (kPacked && !kSplitQ) {
            const uint64_t x = wq[base + lane];
            h = (MaskT)x;
            dv = (AccT)(x >> 32);
          } else {
            h = wqh[base + lane];
            dv = wqd[base + lane];
          }
          if constexpr (kRawCost) dv &= 0xffffu;
        }
        while (h) {
          const int c = Ops::template pop_high<kFlo>(h);
#if PMB_X_RED
          // a shared-memory reduction: lane-private column (no contention),
          // and the lane does not wait for a load-add-store round trip
          if constexpr (sizeof(AccT) == 4) atomicAdd(reinterpret_cast<unsigned*>(myacc + c * 32), (unsigned)dv);
          else atomicAdd(reinterpret_cast<unsigned long long*>(myacc + c * 32), (unsigned long long)dv);
#else
          myacc[c * 32] += dv;
#endif
        }
      }
      __syncwarp();  // the queue is rewritten next
    };
    // the 16 masks of chunk `cur` (idle lanes hold sentinel sites: zero masks)
    auto lookup = [&](const Chunk<OrdT, DistT>& cur, MaskT (&t)[kChunk]) {
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        PMB_CHECK(cur.site(j) < Ts);
        if constexpr (kTSmem) t[j] = Tsm[cur.site(j)];
        else t[j] = (MaskT)(__ldg(Tg + cur.site(j)) >> half);
      }
    };
    // the column phase of one chunk: walk `al` over the masks, appending hit
    // columns to the warp queue, then drain it; kb = the chunk's first column
    auto columns = [&](const Chunk<OrdT, DistT>& cur, const MaskT (&t)[kChunk], MaskT& al, int kb) {
      uint32_t qn = 0;  // warp-uniform queue length
      if constexpr (kPair) {
        // column pairs: one ballot per pair, and a lane with a hit in either
        // column appends both columns' records with one 16-byte store (an empty
        // mask drains as a no-op)
#pragma unroll
        for (int j = 0; j < kChunk; j += 2) {
          if (qn > (uint32_t)(kQ - 64)) {
            drain(qn);
            qn = 0;
          }
          const MaskT h0 = al & t[j];
          al &= ~t[j];
          const MaskT h1 = al & t[j + 1];
          al &= ~t[j + 1];
          const unsigned hb = __ballot_sync(kFull, (h0 | h1) != 0);
          if (h0 | h1) {
            const uint32_t q = qn + 2 * __popc(hb & lt);
            PMB_CHECK(q + 1 < (uint32_t)kQ);
            *reinterpret_cast<uint4*>(wq + q) =
                make_uint4((uint32_t)h0, (uint32_t)cur.cost(j), (uint32_t)h1, (uint32_t)cur.cost(j + 1));
          }
          qn += 2 * __popc(hb);
        }
      } else {
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          if constexpr (kQ < kChunk * 32) {
            // every kQCheck columns (warp-uniform): the next kQCheck columns could overflow
            if (j % kQCheck == 0 && qn > (uint32_t)(kQ - 32 * kQCheck)) {
              drain(qn);
              qn = 0;
            }
          }
          const MaskT h = al & t[j];
          al &= ~t[j];
          const unsigned hb = __ballot_sync(kFull, h != 0);
          if (h) {
            // kDepth: the 1-based stopping column k* instead of the cost
            // (B_eval = 12 * sum_i k*_i + 8 * ceil(m/64))
            AccT dval;
            if constexpr (kDepth) dval = (AccT)(kb + j + 1);
            else if constexpr (kRawCost) dval = (AccT)cur.cost_raw(j);
            else dval = (AccT)cur.cost(j);
            const uint32_t q = qn + __popc(hb & lt);
            PMB_CHECK(q < (uint32_t)kQ);
            if constexpr (kPacked && !kSplitQ) {
              wq[q] = (uint64_t)h | ((uint64_t)dval << 32);
            } else {
              wqh[q] = h;
              wqd[q] = dval;
            }
          }
          qn += __popc(hb);
        }
      }
      drain(qn);
    };
    // One 16-column step on chunk `cur`; `nxt` already holds the following
    // chunk and `cur` is refilled with the one after it.  Returns false once
    // the warp has no client left (or at most `coop` once the segment's
    // clients are all claimed: the cooperative tail below takes them).
    auto step = [&](Chunk<OrdT, DistT>& cur, Chunk<OrdT, DistT>& nxt,
                    Chunk<OrdT, DistT>& nxt2) -> bool {
      unsigned need = __ballot_sync(kFull, i < 0);
      while (need && !exhausted) {  // warp-uniform client claiming
        if (wb_next >= wb_end) {
          // batches of 32 clients, but only as many as lanes need once fewer
          // than tail_claim are left: a warp holding a private batch while the
          // others run dry stretches the segment's tail
          int base = 0, take = 32;
          if (lane == 0) {
            if (c1 - *reinterpret_cast<volatile int*>(next_client) < tail_claim) take = __popc(need);
            base = atomicAdd(next_client, take);
          }
          base = __shfl_sync(kFull, base, 0);
          take = __shfl_sync(kFull, take, 0);
          if (base >= c1) {
            exhausted = true;
            break;
          }
          wb_next = base;
          wb_end = min(base + take, c1);
        }
        const int rank = __popc(need & lt);
        const int avail = wb_end - wb_next;
        if (i < 0 && rank < avail) {
          i = wb_next + rank;
          PMB_CHECK(i >= c0 && i < c1 && c1 <= n);
          k = 0;
          alive = vmask;
          orow = ord + (size_t)i * Wp;
          drow = dist + (size_t)i * Wp;
          cur.load(orow, drow, 0);
          if (kChunk < Wp) nxt.load(orow, drow, kChunk);
          if (kBufs == 3 && 2 * kChunk < Wp) nxt2.load(orow, drow, 2 * kChunk);
        }
        wb_next += min(__popc(need), avail);
        need = __ballot_sync(kFull, i < 0);
      }
      {
        const unsigned busy = __ballot_sync(kFull, i >= 0);
        if (busy == 0 || (exhausted && __popc(busy) <= (coop & 0xff))) return false;
      }
      // Every lane runs the column phase (idle lanes hold sentinel sites and
      // alive == 0), so the warp can append its hit columns to one queue with
      // ballots instead of per-lane slots.
      MaskT t[kChunk];
      lookup(cur, t);
      columns(cur, t, alive, k);
      if (i >= 0) {
        k += kChunk;
        if (alive == 0 || k >= Wp) {
          if (alive) atomicMin(err, (unsigned long long)g * kG + Ops::low_index(alive));
          i = -1;
          alive = 0;  // the idle lane's stale chunks keep valid site indices (< Ts): its lookups never hit
#if !PMB_X_NOSENT
          cur.set_sentinel(sentinel);
          nxt.set_sentinel(sentinel);
          nxt2.set_sentinel(sentinel);
#endif
        } else if (k + (kBufs - 1) * kChunk < Wp) {
          PMB_CHECK(k + kBufs * kChunk <= Wp);
          cur.load(orow, drow, k + (kBufs - 1) * kChunk);
        }
      }
      return true;
    };
    if constexpr (kBufs == 3) {
      while (step(ca, cb, cc) && step(cb, cc, ca) && step(cc, ca, cb)) {
      }
    } else {
      while (step(ca, cb, cb) && step(cb, ca, ca)) {
      }
    }
    {
      // Cooperative tail.  Once the segment's clients are all claimed, a warp
      // with few clients left would step 16 columns at a time with most lanes
      // idle until its longest walk ends (the walk of the last of 32
      // chromosomes, ~(m/p) H_32 columns: the launch tail).  Instead (at most
      // coop & 0xff clients left) the clients walk side by side, each on a
      // segment of S lanes -- the largest power of two with S x clients <= 32,
      // at most 1 << (coop >> 8) -- lane r of a segment taking columns
      // [k + 16 r, k + 16 r + 16), re-packed every pass as clients finish.  A
      // chromosome's first open site is in the lowest lane whose columns hold
      // one, so lane r walks with the chromosomes no lower lane of its segment
      // hits (an exclusive OR-scan of the lanes' hit unions) and the records
      // are exactly those of the sequential walk.
      {
        const int lg_max = (coop >> 8) & 31;
        for (;;) {
          const unsigned act = __ballot_sync(kFull, i >= 0);
          if (act == 0) break;
          const int na = __popc(act);
          const int lgS = min(lg_max, 5 - (32 - __clz(na - 1)));
          const int S = 1 << lgS;
          const int seg = lane >> lgS, sl = lane & (S - 1);
          const bool on = seg < na;
          const int L = on ? (int)__fns(act, 0, seg + 1) : 0;
          const int ci = __shfl_sync(kFull, i, L);
          const int ck = __shfl_sync(kFull, k, L);
          MaskT A = __shfl_sync(kFull, alive, L);
          if (!on) A = 0;
          const int kk = ck + sl * kChunk;
          if (on && kk < Wp) ca.load(ord + (size_t)ci * Wp, dist + (size_t)ci * Wp, kk);
          else ca.set_sentinel(sentinel);
          MaskT t[kChunk];
          lookup(ca, t);
          MaskT U = 0;
#pragma unroll
          for (int j = 0; j < kChunk; ++j) U |= t[j];
          U &= A;
          MaskT P = U;  // inclusive OR over the segment's lanes <= sl
          for (int o = 1; o < S; o <<= 1) {
            const MaskT v = __shfl_up_sync(kFull, P, o, S);
            if (sl >= o) P |= v;
          }
          MaskT below = __shfl_up_sync(kFull, P, 1, S);
          if (sl == 0) below = 0;
          MaskT al = A & ~below;
          columns(ca, t, al, kk);
          const MaskT left = A & ~__shfl_sync(kFull, P, S - 1, S);  // uniform in the segment
          // back to the owning lanes: the client of rank r walked on segment r
          const MaskT got = __shfl_sync(kFull, left, (__popc(act & lt) << lgS) & 31);
          if (i >= 0) {
            k += S * kChunk;
            alive = got;
            if (alive == 0 || k >= Wp) {
              if (alive) atomicMin(err, (unsigned long long)g * kG + Ops::low_index(alive));
              i = -1;
              alive = 0;
            }
          }
        }
      }
    }
    __syncthreads();
    for (int c = tid; c < (int)nvalid; c += blockDim.x) {  // chromosome c: sum every lane's counter
      unsigned long long s = 0;
      for (int w = 0; w < nwarps; ++w) {
        const AccT* a = acc + ((size_t)w * kG + c) * 32;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) s += (unsigned long long)a[(l + c) & 31];
      }
      atomicAdd(&costs[(size_t)g * kG + c], s);
    }
    __syncthreads();
  }
}

static size_t scan_smem(int m, int warps, bool acc32, bool tsmem, int G, int qrec = kChunk * 32) {
  const size_t ab = acc32 ? 4 : 8, mb = G / 8;
  const size_t tb = tsmem ? (scan_t_stride(m) * mb + 15) / 16 * 16 : 0;
  return tb + (size_t)warps * (32 * G * ab + (size_t)qrec * (mb + ab)) + 16;
}

template <class OrdT, class DistT, class AccT, bool kDepth>
static const void* scan_fn_depth(int G, bool tsmem) {
  if (G == 64)
    return tsmem ? reinterpret_cast<const void*>(k_scan<OrdT, DistT, AccT, uint64_t, true, kDepth>)
                 : reinterpret_cast<const void*>(k_scan<OrdT, DistT, AccT, uint64_t, false, kDepth>);
  return tsmem ? reinterpret_cast<const void*>(k_scan<OrdT, DistT, AccT, uint32_t, true, kDepth>)
               : reinterpret_cast<const void*>(k_scan<OrdT, DistT, AccT, uint32_t, false, kDepth>);
}

static thread_local bool g_depth = false;  // selects the kDepth instantiation in scan_kernel_ptr

template <class OrdT, class DistT, class AccT>
static const void* scan_fn_acc(int G, bool tsmem) {
  return g_depth ? scan_fn_depth<OrdT, DistT, AccT, true>(G, tsmem)
                 : scan_fn_depth<OrdT, DistT, AccT, false>(G, tsmem);
}

static const void* scan_kernel_ptr(const DevTables& t, bool acc32, int G, bool ts, int wide = 0,
                                   bool pair = false) {
  if (wide && t.site_bytes == 2 && t.dist_bytes == 2 && acc32 && G == 32 && ts && !g_depth) {
    // wide = warps per CTA of the variant (kWideWarps: one CTA per SM)
    if (pair && wide == kWideWarps)
      return reinterpret_cast<const void*>(k_scan<uint16_t, uint16_t, uint32_t, uint32_t, true, false, kWideWarps, kPairQueue, kWideWarps, true>);
    if (wide == 2) return reinterpret_cast<const void*>(k_scan<uint16_t, uint16_t, uint32_t, uint32_t, true, false, kWideWarps, kWideQueue, 2>);
    if (wide == 4) return reinterpret_cast<const void*>(k_scan<uint16_t, uint16_t, uint32_t, uint32_t, true, false, kWideWarps, kWideQueue, 4>);
    return reinterpret_cast<const void*>(k_scan<uint16_t, uint16_t, uint32_t, uint32_t, true, false, kWideWarps, kWideQueue>);
  }
  if (t.site_bytes == 2) {
    if (t.dist_bytes == 2) return acc32 ? scan_fn_acc<uint16_t, uint16_t, uint32_t>(G, ts) : scan_fn_acc<uint16_t, uint16_t, uint64_t>(G, ts);
    if (t.dist_bytes == 4) return acc32 ? scan_fn_acc<uint16_t, uint32_t, uint32_t>(G, ts) : scan_fn_acc<uint16_t, uint32_t, uint64_t>(G, ts);
    return acc32 ? scan_fn_acc<uint16_t, uint64_t, uint32_t>(G, ts) : scan_fn_acc<uint16_t, uint64_t, uint64_t>(G, ts);
  }
  if (t.dist_bytes == 2) return acc32 ? scan_fn_acc<uint32_t, uint16_t, uint32_t>(G, ts) : scan_fn_acc<uint32_t, uint16_t, uint64_t>(G, ts);
  if (t.dist_bytes == 4) return acc32 ? scan_fn_acc<uint32_t, uint32_t, uint32_t>(G, ts) : scan_fn_acc<uint32_t, uint32_t, uint64_t>(G, ts);
  return acc32 ? scan_fn_acc<uint32_t, uint64_t, uint32_t>(G, ts) : scan_fn_acc<uint32_t, uint64_t, uint64_t>(G, ts);
}

// The planner's tuning overrides (PMB_SCAN_*; A/B experiments and tests), read
// in one pass over the environment: plan_scan runs once per evaluation and
// six getenv calls cost ~1 us of host time each time.
struct ScanKnobs {
  const char* shape = nullptr;      // "G,warps[,ctas per SM]": pins the shape
  const char* wide = nullptr;       // "0": no many-warp variant
  const char* pair = nullptr;       // "0"/"1": column pairs off/on
  const char* coop = nullptr;       // clients per warp at which the cooperative tail starts
  const char* coopseg = nullptr;    // log2 of the most lanes per client in the tail
  const char* tailclaim = nullptr;  // clients left per warp below which claims shrink
  const char* split = nullptr;      // clients per CTA segment below which the split shapes are used
};

static ScanKnobs scan_knobs() {
  ScanKnobs k;
  for (char** e = environ; e && *e; ++e) {
    const char* v = *e;
    if (std::strncmp(v, "PMB_SCAN_", 9) != 0) continue;
    v += 9;
    const struct { const char* name; const char** out; } names[] = {
        {"SHAPE=", &k.shape}, {"WIDE=", &k.wide}, {"PAIR=", &k.pair},
        {"COOP=", &k.coop}, {"COOPSEG=", &k.coopseg}, {"TAILCLAIM=", &k.tailclaim}, {"SPLIT=", &k.split}};
    for (const auto& nm : names) {
      const size_t l = std::strlen(nm.name);
      if (std::strncmp(v, nm.name, l) == 0) *nm.out = v + l;
    }
  }
  return k;
}

ScanPlan plan_scan(const DevTables& t, size_t count, int sms, size_t max_smem, bool depth_mode) {
  const ScanKnobs knob = scan_knobs();
  ScanPlan sp;
  // (group width, warps per CTA, CTAs per SM, masks in smem?) in preference
  // order.  Measured on B200 (profiles/r01_ncu_kernels.md):
  // * 32-wide groups beat 64-wide at every BASELINE shape (64-wide doubles the
  //   mask and counter footprint and the per-lane hit bursts);
  // * a CTA must leave L1 room for the lanes' in-flight row prefetches --
  //   shared memory above ~200 KB halves throughput;
  // * when a CTA segment (its share of one group's clients) is short -- small
  //   n (pmed40) or few units per CTA (syn5k) -- the per-segment barriers leave
  //   warps idle, so the same 16 warps per SM run as 8 x 2 or 4 x 4 CTAs whose
  //   barriers overlap (pmed40 0.114 -> 0.082 ms, syn5k 0.181 -> 0.161 ms);
  //   with long segments (>= ~1350 clients per SM) the 24-warp CTA is faster.
  // The last entry reads the masks from global memory and always fits.
  const struct { int G, warps, cps; bool tsmem; } shapes[] = {
      {32, 2, 8, true}, {32, 4, 4, true}, {32, 8, 2, true},
      {32, 16, 1, true}, {32, 14, 1, true}, {32, 12, 1, true}, {32, 10, 1, true}, {32, 8, 1, true},
      {32, 6, 1, true},  {32, 4, 1, true},  {32, 8, 1, false}};
  const size_t chunk_bytes = (size_t)kChunk * (t.site_bytes + t.dist_bytes);
  const size_t l1_total = 228 * 1024;
  const unsigned long long vmax = depth_mode ? (unsigned long long)t.Wp : (unsigned long long)t.max_cost;
  // clients per CTA segment (a segment never crosses a group)
  const long long units_per_sm = ((long long)((count + 31) / 32) * t.n + sms - 1) / sms;
  // segments below ~1350 clients per SM (syn5k, the pmed40 shape, 256-chromosome
  // syn20k batches) run the split shapes; above it the 24-warp CTA wins
  // (syn20k 384-768 chromosomes: -4-6 %, profiles/r02_k2_ab.md)
  const long long split_below = knob.split ? std::atoll(knob.split) : 1350;
  const bool split = std::min<long long>(units_per_sm, t.n) < split_below;
  // PMB_SCAN_SHAPE="G,warps[,ctas per SM]" pins the shape (tuning experiments only)
  const char* force = knob.shape;
  int fG = 0, fW = 0, fC = 1;
  if (force) sscanf(force, "%d,%d,%d", &fG, &fW, &fC);
  for (const auto& sh0 : shapes) {
    auto sh = sh0;
    if (fG) {
      if (&sh0 != &shapes[0]) break;
      sh.G = fG;
      sh.warps = fW;
      sh.cps = std::max(1, fC);
      sh.tsmem = true;
    } else if (sh.cps > 1 && !split) {
      continue;
    }
    const int ctas = sms * sh.cps;
    const size_t groups = (count + sh.G - 1) / sh.G;
    const long long U = (long long)groups * t.n;
    const long long seg = (U + ctas - 1) / ctas;  // clients one lane counter can see (upper bound)
    for (int pass = 0; pass < 2; ++pass) {
      const bool acc32 =
          pass == 0 && (unsigned long long)std::min<long long>(seg, t.n) * vmax < (1ull << 32);
      if (pass == 0 && !acc32) continue;
      const size_t smem = scan_smem(t.m, sh.warps, acc32, sh.tsmem, sh.G);
      // shared memory of all CTAs on the SM (+1 KB reserved each) plus L1 room
      // for the in-flight row loads of all their warps
      const size_t inflight = (size_t)sh.cps * sh.warps * 32 * chunk_bytes / 2;
      const size_t resident = (size_t)sh.cps * (smem + 1024);
      if (smem <= max_smem && (fG || !sh.tsmem || resident + inflight <= l1_total)) {
        sp.G = sh.G;
        sp.tsmem = sh.tsmem;
        sp.warps = sh.warps;
        sp.acc32 = acc32;
        sp.smem = smem;
        sp.ctas = ctas;
        // long segments, narrow tables: the many-warp variant (24 warps, 80
        // registers, two row chunks in flight, a 256-record queue drained
        // mid-chunk when it could overflow) -- measured 7 % faster at syn20k
        // than 16 warps with three chunks (tools/wide_sweep.sh: 20-32 warps,
        // 64-256 records); PMB_SCAN_WIDE=0 turns it off
        const char* ew = knob.wide;
        if (!fG && !split && !(ew && ew[0] == '0') && sp.G == 32 && sp.tsmem && sp.acc32 && !depth_mode &&
            t.site_bytes == 2 && t.dist_bytes == 2) {
          const size_t sm2 = scan_smem(t.m, kWideWarps, true, true, 32, kWideQueue);
          if (sm2 <= max_smem) {
            sp.wide = kWideWarps;
            sp.warps = kWideWarps;
            sp.ctas = sms;
            sp.smem = sm2;
            // long walks (m >= 75 p: few open sites, so few hits per column):
            // column pairs -- one ballot and one 16-byte queue store per two
            // columns.  syn20k 1.41 -> 1.40 ms, sweep p=50 1.42 -> 1.31 ms,
            // p=100 0.78 -> 0.76 ms; at p >= 200 the extra empty records of
            // the denser hits cost more (0.46 -> 0.48 ms) (profiles/r02_k2_ab.md)
            const char* ep = knob.pair;
            sp.pair = ep ? ep[0] == '1' : (long long)t.m >= 75LL * std::max(t.p, 1);
            if (sp.pair) sp.smem = scan_smem(t.m, kWideWarps, true, true, 32, kPairQueue);
          }
        }
        // split shapes (short segments): the same variant as 12 x 2-warp (or
        // 6 x 4-warp) CTAs per SM when the CTAs' masks fit -- small m, e.g. the
        // paper's GA shape: pmed40 0.079 -> 0.074 ms (8-warp CTAs lose to the
        // 16-warp split shapes; tools/splitw_sweep.sh)
        if (!fG && split && !(ew && ew[0] == '0') && sp.G == 32 && sp.tsmem && sp.acc32 && !depth_mode &&
            t.site_bytes == 2 && t.dist_bytes == 2) {
          for (int cw : {2, 4}) {
            const size_t sm2 = scan_smem(t.m, cw, true, true, 32, kWideQueue);
            const int cps = kWideWarps / cw;
            if (sm2 <= max_smem && (size_t)cps * (sm2 + 1024) <= l1_total) {
              sp.wide = cw;
              sp.warps = cw;
              sp.ctas = sms * cps;
              sp.smem = sm2;
              break;
            }
          }
        }
        // cooperative tail (k_scan): a warp's last <= kCoop clients walk on
        // lane segments (profiles/r02_k2_ab.md; PMB_SCAN_COOP=<clients> and
        // PMB_SCAN_COOPSEG=<log2 most lanes per client> for A/B runs)
        const char* ec = knob.coop;
        const char* es = knob.coopseg;
        sp.coop = std::min(32, std::max(0, ec ? std::atoi(ec) : kCoop)) |
                  (std::min(5, std::max(0, es ? std::atoi(es) : 5)) << 8);
        const char* et = knob.tailclaim;  // clients left per warp (x warps)
        sp.tail_claim = (et ? std::atoi(et) : kTailClaim) * sp.warps;
        return sp;
      }
    }
  }
  sp.ctas = 0;
  return sp;
}

cudaError_t launch_scan(const DevTables& t, const ScanPlan& sp, const uint64_t* T, size_t count,
                        unsigned long long* costs_acc, unsigned long long* err_first_bad,
                        int depth_mode, cudaStream_t st) {
  g_depth = depth_mode != 0;
  const void* fn = scan_kernel_ptr(t, sp.acc32, sp.G, sp.tsmem, sp.wide, sp.pair);
  // raise the kernel's dynamic shared-memory cap only when it grows (the call
  // costs host time on every launch otherwise; the GA launches K2 ~10x per generation)
  static thread_local std::vector<std::pair<const void*, size_t>> raised;
  size_t* have = nullptr;
  for (auto& f : raised)
    if (f.first == fn) have = &f.second;
  cudaError_t e = cudaSuccess;
  if (!have || *have < sp.smem) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.smem);
    if (e != cudaSuccess) return e;
    if (have) *have = sp.smem;
    else raised.emplace_back(fn, sp.smem);
  }
  const int groups = (int)((count + sp.G - 1) / sp.G);
  const int ctas = (int)std::min<long long>(sp.ctas, (long long)groups * t.n);
  size_t Ts = scan_t_stride(t.m);
  const void* ord = t.ord;
  const void* dist = t.dist;
  int n = t.n, Wp = t.Wp, coop = sp.coop, tail_claim = sp.tail_claim;
  void* args[] = {(void*)&ord, (void*)&dist, (void*)&n, (void*)&Wp, (void*)&T, (void*)&Ts,
                  (void*)&count, (void*)&groups, (void*)&costs_acc, (void*)&err_first_bad, (void*)&coop,
                  (void*)&tail_claim};
  e = cudaLaunchKernel(fn, dim3(ctas), dim3(sp.warps * 32), args, sp.smem, st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---- measurement: per-(group, client) walk lengths ------------------------
//
// The scan's work per (32-chromosome group g, client i) is the row walk up to
// the column where the last of the group's chromosomes finds an open site:
// walk_gi = max_{c in g} k*_ic.  This kernel (measurement only -- never on the
// evaluation path) reports sum_i walk_gi per group and max_g walk_gi per
// client, from which bench.py derives the reuse-aware byte floors of the
// roofline: the bytes K2 must stream from L2 (sum over groups) and the bytes
// it must read from DRAM at least once (sum over clients of the maximum).
// One thread per (group, client); masks read from the transposed population.
template <class OrdT>
__global__ void __launch_bounds__(256) k_walks(const OrdT* __restrict__ ord, int n, int W, int Wp,
                                               const uint64_t* __restrict__ T, size_t Ts, size_t count,
                                               unsigned long long* __restrict__ group_sum,
                                               unsigned int* __restrict__ client_max) {
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int groups = (int)((count + 31) / 32);
  int walk = 0, g = 0;
  if (u < (long long)groups * n) {
    g = (int)(u / n);
    const int i = (int)(u % n);
    const uint64_t* Tg = T + (size_t)(g / 2) * Ts;
    const int half = (g & 1) * 32;
    const size_t nvalid = min((size_t)32, count - (size_t)g * 32);
    uint32_t alive = nvalid == 32 ? ~0u : ((1u << nvalid) - 1);
    const OrdT* row = ord + (size_t)i * Wp;
    int k = 0;
    for (; k < W && alive; ++k) alive &= ~(uint32_t)(__ldg(Tg + row[k]) >> half);
    walk = k;
    atomicMax(client_max + i, (unsigned)walk);
  }
  // lanes of a warp mostly share a group: one atomic per (warp, group) run
  const int g0 = __shfl_sync(kFull, g, 0);
  const bool same = __all_sync(kFull, g == g0 || u >= (long long)groups * n);
  if (same) {
    const unsigned long long s = warp_sum((unsigned long long)walk);
    if (lane_id() == 0 && s) atomicAdd(group_sum + g0, s);
  } else if (walk) {
    atomicAdd(group_sum + g, (unsigned long long)walk);
  }
}

cudaError_t launch_walks(const DevTables& t, const uint64_t* T, size_t count, unsigned long long* group_sum,
                         unsigned int* client_max, cudaStream_t st) {
  const long long units = (long long)((count + 31) / 32) * t.n;
  const unsigned blocks = (unsigned)((units + 255) / 256);
  if (t.site_bytes == 2)
    k_walks<uint16_t><<<blocks, 256, 0, st>>>((const uint16_t*)t.ord, t.n, t.W, t.Wp, T, scan_t_stride(t.m),
                                               count, group_sum, client_max);
  else
    k_walks<uint32_t><<<blocks, 256, 0, st>>>((const uint32_t*)t.ord, t.n, t.W, t.Wp, T, scan_t_stride(t.m),
                                               count, group_sum, client_max);
  return cudaGetLastError();
}

}  // namespace pmb
