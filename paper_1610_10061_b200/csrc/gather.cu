// K2b: gather-min population fitness (instance.cpp:32-48), and the open-site
// lists it reads.
//
// fitness = sum_i min_{j open} cost(i, j) (equal to the scan of
// ordering.cpp:40-59 by acceptance.cpp:86-116).  A thread owns 16 bytes of
// consecutive clients (8 at u16 costs); each open site j of a chromosome is
// one 16-byte read of the site-major row dT[j][i0..] and a packed min.  Wins
// when p is small (the scan reads ~m/p columns per client, the gather p):
// AUTO picks the scan iff p >= 1.1 sqrt(m), measured.  The reference's
// scan-width contract (ordering.cpp:50-52) is enforced exactly: with popcount
// >= p it cannot fail (W = m-p+1 columns always contain one of p distinct
// sites); with fewer open sites the (cost, site)-smallest open site must not
// sort after column W-1.  A separate translation unit from the scan (K2,
// fitness.cu): the two kernels want different ptxas register heuristics.
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pmb {

// ---- K2b: gather-min -----------------------------------------------------------

// One warp per chromosome: compact the open sites (< m) into a list.
__global__ void __launch_bounds__(256) k_open_lists(const uint64_t* __restrict__ words, size_t count,
                                                    int wp, int m, uint32_t* __restrict__ lists,
                                                    uint32_t* __restrict__ counts, int cap,
                                                    unsigned long long* __restrict__ costs,
                                                    unsigned long long* __restrict__ err_init) {
  // the call's error word starts at "none" (replaces a memset; the gather runs after)
  if (err_init && blockIdx.x == 0 && threadIdx.x == 0) *err_init = ~0ull;
  const size_t c = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= count) return;
  const int lane = threadIdx.x & 31;
  if (lane == 0) costs[c] = 0;  // the gather accumulates into costs (replaces a memset launch)
  const unsigned lt = lanemask_lt();
  const uint64_t* w = words + c * wp;
  uint32_t* list = lists + c * (size_t)cap;
  uint32_t total = 0;
  for (int w0 = 0; w0 < wp; w0 += 32) {
    const int wi = w0 + lane;
    uint64_t x = wi < wp ? w[wi] : 0;
    if (wi == wp - 1 && (m & 63)) x &= (1ull << (m & 63)) - 1;  // bits >= m are not sites
    const uint32_t pc = __popcll(x);
    uint32_t incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t pos = total + incl - pc;
    while (x) {
      const int b = __ffsll((long long)x) - 1;
      x &= x - 1;
      if (pos < (uint32_t)cap) list[pos] = (uint32_t)(wi * 64 + b);
      ++pos;
    }
    total += __shfl_sync(kFull, incl, 31);
    (void)lt;
  }
  if (lane == 0) counts[c] = total;
}

constexpr int kGatherThreads = 256;

// V consecutive clients per thread through one 16-byte load per open site.
template <class DistT>
struct GVec {
  static constexpr int V = 16 / sizeof(DistT);
  uint4 v;
  __device__ __forceinline__ void set_max() { v = make_uint4(~0u, ~0u, ~0u, ~0u); }
  __device__ __forceinline__ void min_with(const uint4 o) {
    if constexpr (sizeof(DistT) == 2) {
      v.x = __vminu2(v.x, o.x);
      v.y = __vminu2(v.y, o.y);
      v.z = __vminu2(v.z, o.z);
      v.w = __vminu2(v.w, o.w);
    } else if constexpr (sizeof(DistT) == 4) {
      v.x = min(v.x, o.x);
      v.y = min(v.y, o.y);
      v.z = min(v.z, o.z);
      v.w = min(v.w, o.w);
    } else {
      const uint64_t a0 = (uint64_t)v.x | ((uint64_t)v.y << 32), b0 = (uint64_t)o.x | ((uint64_t)o.y << 32);
      const uint64_t a1 = (uint64_t)v.z | ((uint64_t)v.w << 32), b1 = (uint64_t)o.z | ((uint64_t)o.w << 32);
      const uint64_t m0 = a0 < b0 ? a0 : b0, m1 = a1 < b1 ? a1 : b1;
      v = make_uint4((uint32_t)m0, (uint32_t)(m0 >> 32), (uint32_t)m1, (uint32_t)(m1 >> 32));
    }
  }
  __device__ __forceinline__ uint64_t elem(int q) const {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
    if constexpr (sizeof(DistT) == 2) return (w[q >> 1] >> ((q & 1) * 16)) & 0xffffu;
    else if constexpr (sizeof(DistT) == 4) return w[q];
    else return (uint64_t)w[2 * q] | ((uint64_t)w[2 * q + 1] << 32);
  }
};

// Register budget (A/B switch): ptxas keeps 32 registers at the default
// budget and issues the 8 client-vector loads as two halves; forcing 64 / 80 /
// 94 registers (minimum 4 / 3 / 2 CTAs per SM) keeps all 8 in flight but loses
// occupancy and measured slower at every shape (pmed40 0.213 -> 0.24-0.36 ms).
#ifndef PMB_GATHER_MINB
#define PMB_GATHER_MINB 0
#endif
template <class DistT, class OrdT>
__global__ void __launch_bounds__(kGatherThreads, PMB_GATHER_MINB)
    k_gather(const DistT* __restrict__ dT, int nP, const OrdT* __restrict__ ord,
             const DistT* __restrict__ dist, int n, int m, int p, int W, int Wp,
             const uint64_t* __restrict__ words, int wp, const uint32_t* __restrict__ lists,
             const uint32_t* __restrict__ counts, int cap, size_t count, int chunk,
             unsigned long long* __restrict__ costs, unsigned long long* __restrict__ err, int mode) {
  using Vec = GVec<DistT>;
  constexpr int V = Vec::V;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* part = reinterpret_cast<unsigned long long*>(smem);  // [warps][chunk]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kGatherThreads / 32;
  const int i0 = (blockIdx.x * kGatherThreads + tid) * V;  // first client of this thread
  const int nv = i0 < n ? min(V, n - i0) : 0;               // real clients among the V
  const DistT* col = dT + i0;
  // chromosome chunks stride over gridDim.y (<= 65535): any population size launches
  for (size_t cbase = (size_t)blockIdx.y * chunk; cbase < count; cbase += (size_t)gridDim.y * chunk) {
  const int cn = (int)min((size_t)chunk, count - cbase);
  for (int cl = 0; cl < cn; ++cl) {
    const size_t c = cbase + cl;
    const uint32_t pc = counts[c];
    unsigned long long sum = 0;
    if (pc == 0) {
      if (tid == 0 && blockIdx.x == 0) atomicMin(err, (unsigned long long)c);
    } else if (pc <= (uint32_t)cap && !(mode == 0 && pc < (uint32_t)p)) {
      // common case: min over the open list, V clients per 16-byte load
      Vec best;
      best.set_max();
      if (nv > 0) {
        const uint32_t* list = lists + c * (size_t)cap;
        uint32_t t = 0;
        PMB_CHECK(i0 + V <= nP && pc <= (uint32_t)cap);
        // 8 open sites per step: their indices arrive as two 16-byte loads
        // (lists are 16-byte aligned, cap % 4 == 0) and the 8 client-vector
        // loads are all in flight before the first min (the kernel is bound by
        // L2 latency, not bandwidth)
        for (; t + 8 <= pc; t += 8) {
          const uint4 ja = __ldg(reinterpret_cast<const uint4*>(list + t));
          const uint4 jb = __ldg(reinterpret_cast<const uint4*>(list + t + 4));
          const uint32_t js[8] = {ja.x, ja.y, ja.z, ja.w, jb.x, jb.y, jb.z, jb.w};
          uint4 x[8];
#ifdef PMB_BOUNDS
          for (int u = 0; u < 8; ++u) PMB_CHECK(js[u] < (uint32_t)m);
#endif
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const uint4*>(col + (size_t)js[u] * nP));
#pragma unroll
          for (int u = 0; u < 8; ++u) best.min_with(x[u]);
        }
        if (t + 4 <= pc) {
          const uint4 ja = __ldg(reinterpret_cast<const uint4*>(list + t));
          const uint32_t js[4] = {ja.x, ja.y, ja.z, ja.w};
          uint4 x[4];
#ifdef PMB_BOUNDS
          for (int u = 0; u < 4; ++u) PMB_CHECK(js[u] < (uint32_t)m);
#endif
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = __ldg(reinterpret_cast<const uint4*>(col + (size_t)js[u] * nP));
#pragma unroll
          for (int u = 0; u < 4; ++u) best.min_with(x[u]);
          t += 4;
        }
        for (; t < pc; ++t) best.min_with(__ldg(reinterpret_cast<const uint4*>(col + (size_t)__ldg(list + t) * nP)));
#pragma unroll
        for (int q = 0; q < V; ++q)
          if (q < nv) sum += best.elem(q);
      }
    } else {
      // general path: walk the words in site order, track the (cost, site)
      // minimum per client and, under the fitness contract with fewer than p
      // open sites, check it sorts within the first W columns (ordering.cpp:50-52).
      bool bad = false;
      for (int q = 0; q < nv; ++q) {
        const int i = i0 + q;
        uint64_t best = ~0ull;
        uint32_t bj = 0;
        const uint64_t* w = words + c * wp;
        for (int wi = 0; wi < wp; ++wi) {
          uint64_t x = __ldg(w + wi);
          if (wi == wp - 1 && (m & 63)) x &= (1ull << (m & 63)) - 1;
          while (x) {
            const uint32_t j = wi * 64 + (__ffsll((long long)x) - 1);
            x &= x - 1;
            const uint64_t v = (uint64_t)dT[(size_t)j * nP + i];
            if (v < best) {  // strict: ascending j keeps the lowest site on ties
              best = v;
              bj = j;
            }
          }
        }
        sum += best;
        if (mode == 0 && pc < (uint32_t)p) {
          const uint64_t dlast = (uint64_t)dist[(size_t)i * Wp + (W - 1)];
          const uint32_t jlast = (uint32_t)ord[(size_t)i * Wp + (W - 1)];
          bad |= !(best < dlast || (best == dlast && bj <= jlast));
        }
      }
      if (__any_sync(kFull, bad) && lane == 0) atomicMin(err, (unsigned long long)c);
    }
    sum = warp_sum(sum);
    if (lane == 0) part[warp * chunk + cl] = sum;
  }
  __syncthreads();
  for (int cl = tid; cl < cn; cl += kGatherThreads) {
    unsigned long long s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += part[w * chunk + cl];
    atomicAdd(&costs[cbase + cl], s);
  }
  __syncthreads();  // `part` is rewritten by the next chunk
  }
}

// ---- K2b fused: lists in shared memory, one launch ---------------------------
//
// The same gather-min with the open-site list built by each CTA in shared
// memory (a block scan over the chromosome's words; u16 entries) and no zeroed
// cost array: a work item is (chromosome, slab of <= 1024 x V clients).  With
// one slab the CTA stores the chromosome's cost; with several, each stores its
// partial sum and the last slab to arrive (threadfence + a per-chromosome
// counter it resets) adds them and stores the cost.  Errors go to a context
// word that stays "none" between calls: CTAs atomicMin into it, and the last
// CTA to finish (threadfence + arrival counter, reset by that CTA) hands the
// value to the call's error word -- a store for a host call's per-chunk slot, a
// min into the sticky context word -- and re-arms it.
template <class DistT, class OrdT>
__global__ void __launch_bounds__(1024, 2)  // <= 32 registers: three 640-thread CTAs per SM at syn5k
    k_gather_fused(const DistT* __restrict__ dT, int nP, const OrdT* __restrict__ ord,
                   const DistT* __restrict__ dist, int n, int m, int p, int W, int Wp,
                   const uint64_t* __restrict__ words, int wp, size_t count, int nslab,
                   unsigned long long* __restrict__ costs, unsigned long long* partial, unsigned int* arrive,
                   unsigned long long* err_work, unsigned int* done, unsigned long long* err_out, int err_store,
                   int mode) {
  using Vec = GVec<DistT>;
  constexpr int V = Vec::V;
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* list = reinterpret_cast<uint16_t*>(smem);  // the open sites, ascending (m <= 65535)
  __shared__ unsigned long long red[32];
  __shared__ uint32_t wtot[32];
  __shared__ int anybad, last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const size_t items = count * (size_t)nslab;
  for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
    const size_t c = it / nslab;
    const int slab = (int)(it % nslab);
    const int i0 = (slab * (int)blockDim.x + tid) * V;  // first client of this thread
    const int nv = i0 < n ? min(V, n - i0) : 0;
    const DistT* col = dT + i0;
    // 1. the open-site list: a block scan of the words' popcounts
    const uint64_t* w = words + c * wp;
    uint32_t total = 0;
    if (tid == 0) anybad = 0;
    for (int w0 = 0; w0 < wp; w0 += blockDim.x) {
      const int wi = w0 + tid;
      uint64_t x = wi < wp ? __ldg(w + wi) : 0;
      if (wi == wp - 1 && (m & 63)) x &= (1ull << (m & 63)) - 1;  // bits >= m are not sites
      const uint32_t pc = __popcll(x);
      uint32_t incl = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wtot[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const uint32_t v = lane < nwarps ? wtot[lane] : 0;
        uint32_t wi2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, wi2, o);
          if (lane >= o) wi2 += t;
        }
        if (lane < nwarps) wtot[lane] = wi2 - v;  // exclusive warp offsets
        if (lane == 31) red[0] = wi2;           // this pass's total
      }
      __syncthreads();
      uint32_t pos = total + wtot[warp] + incl - pc;
      while (x) {
        list[pos++] = (uint16_t)(wi * 64 + __ffsll((long long)x) - 1);
        x &= x - 1;
      }
      total += (uint32_t)red[0];
      __syncthreads();
    }
    // 2. this slab's share of the chromosome's cost
    unsigned long long sum = 0;
    bool bad = false;
    if (total == 0) {
      bad = true;  // no open site at all
    } else if (!(mode == 0 && total < (uint32_t)p)) {
      // common case: min over the list, V clients per 16-byte load, 8 in flight
      Vec best;
      best.set_max();
      if (nv > 0) {
        uint32_t t = 0;
        for (; t + 8 <= total; t += 8) {
          const uint4 jv = *reinterpret_cast<const uint4*>(list + t);  // 8 u16 site indices
          const uint32_t js[8] = {jv.x & 0xffffu, jv.x >> 16, jv.y & 0xffffu, jv.y >> 16,
                                  jv.z & 0xffffu, jv.z >> 16, jv.w & 0xffffu, jv.w >> 16};
          uint4 xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) xv[u] = __ldg(reinterpret_cast<const uint4*>(col + (size_t)js[u] * nP));
#pragma unroll
          for (int u = 0; u < 8; ++u) best.min_with(xv[u]);
        }
        for (; t < total; ++t) best.min_with(__ldg(reinterpret_cast<const uint4*>(col + (size_t)list[t] * nP)));
#pragma unroll
        for (int q = 0; q < V; ++q)
          if (q < nv) sum += best.elem(q);
      }
    } else {
      // fewer than p open sites under the fitness contract: the (cost, site)
      // smallest open site (ascending list, strict <: the lowest site on ties)
      // must not sort after column W-1 (ordering.cpp:50-52)
      for (int q = 0; q < nv; ++q) {
        const int i = i0 + q;
        uint64_t bv = ~0ull;
        uint32_t bj = 0;
        for (uint32_t t = 0; t < total; ++t) {
          const uint32_t j = list[t];
          const uint64_t v = (uint64_t)dT[(size_t)j * nP + i];
          if (v < bv) {
            bv = v;
            bj = j;
          }
        }
        sum += bv;
        const uint64_t dlast = (uint64_t)dist[(size_t)i * Wp + (W - 1)];
        const uint32_t jlast = (uint32_t)ord[(size_t)i * Wp + (W - 1)];
        bad |= !(bv < dlast || (bv == dlast && bj <= jlast));
      }
    }
    // 3. block sum; the cost (or this slab's part of it) is stored, a failure
    // reported by whichever slab sees it
    sum = warp_sum(sum);
    if (__any_sync(kFull, bad) && lane == 0) anybad = 1;
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
      for (int x = 0; x < nwarps; ++x) s += red[x];
      if (anybad) atomicMin(err_work, (unsigned long long)c);
      if (nslab == 1) {
        costs[c] = s;
      } else {
        partial[it] = s;
        __threadfence();
        last = atomicAdd(arrive + c, 1u) == (unsigned)nslab - 1;
        if (last) {
          __threadfence();
          unsigned long long tot = 0;
          for (int k = 0; k < nslab; ++k) tot += *(volatile unsigned long long*)(partial + c * nslab + k);
          costs[c] = tot;
          arrive[c] = 0;  // re-armed for the next call
        }
      }
    }
    __syncthreads();  // list, red and the flags are rewritten for the next item
  }
  // 4. the last CTA hands the error word over and re-arms it
  if (tid == 0) {
    __threadfence();
    const unsigned t = atomicAdd(done, 1u);
    if (t == gridDim.x - 1) {
      __threadfence();
      const unsigned long long v = atomicExch(err_work, ~0ull);
      *done = 0;
      if (err_store) *err_out = v;
      else if (v != ~0ull) atomicMin(err_out, v);
    }
  }
}

// Work split: threads per CTA and client slabs per chromosome (balanced slabs
// of at most 1024 threads).
static void fused_split(const DevTables& t, int* threads, int* nslab) {
  const int V = 16 / t.dist_bytes;
  const int tn = (t.n + V - 1) / V;
  *nslab = (tn + 1023) / 1024;
  *threads = ((tn + *nslab - 1) / *nslab + 31) / 32 * 32;
}

int gather_fused_slabs(const DevTables& t) {
  int th, ns;
  fused_split(t, &th, &ns);
  return ns;
}

template <class DistT, class OrdT>
static cudaError_t launch_gather_fused_t(const DevTables& t, const uint64_t* words, size_t count, int wp,
                                         unsigned long long* costs, unsigned long long* partial,
                                         unsigned int* arrive, unsigned long long* err_work, unsigned int* done,
                                         unsigned long long* err_out, int err_store, int mode, int sms,
                                         cudaStream_t st) {
  int threads, nslab;
  fused_split(t, &threads, &nslab);
  const size_t smem = ((size_t)t.m + 16) * 2;
  auto kern = k_gather_fused<DistT, OrdT>;
  static thread_local size_t raised = 0;
  if (smem > 48 * 1024 && smem > raised) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    raised = smem;
  }
  const int per_sm = std::max(1, std::min(2048 / threads, (int)((200u << 10) / (smem + 1024))));
  const unsigned grid = (unsigned)std::min<size_t>(count * nslab, (size_t)sms * per_sm * 4);
  kern<<<grid, threads, smem, st>>>((const DistT*)t.dT, t.nP, (const OrdT*)t.ord, (const DistT*)t.dist, t.n, t.m,
                                    t.p, t.W, t.Wp, words, wp, count, nslab, costs, partial, arrive, err_work,
                                    done, err_out, err_store, mode);
  return cudaGetLastError();
}

bool gather_fused_fits(const DevTables& t) { return t.m <= 65535; }

cudaError_t launch_gather_fused(const DevTables& t, const uint64_t* words, size_t count, int words_per,
                                unsigned long long* costs, unsigned long long* partial, unsigned int* arrive,
                                unsigned long long* err_work, unsigned int* done, unsigned long long* err_out,
                                int err_store, int mode, int sms, cudaStream_t st) {
#define PMB_FUSED(D, O) \
  return launch_gather_fused_t<D, O>(t, words, count, words_per, costs, partial, arrive, err_work, done, err_out, \
                                     err_store, mode, sms, st)
  if (t.site_bytes == 2) {
    if (t.dist_bytes == 2) PMB_FUSED(uint16_t, uint16_t);
    if (t.dist_bytes == 4) PMB_FUSED(uint32_t, uint16_t);
    PMB_FUSED(uint64_t, uint16_t);
  }
  if (t.dist_bytes == 2) PMB_FUSED(uint16_t, uint32_t);
  if (t.dist_bytes == 4) PMB_FUSED(uint32_t, uint32_t);
  PMB_FUSED(uint64_t, uint32_t);
#undef PMB_FUSED
}

template <class DistT, class OrdT>
static cudaError_t launch_gather_t(const DevTables& t, const uint64_t* words, size_t count, int wp,
                                   const uint32_t* lists, const uint32_t* counts, int cap,
                                   unsigned long long* costs, unsigned long long* err, int mode,
                                   int sms, cudaStream_t st) {
  constexpr int V = 16 / sizeof(DistT);
  const int xblocks = (t.n + kGatherThreads * V - 1) / (kGatherThreads * V);
  // enough CTAs for ~8 resident CTAs per SM
  const long long want = (long long)sms * 8;
  const int chunk = (int)std::max<long long>(1, std::min<long long>(256, (long long)count * xblocks / want));
  const unsigned yblocks = (unsigned)std::min<size_t>((count + chunk - 1) / chunk, 65535);
  const size_t smem = (size_t)(kGatherThreads / 32) * chunk * 8;
  k_gather<DistT, OrdT><<<dim3(xblocks, yblocks), kGatherThreads, smem, st>>>(
      (const DistT*)t.dT, t.nP, (const OrdT*)t.ord, (const DistT*)t.dist, t.n, t.m, t.p, t.W, t.Wp, words,
      wp, lists, counts, cap, count, chunk, costs, err, mode);
  return cudaGetLastError();
}

cudaError_t launch_open_lists(const uint64_t* words, size_t count, int words_per, int m,
                              uint32_t* open_lists, uint32_t* open_counts, int open_cap,
                              unsigned long long* costs, unsigned long long* err_init, cudaStream_t st) {
  k_open_lists<<<(unsigned)((count + 7) / 8), 256, 0, st>>>(words, count, words_per, m, open_lists,
                                                             open_counts, open_cap, costs, err_init);
  return cudaGetLastError();
}

cudaError_t launch_gather(const DevTables& t, const uint64_t* words, size_t count, int words_per,
                          uint32_t* open_lists, uint32_t* open_counts, int open_cap,
                          unsigned long long* costs_acc, unsigned long long* err_first_bad, int mode,
                          int sms, cudaStream_t st) {
  if (t.site_bytes == 2) {
    if (t.dist_bytes == 2) return launch_gather_t<uint16_t, uint16_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
    if (t.dist_bytes == 4) return launch_gather_t<uint32_t, uint16_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
    return launch_gather_t<uint64_t, uint16_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
  }
  if (t.dist_bytes == 2) return launch_gather_t<uint16_t, uint32_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
  if (t.dist_bytes == 4) return launch_gather_t<uint32_t, uint32_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
  return launch_gather_t<uint64_t, uint32_t>(t, words, count, words_per, open_lists, open_counts, open_cap, costs_acc, err_first_bad, mode, sms, st);
}

}  // namespace pmb
