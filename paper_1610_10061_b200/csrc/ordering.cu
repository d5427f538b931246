// K1: device construction of the ordering tables.
//
// Replaces pmedian::build_ordering (/root/reference/proj/src/ordering.cpp:10-38):
// per client row, order the sites by (cost, site index) ascending -- the
// reference's comparator with its lower-index tie-break (ordering.cpp:25-28) --
// and keep the first W = m - p + 1 columns (ordering.cpp:17).
//
// Device layout (row-major, row stride Wp = round_up(W, 16) elements):
//   ord[i][k]  = pi_ik             (OrdT = u16 when m < 65535, else u32)
//   dist[i][k] = cost(i, pi_ik)    (DistT = u16 / u32 / u64 by max cost)
//   columns k in [W, Wp) hold the sentinel site m (never open) and cost 0.
// The reference stores first differences (increments, ordering.cpp:29-35); we
// store their prefix sums -- the sorted row itself -- because the fitness scan
// only ever needs the prefix sum up to the stopping column, which equals
// dist[i][k*] exactly (pinned by proj/tests/test_formulation.cpp:63-83).
// pm_get_tables re-derives the reference's increments for parity checks.
//
// Algorithm: one CTA per row (persistent over rows), a stable LSD radix sort
// over the cost bits only.  Rows start in site order and every pass is stable,
// so equal costs keep ascending site order: exactly the reference's order.
// Keys are packed (cost << sitebits | site) into u32 or u64 when they fit, so
// the site rides along for free; otherwise the u64 cost is the key and the site
// a separate payload.  Ranking within a 1024-element tile uses __match_any_sync
// per warp plus a per-digit exclusive scan across warps.
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace pmb {

// ---- validation scan: max cost and negativity (instance.cpp:20-24) --------

__global__ void k_validate_costs(const int64_t* __restrict__ costs, size_t count,
                             unsigned long long* __restrict__ out_max, int* __restrict__ out_neg) {
  int64_t mx = 0;
  int neg = 0;
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < count;
       x += (size_t)gridDim.x * blockDim.x) {
    const int64_t c = costs[x];
    neg |= c < 0;
    mx = c > mx ? c : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t v = __shfl_xor_sync(kFull, mx, o);
    mx = v > mx ? v : mx;
  }
  neg = __any_sync(kFull, neg);
  if (lane_id() == 0) {
    atomicMax(out_max, (unsigned long long)mx);
    if (neg) atomicOr(out_neg, 1);
  }
}

// ---- one pass over the int64 matrix: validation + the narrow copies ------
//
// Instance validation (instance.cpp:20-29: max cost, negativity) fused with
// the two narrow copies the device path keeps, written speculatively at u16
// (valid when the max cost fits, which the host checks from the same pass):
//   c16[i][j] = cost(i, j), row stride mP = round_up(m, 8) -- K1's input, a
//               quarter of the int64 bytes, 16-byte vector loads per row;
//   dT[j][i]  = cost(i, j), row stride nP -- the gather kernel's site-major table.
// So the 8-byte matrix is read from HBM once (previously three times:
// validation, K1, transpose).  32 x 32 tiles through shared memory; a
// persistent grid keeps one max / flag per CTA.
__global__ void __launch_bounds__(256) k_prep_costs(const int64_t* __restrict__ costs, int n, int m, int mP, int nP,
                                                    uint16_t* __restrict__ c16, uint16_t* __restrict__ dT,
                                                    unsigned long long* __restrict__ out_max,
                                                    int* __restrict__ out_neg) {
  // 64 rows x 32 columns per tile: 8 independent 8-byte loads per thread in
  // flight (enough bytes in flight per SM to stream HBM)
  constexpr int kR = 64;
  __shared__ uint16_t tile[kR][34];  // 17 words per row: transposed reads hit distinct banks
  __shared__ unsigned long long smax[8];
  __shared__ int sneg[8];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tilesX = (m + 31) / 32, tilesY = (nP + kR - 1) / kR;
  const long long total = (long long)tilesX * tilesY;
  int64_t mx = 0;
  int neg = 0;
  for (long long t = blockIdx.x; t < total; t += gridDim.x) {
    const int i0 = (int)(t / tilesX) * kR, j0 = (int)(t % tilesX) * 32;
    const int j = j0 + tx;
    int64_t v[kR / 8];
#pragma unroll
    for (int q = 0; q < kR / 8; ++q) {
      const int i = i0 + ty + 8 * q;
      v[q] = (i < n && j < m) ? __ldg(costs + (size_t)i * m + j) : 0;
    }
#pragma unroll
    for (int q = 0; q < kR / 8; ++q) {
      const int r = ty + 8 * q, i = i0 + r;
      mx = v[q] > mx ? v[q] : mx;
      neg |= v[q] < 0;
      const uint16_t u = (uint16_t)v[q];
      if (i < n && j < m) c16[(size_t)i * mP + j] = u;
      tile[r][tx] = u;
    }
    __syncthreads();
    // transposed: 32 sites x 64 clients, two clients per thread (4-byte stores)
    for (int r = ty; r < 32; r += 8) {
      const int jj = j0 + r, i = i0 + 2 * tx;
      if (jj < m && i < nP) {
        const uint32_t pair = (uint32_t)tile[2 * tx][r] | ((uint32_t)tile[2 * tx + 1][r] << 16);
        *reinterpret_cast<uint32_t*>(dT + (size_t)jj * nP + i) = pair;  // nP % 16 == 0, i even
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t v = __shfl_xor_sync(kFull, mx, o);
    mx = v > mx ? v : mx;
  }
  neg = __any_sync(kFull, neg);
  if (tx == 0) {
    smax[ty] = (unsigned long long)mx;
    sneg[ty] = neg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    int ng = 0;
    for (int w = 0; w < 8; ++w) {
      b = smax[w] > b ? smax[w] : b;
      ng |= sneg[w];
    }
    atomicMax(out_max, b);
    if (ng) atomicOr(out_neg, 1);
  }
}

// ---- K1: per-row stable radix sort ----------------------------------------

constexpr int kSortThreads = 1024;
static_assert(kSortThreads == 1024, "the digit scan assumes 32 warps");
constexpr int kHistPitch = 33;  // padded [digit][warp] so leaders of one warp hit distinct banks

template <class KeyT, bool kPayload>
__device__ __forceinline__ unsigned digit_of(KeyT key, int shift) {
  return (unsigned)(key >> shift) & 0xffu;
}

template <class KeyT, bool kPayload, class OrdT, class DistT, bool kSmem>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_build_rows(const int64_t* __restrict__ costs, int n, int m, int W, int Wp, int sitebits,
                 int npasses, OrdT* __restrict__ ord, DistT* __restrict__ dist,
                 KeyT* __restrict__ gkeys, uint32_t* __restrict__ gpay) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bucket = reinterpret_cast<uint32_t*>(smem);  // 256
  uint32_t* tcount = bucket + 256;                      // 256
  uint32_t* wh = tcount + 256;                          // 256 * kHistPitch
  int* flag = reinterpret_cast<int*>(wh + 256 * kHistPitch);
  unsigned char* bufbase = smem + ((256 + 256 + 256 * kHistPitch + 4) * 4 + 15) / 16 * 16;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  KeyT *A, *B;
  uint32_t *PA = nullptr, *PB = nullptr;
  if constexpr (kSmem) {
    A = reinterpret_cast<KeyT*>(bufbase);
    B = A + m;
    if constexpr (kPayload) {
      PA = reinterpret_cast<uint32_t*>(B + m);
      PB = PA + m;
    }
  } else {
    A = gkeys + (size_t)blockIdx.x * 2 * m;
    B = A + m;
    if constexpr (kPayload) {
      PA = gpay + (size_t)blockIdx.x * 2 * m;
      PB = PA + m;
    }
  }
  const unsigned lt = lanemask_lt();
  const KeyT sitemask = kPayload ? KeyT(0) : ((KeyT(1) << sitebits) - 1);
  const int shift0 = kPayload ? 0 : sitebits;

  for (int x = tid; x < 256 * kHistPitch; x += kSortThreads) wh[x] = 0;

  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const int64_t* crow = costs + (size_t)r * m;
    KeyT* src = A;
    KeyT* dst = B;
    uint32_t* psrc = PA;
    uint32_t* pdst = PB;
    if (tid < 256) bucket[tid] = 0;
    __syncthreads();
    for (int x = tid; x < m; x += kSortThreads) {
      const uint64_t c = (uint64_t)crow[x];
      KeyT key;
      if constexpr (kPayload) {
        key = (KeyT)c;
        psrc[x] = (uint32_t)x;
      } else {
        key = ((KeyT)c << sitebits) | (KeyT)x;
      }
      src[x] = key;
      if (npasses > 0) atomicAdd(&bucket[digit_of<KeyT, kPayload>(key, shift0)], 1u);
    }
    __syncthreads();

    for (int q = 0; q < npasses; ++q) {
      const int shift = shift0 + 8 * q;
      if (q > 0) {
        if (tid < 256) bucket[tid] = 0;
        __syncthreads();
        for (int x = tid; x < m; x += kSortThreads)
          atomicAdd(&bucket[digit_of<KeyT, kPayload>(src[x], shift)], 1u);
        __syncthreads();
      }
      // A pass whose digit is constant over the row is the identity: skip it.
      const bool skip = bucket[digit_of<KeyT, kPayload>(src[0], shift)] == (uint32_t)m;
      if (skip) continue;  // uniform across the CTA
      if (warp == 0) {     // exclusive scan of the 256 digit counts
        uint32_t v[8], s = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = bucket[lane * 8 + j];
          s += v[j];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        uint32_t run = incl - s;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          bucket[lane * 8 + j] = run;
          run += v[j];
        }
      }
      __syncthreads();

      for (int t0 = 0; t0 < m; t0 += kSortThreads) {
        const int x = t0 + tid;
        const bool valid = x < m;
        const KeyT key = valid ? src[x] : KeyT(0);
        const uint32_t pay = (kPayload && valid) ? psrc[x] : 0u;
        const unsigned d = valid ? digit_of<KeyT, kPayload>(key, shift) : 256u;
        const unsigned peers = __match_any_sync(kFull, d);
        const unsigned rank = __popc(peers & lt);
        if (valid && rank == 0) wh[d * kHistPitch + warp] = __popc(peers);
        __syncthreads();
        // per digit: exclusive prefix over warps (warp w owns digits w, w+32, ...)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int dd = warp + 32 * j;
          const uint32_t v = wh[dd * kHistPitch + lane];
          uint32_t incl = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
          }
          wh[dd * kHistPitch + lane] = incl - v;
          if (lane == 31) tcount[dd] = incl;
        }
        __syncthreads();
        if (valid) {
          const uint32_t pos = bucket[d] + wh[d * kHistPitch + warp] + rank;
          dst[pos] = key;
          if constexpr (kPayload) pdst[pos] = pay;
        }
        __syncthreads();
        // the scan wrote prefixes into every (digit, warp) cell: clear the
        // cells this warp scanned so the next tile starts from zero counts
#pragma unroll
        for (int j = 0; j < 8; ++j) wh[(warp + 32 * j) * kHistPitch + lane] = 0;
        if (tid < 256) bucket[tid] += tcount[tid];
        // the cells cleared above belong to other warps' columns, which those
        // warps write again in the next tile: finish every clear first
        __syncthreads();
      }
      __syncthreads();
      KeyT* tk = src;
      src = dst;
      dst = tk;
      uint32_t* tp = psrc;
      psrc = pdst;
      pdst = tp;
    }

    OrdT* orow = ord + (size_t)r * Wp;
    DistT* drow = dist + (size_t)r * Wp;
    for (int k = tid; k < Wp; k += kSortThreads) {
      if (k < W) {
        const KeyT key = src[k];
        uint32_t site;
        uint64_t d;
        if constexpr (kPayload) {
          site = psrc[k];
          d = (uint64_t)key;
        } else {
          site = (uint32_t)(key & sitemask);
          d = (uint64_t)(key >> sitebits);
        }
        orow[k] = (OrdT)site;
        drow[k] = (DistT)d;
      } else {
        orow[k] = (OrdT)m;  // sentinel: T[m] == 0, never open
        drow[k] = (DistT)0;
      }
    }
    __syncthreads();
    (void)flag;
  }
}

// ---- K1 (packed keys): warp-slice stable LSD radix sort ---------------------
//
// Each of the 32 warps owns a contiguous slice of the row.  Per pass: every
// warp histograms its slice (match_any leaders bump the warp's private
// counters -- no atomics), one exclusive scan over (digit, warp) turns the
// counts into scatter offsets, and every warp scatters its slice in order
// (rank within a 32-element step from match_any, then the leader advances the
// warp's offset).  Slices in warp order and steps in lane order keep the
// pass stable; only 3 block barriers per pass.
constexpr int kWsWarps = kSortThreads / 32;

// Lanes holding the same digit (valid lanes only): one ballot per digit bit
// (the warp multi-split trick) -- far cheaper than MATCH.ANY over 32 distinct
// values, which the profile showed serialising.
template <int kBits>
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool valid, int nbits = kBits) {
  unsigned peers = __ballot_sync(kFull, valid);
#pragma unroll
  for (int b = 0; b < kBits; ++b) {
    if (b >= nbits) break;  // warp-uniform
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(kFull, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

template <class KeyT, class OrdT, class DistT, bool kSmem, class CostT>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_build_rows_ws(const CostT* __restrict__ costs, int cstride, int n, int m, int W, int Wp, int sitebits,
                    int npasses, int dbits, OrdT* __restrict__ ord, DistT* __restrict__ dist,
                    KeyT* __restrict__ gkeys, const int* __restrict__ rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);  // [warp][256]
  uint32_t* tot = cnt + kWsWarps * 256;               // [256]
  unsigned char* bufbase = smem + ((kWsWarps * 256 + 256 + 4) * 4 + 15) / 16 * 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  KeyT* A = kSmem ? reinterpret_cast<KeyT*>(bufbase) : gkeys + (size_t)blockIdx.x * 2 * m;
  KeyT* B = A + m;
  const unsigned lt = lanemask_lt();
  const KeyT sitemask = (KeyT(1) << sitebits) - 1;
  const unsigned dmask = (1u << dbits) - 1;
  const int slice = (m + kWsWarps - 1) / kWsWarps;
  const int s0 = min(m, warp * slice), s1 = min(m, s0 + slice);
  uint32_t* mycnt = cnt + warp * 256;

  // rows == nullptr: every row; else rows[0] rows listed in rows[1..] (the
  // rows the counting-sort path handed back)
  const int nr = rows ? rows[0] : n;
  for (int ri = blockIdx.x; ri < nr; ri += gridDim.x) {
    const int r = rows ? rows[1 + ri] : ri;
    const CostT* crow = costs + (size_t)r * cstride;
    // keys of the warp's slice, with the first pass's digit histogram (shared
    // atomics: one per key, instead of a ballot ranking pass)
    for (int d = lane; d < 256; d += 32) mycnt[d] = 0;
    __syncwarp();
    for (int x = s0 + lane; x < s1; x += 32) {
      const KeyT key = ((KeyT)(uint64_t)crow[x] << sitebits) | (KeyT)x;
      A[x] = key;
      atomicAdd(&mycnt[(unsigned)(key >> sitebits) & dmask], 1u);
    }
    // with no pass (every cost 0) the write-out below reads other warps'
    // slices straight away: order it after every slice's keys (CTA-uniform)
    if (npasses == 0) __syncthreads();
    KeyT* src = A;
    KeyT* dst = B;
    for (int q = 0; q < npasses; ++q) {
      const int shift = sitebits + q * dbits;
      if (q > 0) {
        for (int d = lane; d < 256; d += 32) mycnt[d] = 0;
        __syncwarp();
        for (int x = s0 + lane; x < s1; x += 32) atomicAdd(&mycnt[(unsigned)(src[x] >> shift) & dmask], 1u);
      }
      __syncthreads();
      if (tid < 256) {  // exclusive prefix over warps per digit; digit totals
        uint32_t run = 0;
        for (int w = 0; w < kWsWarps; ++w) {
          const uint32_t c = cnt[w * 256 + tid];
          cnt[w * 256 + tid] = run;
          run += c;
        }
        tot[tid] = run;
      }
      __syncthreads();
      const bool skip = tot[(unsigned)(src[0] >> shift) & dmask] == (uint32_t)m;  // constant digit
      if (!skip) {
        if (warp == 0) {  // exclusive scan of the digit totals, added into every warp's offsets
          uint32_t v[8], s = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v[j] = tot[lane * 8 + j];
            s += v[j];
          }
          uint32_t incl = s;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
          }
          uint32_t run = incl - s;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            tot[lane * 8 + j] = run;
            run += v[j];
          }
        }
        __syncthreads();
        for (int d = lane; d < 256; d += 32) mycnt[d] += tot[d];
        __syncwarp();
        for (int x0 = s0; x0 < s1; x0 += 32) {
          const int x = x0 + lane;
          const bool valid = x < s1;
          const KeyT key = valid ? src[x] : KeyT(0);
          const unsigned d = valid ? (unsigned)(key >> shift) & dmask : 0u;
          const unsigned peers = digit_peers<8>(d, valid, dbits);
          const unsigned rank = __popc(peers & lt);
          if (valid) dst[mycnt[d] + rank] = key;
          __syncwarp();
          if (valid && rank == 0) mycnt[d] += __popc(peers);
          __syncwarp();
        }
        __syncthreads();
        KeyT* t = src;
        src = dst;
        dst = t;
      }
    }
    OrdT* orow = ord + (size_t)r * Wp;
    DistT* drow = dist + (size_t)r * Wp;
    for (int k = tid; k < Wp; k += kSortThreads) {
      if (k < W) {
        const KeyT key = src[k];
        orow[k] = (OrdT)(uint32_t)(key & sitemask);
        drow[k] = (DistT)(uint64_t)(key >> sitebits);
      } else {
        orow[k] = (OrdT)m;  // sentinel: T[m] == 0, never open
        drow[k] = (DistT)0;
      }
    }
    __syncthreads();
  }
}

// ---- K1 counting-sort path (costs < 2^15, m < 65536) -------------------------
//
// One pass instead of ceil(costbits/8) radix passes: a histogram of the row's
// costs (shared-memory atomics on u16 counters packed in pairs), one block
// scan, and a scatter through atomic cursors.  The atomics place equal costs in
// arbitrary order, so each bucket is then put back into ascending site order
// (the reference's tie-break, ordering.cpp:25-28) by its owning thread with an
// insertion sort -- buckets are the sites at one exact cost, a handful for
// metric instances.  (That sort is 70 % of the kernel's instructions at
// syn20k; ranking every element within its bucket instead measured slower,
// 2.88 -> 2.98 ms: it scans the whole bucket per element.)  A row with a bucket above kCsMaxBucket is handed back
// (rows list) to the radix kernel, so adversarial ties cost radix time, never
// quadratic time.  512-thread CTAs, two per SM when the row fits in half the
// shared memory: one CTA's HBM row load overlaps the other's sort.
constexpr int kCsThreads = 512;
constexpr uint32_t kCsMaxBucket = 64;

// Every (site, cost) of row `crow`: 16-byte loads of 8 u16 costs (the padded
// u16 copy) or one int64 per element.
template <class CostT, class F>
__device__ __forceinline__ void for_each_cost(const CostT* __restrict__ crow, int m, int tid, F&& f) {
  if constexpr (sizeof(CostT) == 2) {
    const uint4* v = reinterpret_cast<const uint4*>(crow);
    for (int x8 = tid; x8 * 8 < m; x8 += kCsThreads) {
      const uint4 w = __ldg(v + x8);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int x = x8 * 8 + q;
        if (x < m) f(x, (ws[q >> 1] >> ((q & 1) * 16)) & 0xffffu);
      }
    }
  } else {
    for (int x = tid; x < m; x += kCsThreads) f(x, (uint32_t)crow[x]);
  }
}

template <class OrdT, class DistT, class CostT>
__global__ void __launch_bounds__(kCsThreads, 2)
    k_build_rows_cs(const CostT* __restrict__ costs, int cstride, int n, int m, int W, int Wp, int sitebits,
                    int costbits, OrdT* __restrict__ ord, DistT* __restrict__ dist, int* __restrict__ rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t wsum[kCsThreads / 32];
  __shared__ int flag;
  const int nb = 1 << costbits, nw = nb >> 1;  // buckets; u32 words of two u16 counters
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  uint32_t* out = cnt + nw;  // the sorted row, packed (cost << sitebits | site)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t sitemask = (1u << sitebits) - 1;
  const int per = (nw + kCsThreads - 1) / kCsThreads;  // counter words owned by a thread in the scan
  const int w0 = min(nw, tid * per), w1 = min(nw, w0 + per);
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const CostT* crow = costs + (size_t)r * cstride;
    for (int x = tid; x < nw; x += kCsThreads) cnt[x] = 0;
    if (tid == 0) flag = 0;
    __syncthreads();
    for_each_cost(crow, m, tid, [&](int, uint32_t c) { atomicAdd(&cnt[c >> 1], 1u << ((c & 1) << 4)); });
    __syncthreads();
    // exclusive scan over the buckets (each thread a contiguous run of words)
    uint32_t sum = 0;
    bool big = false;
    for (int x = w0; x < w1; ++x) {
      const uint32_t v = cnt[x], lo = v & 0xffffu, hi = v >> 16;
      sum += lo + hi;
      big |= lo > kCsMaxBucket || hi > kCsMaxBucket;
    }
    if (big) flag = 1;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = lane < kCsThreads / 32 ? wsum[lane] : 0;
      uint32_t wi = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(kFull, wi, o);
        if (lane >= o) wi += u;
      }
      if (lane < kCsThreads / 32) wsum[lane] = wi - v;
    }
    __syncthreads();
    const bool handback = flag != 0;
    uint32_t run = wsum[warp] + incl - sum;
    for (int x = w0; x < w1; ++x) {  // counters become bucket cursors (starts)
      const uint32_t v = cnt[x], lo = v & 0xffffu, hi = v >> 16;
      cnt[x] = run | ((run + lo) << 16);
      run += lo + hi;
    }
    __syncthreads();
    if (handback) {  // CTA-uniform
      if (tid == 0) rows[1 + atomicAdd(rows, 1)] = r;
      continue;  // the next row's first barrier orders the reuse of cnt / flag
    }
    for_each_cost(crow, m, tid, [&](int x, uint32_t c) {  // scatter through atomic cursors
      const uint32_t sh = (c & 1) << 4;
      const uint32_t old = atomicAdd(&cnt[c >> 1], 1u << sh);
      out[(old >> sh) & 0xffffu] = (c << sitebits) | (uint32_t)x;
    });
    __syncthreads();
    for (int b = tid; b < nb; b += kCsThreads) {  // bucket b = [end(b-1), end(b)), cursors now at the ends
      const uint32_t e = (cnt[b >> 1] >> ((b & 1) << 4)) & 0xffffu;
      const uint32_t s0 = b == 0 ? 0u : (cnt[(b - 1) >> 1] >> (((b - 1) & 1) << 4)) & 0xffffu;
      for (uint32_t i = s0 + 1; i < e; ++i) {  // insertion sort by site (same cost)
        const uint32_t key = out[i];
        uint32_t j = i;
        while (j > s0 && out[j - 1] > key) {
          out[j] = out[j - 1];
          --j;
        }
        out[j] = key;
      }
    }
    __syncthreads();
    OrdT* orow = ord + (size_t)r * Wp;
    DistT* drow = dist + (size_t)r * Wp;
    for (int k = tid; k < Wp; k += kCsThreads) {
      if (k < W) {
        const uint32_t key = out[k];
        orow[k] = (OrdT)(key & sitemask);
        drow[k] = (DistT)(key >> sitebits);
      } else {
        orow[k] = (OrdT)m;  // sentinel: T[m] == 0, never open
        drow[k] = (DistT)0;
      }
    }
    __syncthreads();
  }
}

// rows longer than this would overflow the u16 cursors
constexpr int kCsMaxM = 65535;

size_t cs_smem(int m, int costbits) {
  return m > kCsMaxM ? ~(size_t)0 : ((size_t)1 << costbits) / 2 * 4 + (size_t)m * 4;
}

// ---- site-major narrow cost matrix for the gather-min kernel (K2b) --------

// dT row stride nP = round_up(n, 16): 16-byte vector loads of consecutive
// clients stay aligned; pad columns are written as 0 (never summed).
template <class DistT>
__global__ void k_transpose_costs(const int64_t* __restrict__ costs, int n, int nP, int m,
                                  DistT* __restrict__ dT) {
  __shared__ int64_t tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    if (i < n && j < m) tile[r][tx] = costs[(size_t)i * m + j];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + tx;
    if (i < nP && j < m) dT[(size_t)j * nP + i] = i < n ? (DistT)tile[tx][r] : (DistT)0;
  }
}

// ---- host launchers --------------------------------------------------------

cudaError_t launch_prep_costs(const int64_t* costs, int n, int m, int mP, int nP, uint16_t* c16, uint16_t* dT,
                              unsigned long long* out_max, int* out_neg, int sms, cudaStream_t st) {
  const long long tiles = (long long)((m + 31) / 32) * ((nP + 63) / 64);
  const int blocks = (int)std::min<long long>((long long)sms * 8, tiles);
  k_prep_costs<<<blocks, 256, 0, st>>>(costs, n, m, mP, nP, c16, dT, out_max, out_neg);
  return cudaGetLastError();
}

cudaError_t launch_validate_costs(const int64_t* costs, size_t count, unsigned long long* out_max,
                              int* out_neg, int sms, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((size_t)sms * 8, (count + 255) / 256 + 1);
  k_validate_costs<<<blocks, 256, 0, st>>>(costs, count, out_max, out_neg);
  return cudaGetLastError();
}

size_t sort_smem_header() { return ((256 + 256 + 256 * kHistPitch + 4) * 4 + 15) / 16 * 16; }

template <class KeyT, bool kPayload, class OrdT, class DistT>
static cudaError_t launch_rows_t(const BuildPlan& bp, const int64_t* costs, const uint16_t* c16, void* ord,
                                 void* dist, void* scratch_keys, uint32_t* scratch_pay, int* rows, cudaStream_t st) {
  const size_t per = (size_t)bp.m * (sizeof(KeyT) + (kPayload ? 4 : 0)) * 2;
  const size_t smem = sort_smem_header() + per;
  if constexpr (!kPayload && sizeof(KeyT) == 4 && sizeof(OrdT) == 2) {
    if (bp.cs_path) {  // counting sort; rows with large tie buckets go to the radix kernel below
      const size_t cs = cs_smem(bp.m, bp.cs_bits);
      cudaError_t e = cudaMemsetAsync(rows, 0, sizeof(int), st);
      if (e != cudaSuccess) return e;
      if (c16) {
        auto kern = k_build_rows_cs<OrdT, DistT, uint16_t>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
        if (e != cudaSuccess) return e;
        kern<<<bp.cs_grid, kCsThreads, cs, st>>>(c16, bp.mP, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits, bp.cs_bits,
                                                  (OrdT*)ord, (DistT*)dist, rows);
      } else {
        auto kern = k_build_rows_cs<OrdT, DistT, int64_t>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
        if (e != cudaSuccess) return e;
        kern<<<bp.cs_grid, kCsThreads, cs, st>>>(costs, bp.m, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits, bp.cs_bits,
                                                  (OrdT*)ord, (DistT*)dist, rows);
      }
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  if constexpr (!kPayload) {  // packed keys: the warp-slice radix sort
    // npasses = ceil(costbits / 8) passes of balanced digits (<= 8 bits: one
    // ballot per digit bit in the ranking), e.g. 2 x 7 bits for 14-bit costs
    const int dbits = bp.npasses ? (bp.costbits + bp.npasses - 1) / bp.npasses : 8;
    const size_t hs = sort_smem_header();
    auto go = [&](auto kern, size_t sm, KeyT* keys) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      if (c16)
        kern<<<bp.grid, kSortThreads, sm, st>>>(c16, bp.mP, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits, bp.npasses, dbits,
                                                (OrdT*)ord, (DistT*)dist, keys, bp.cs_path ? rows : nullptr);
      return cudaGetLastError();
    };
    auto go64 = [&](auto kern, size_t sm, KeyT* keys) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      kern<<<bp.grid, kSortThreads, sm, st>>>(costs, bp.m, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits, bp.npasses, dbits,
                                              (OrdT*)ord, (DistT*)dist, keys, bp.cs_path ? rows : nullptr);
      return cudaGetLastError();
    };
    if (c16) {
      return bp.smem_path ? go(k_build_rows_ws<KeyT, OrdT, DistT, true, uint16_t>, smem, nullptr)
                          : go(k_build_rows_ws<KeyT, OrdT, DistT, false, uint16_t>, hs, (KeyT*)scratch_keys);
    }
    return bp.smem_path ? go64(k_build_rows_ws<KeyT, OrdT, DistT, true, int64_t>, smem, nullptr)
                        : go64(k_build_rows_ws<KeyT, OrdT, DistT, false, int64_t>, hs, (KeyT*)scratch_keys);
  }
  if (bp.smem_path) {
    auto kern = k_build_rows<KeyT, kPayload, OrdT, DistT, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<bp.grid, kSortThreads, smem, st>>>(costs, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits,
                                              bp.npasses, (OrdT*)ord, (DistT*)dist, nullptr, nullptr);
  } else {
    auto kern = k_build_rows<KeyT, kPayload, OrdT, DistT, false>;
    const size_t hs = sort_smem_header();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
    if (e != cudaSuccess) return e;
    kern<<<bp.grid, kSortThreads, hs, st>>>(costs, bp.n, bp.m, bp.W, bp.Wp, bp.sitebits,
                                            bp.npasses, (OrdT*)ord, (DistT*)dist,
                                            (KeyT*)scratch_keys, scratch_pay);
  }
  return cudaGetLastError();
}

template <class OrdT, class DistT>
static cudaError_t launch_rows_od(const BuildPlan& bp, const int64_t* costs, const uint16_t* c16, void* ord,
                                  void* dist, void* sk, uint32_t* sp, int* rows, cudaStream_t st) {
  switch (bp.key_kind) {
    case KeyKind::kPacked32:
      return launch_rows_t<uint32_t, false, OrdT, DistT>(bp, costs, c16, ord, dist, sk, sp, rows, st);
    case KeyKind::kPacked64:
      return launch_rows_t<uint64_t, false, OrdT, DistT>(bp, costs, c16, ord, dist, sk, sp, rows, st);
    default:  // payload keys: costs wider than 64 - sitebits bits, never the u16 copy
      return launch_rows_t<uint64_t, true, OrdT, DistT>(bp, costs, nullptr, ord, dist, sk, sp, rows, st);
  }
}

cudaError_t launch_build_rows(const BuildPlan& bp, const int64_t* costs, const uint16_t* c16, void* ord,
                              void* dist, void* scratch_keys, uint32_t* scratch_pay, int* rows, cudaStream_t st) {
  if (bp.site_bytes == 2) {
    if (bp.dist_bytes == 2) return launch_rows_od<uint16_t, uint16_t>(bp, costs, c16, ord, dist, scratch_keys, scratch_pay, rows, st);
    if (bp.dist_bytes == 4) return launch_rows_od<uint16_t, uint32_t>(bp, costs, nullptr, ord, dist, scratch_keys, scratch_pay, rows, st);
    return launch_rows_od<uint16_t, uint64_t>(bp, costs, nullptr, ord, dist, scratch_keys, scratch_pay, rows, st);
  }
  if (bp.dist_bytes == 2) return launch_rows_od<uint32_t, uint16_t>(bp, costs, c16, ord, dist, scratch_keys, scratch_pay, rows, st);
  if (bp.dist_bytes == 4) return launch_rows_od<uint32_t, uint32_t>(bp, costs, nullptr, ord, dist, scratch_keys, scratch_pay, rows, st);
  return launch_rows_od<uint32_t, uint64_t>(bp, costs, nullptr, ord, dist, scratch_keys, scratch_pay, rows, st);
}

cudaError_t launch_transpose_costs(const int64_t* costs, int n, int nP, int m, int dist_bytes, void* dT,
                                   cudaStream_t st) {
  dim3 grid((m + 31) / 32, (nP + 31) / 32), block(32, 8);
  if (dist_bytes == 2) k_transpose_costs<uint16_t><<<grid, block, 0, st>>>(costs, n, nP, m, (uint16_t*)dT);
  else if (dist_bytes == 4) k_transpose_costs<uint32_t><<<grid, block, 0, st>>>(costs, n, nP, m, (uint32_t*)dT);
  else k_transpose_costs<uint64_t><<<grid, block, 0, st>>>(costs, n, nP, m, (uint64_t*)dT);
  return cudaGetLastError();
}

}  // namespace pmb
