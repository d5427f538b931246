// Device restatements of the reference GA's pure building blocks:
//   splitmix RandomStream   proj/include/pmedian/rng.hpp:11-51
//   crossover               proj/src/ga.cpp:35-63
//   circular/block shift    proj/src/ga.cpp:65-90
//   random_shift_mutation   proj/src/ga.cpp:92-104
//   crossover_couple        proj/src/ga.cpp:106-111
// All operate on a chromosome's raw words (chromosome.hpp:24: site j = bit
// j&63 of word j>>6) and reproduce the reference bit for bit, including every
// RNG draw in the reference's order.  Word-level implementations: a shift
// costs O(m/64), a crossover O(m/64 + exchange count).
#pragma once

#include <stdint.h>

namespace pmb {

// ---- RandomStream (rng.hpp) ---------------------------------------------------

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Stream {
  uint64_t state;
  __host__ __device__ static Stream derive(uint64_t master, const uint64_t* key, int nkey) {
    uint64_t s = mix64(master ^ 0x6a09e667f3bcc909ULL);
    for (int i = 0; i < nkey; ++i) s = mix64(s ^ mix64(key[i] + 0x9e3779b97f4a7c15ULL));
    return Stream{s};
  }
  __host__ __device__ uint64_t next() {
    state += 0x9e3779b97f4a7c15ULL;
    return mix64(state);
  }
  __host__ __device__ uint64_t below(uint64_t bound) {
    if ((bound & (bound - 1)) == 0) return next() & (bound - 1);
#ifdef __CUDA_ARCH__
    if (bound < 65536) {  // the GA's bounds (m, p/2, span lengths): 32-bit remainders only
      const uint32_t d = (uint32_t)bound;
      const uint32_t t32 = (0xffffffffu % d + 1) % d;  // 2^32 mod d
      const uint64_t threshold = (t32 * t32) % d;      // 2^64 mod d == (0 - bound) % bound
      uint64_t v = next();
      while (v < threshold) v = next();
      return mod_small(v, d);
    }
#endif
    const uint64_t threshold = (0 - bound) % bound;
    uint64_t v = next();
    while (v < threshold) v = next();
    return v % bound;
  }
  // v mod d for d < 2^16 in 16-bit long-division steps (each a 32-bit remainder;
  // a 64-bit remainder is a long software sequence on the GPU)
  __host__ __device__ static uint64_t mod_small(uint64_t v, uint32_t d) {
    uint32_t r = (uint32_t)(v >> 48) % d;
    r = ((r << 16) | (uint32_t)((v >> 32) & 0xffffu)) % d;
    r = ((r << 16) | (uint32_t)((v >> 16) & 0xffffu)) % d;
    r = ((r << 16) | (uint32_t)(v & 0xffffu)) % d;
    return r;
  }
  __host__ __device__ bool coin() { return (next() & 1) != 0; }
};

// Key prefixes of ga.cpp:19-21.
constexpr uint64_t kHostTag = 1, kCoupleTag = 2, kMutationTag = 3;

// ---- bit helpers --------------------------------------------------------------------

__device__ __forceinline__ uint64_t low_mask(int cnt) {  // cnt in [0, 64]
  return cnt >= 64 ? ~0ull : ((1ull << cnt) - 1);
}

// cnt (<= 64) bits starting at absolute position s (no wrap).
__device__ __forceinline__ uint64_t extract_linear(const uint64_t* w, int s, int cnt) {
  if (cnt <= 0) return 0;
  const int w0 = s >> 6, off = s & 63;
  uint64_t v = w[w0] >> off;
  if (off != 0 && off + cnt > 64) v |= w[w0 + 1] << (64 - off);
  return v & low_mask(cnt);
}

// cnt bits of the cyclic range [base, base+len): relative positions r, r+1, ... (mod len).
__device__ __forceinline__ uint64_t extract_cyclic(const uint64_t* w, int base, int len, int r, int cnt) {
  if (r + cnt <= len) return extract_linear(w, base + r, cnt);
  const int first = len - r;
  return extract_linear(w, base + r, first) | (extract_linear(w, base, cnt - first) << first);
}

// Word wi of out, where out[lo + (t + offset) % len] = in[lo + t] for t < len
// and every other bit is copied.  circular_shift is the case lo = 0, len = m
// (ga.cpp:65-75); block_shift the general one (ga.cpp:77-90).  `offset` is
// already reduced to [0, len).
__device__ __forceinline__ uint64_t rotate_word(const uint64_t* in, int lo, int len, int offset, int wi) {
  uint64_t v = in[wi];
  const int hi = lo + len - 1;
  const int q0 = max(wi * 64, lo), q1 = min(wi * 64 + 63, hi);
  if (q0 <= q1 && offset != 0) {
    const int cnt = q1 - q0 + 1;
    int r = (q0 - lo - offset) % len;
    if (r < 0) r += len;
    const uint64_t bits = extract_cyclic(in, lo, len, r, cnt);
    const int sh = q0 - wi * 64;
    const uint64_t mask = low_mask(cnt) << sh;
    v = (v & ~mask) | ((bits << sh) & mask);
  }
  return v;
}

__device__ void rotate_range(const uint64_t* in, uint64_t* out, int m, int lo, int len, int offset) {
  const int wp = (m + 63) >> 6;
  for (int wi = 0; wi < wp; ++wi) out[wi] = rotate_word(in, lo, len, offset, wi);
}

// The draws of random_shift_mutation (ga.cpp:92-104) in the reference's order:
// coin(whole), coin(direction: true = Left), then k, or a, b, k.  Returns the
// rotated range [lo, lo + len) and its offset.
struct ShiftDraw {
  int lo, len, offset;
};

__device__ __forceinline__ ShiftDraw draw_shift(int m, Stream& rng) {
  const bool whole = rng.coin();
  const bool left = rng.coin();
  if (whole) {
    const int k = 1 + (int)rng.below((uint64_t)(m - 1));
    const int offset = left ? m - k : k;  // ga.cpp:70
    return ShiftDraw{0, m, offset % m};
  }
  const int a = (int)rng.below((uint64_t)m);
  int b = (int)rng.below((uint64_t)(m - 1));
  if (b >= a) ++b;
  const int lo = min(a, b), hi = max(a, b);
  const int len = hi - lo + 1;
  const int k = (int)rng.below((uint64_t)len);
  const int offset = k == 0 ? 0 : (left ? len - k : k);  // ga.cpp:83-85
  return ShiftDraw{lo, len, offset};
}

__device__ void random_shift_mutation(const uint64_t* in, uint64_t* out, int m, Stream& rng) {
  const ShiftDraw d = draw_shift(m, rng);
  rotate_range(in, out, m, d.lo, d.len, d.offset);
}

// The lowest k set bits of x (all of x when it has at most k).
__device__ __forceinline__ uint64_t lowest_bits(uint64_t x, int k) {
  if (k <= 0) return 0;
  for (int n = __popcll(x); n > k; --n) x ^= 1ull << (63 - __clzll((long long)x));
  return x;
}

// crossover (ga.cpp:35-63): child starts as a; scanning cyclically from
// `start`, differing positions adopt b's gene while the closed->open and
// open->closed quotas (exchanges/2 each) last; success iff both quotas are
// used up.  Word-level: the scan visits words start>>6 .. wp-1, then
// 0 .. start>>6 (wp + 1 steps, the start word split in two), taking the
// lowest still-allowed differing bits of each class; a single loop with no
// early exit (an earlier nested-loop form with a mid-loop return was
// observed to run differently from its source on sm_100a in some processes).
__device__ bool crossover(const uint64_t* a, const uint64_t* b, uint64_t* child, int m, int start,
                          int exchanges) {
  const int wp = (m + 63) >> 6, sw = start >> 6;
  for (int wi = 0; wi < wp; ++wi) child[wi] = a[wi];
  int oq = exchanges / 2, cq = exchanges / 2;
  bool done = oq == 0 && cq == 0;
  // steps in groups of 4 whose parent words are loaded up front (4 loads in
  // flight instead of one dependent round trip per step); still one flat loop
  // per group with no early exit
  for (int s0 = 0; s0 <= wp && !done; s0 += 4) {
    uint64_t aw[4], bw[4];
    int wis[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int step = s0 + u;
      const bool first = step < wp - sw;  // [start, m) first, then [0, start)
      wis[u] = first ? sw + step : step - (wp - sw);
      aw[u] = step <= wp ? a[wis[u]] : 0;
      bw[u] = step <= wp ? b[wis[u]] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int step = s0 + u;
      if (step > wp || done) continue;
      const bool first = step < wp - sw;
      const int wi = wis[u];
      uint64_t range = ~0ull;
      if (first) {
        if (wi == sw) range &= ~0ull << (start & 63);
        if (wi == wp - 1) range &= low_mask(((m - 1) & 63) + 1);
      } else if (wi == sw) {
        range &= low_mask(start & 63);
      }
      const uint64_t diff = (aw[u] ^ bw[u]) & range;
      const uint64_t take_o = lowest_bits(diff & ~aw[u], oq);
      const uint64_t take_c = lowest_bits(diff & aw[u], cq);
      oq -= __popcll(take_o);
      cq -= __popcll(take_c);
      child[wi] = (child[wi] | take_o) & ~take_c;
      done = oq == 0 && cq == 0;
    }
  }
  return done;
}

__host__ __device__ __forceinline__ uint32_t crossover_couple(uint32_t t, uint32_t round, uint32_t nt) {
  const uint32_t sub = nt >> round, stride = sub / 2;  // ga.cpp:106-111
  return (t % sub) >= stride ? t - stride : t + stride;
}

}  // namespace pmb
