// Host restatement of the reference's exact population draw
// (proj/src/combinatorics.cpp:9-75): binomial, lexicographic unranking and the
// multiword rejection draw, on a small unsigned big integer (the reference uses
// boost::multiprecision::cpp_int, absent here).  Used by run_ga's
// reference-exact population mode; pure host integer code.
#pragma once

#include <cstddef>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "ga_ops.cuh"

namespace pmb {

class UBig {
 public:
  UBig() = default;
  explicit UBig(uint64_t v) {
    if (v) l_.push_back(v);
  }
  bool is_zero() const { return l_.empty(); }
  size_t limbs() const { return l_.size(); }
  // little-endian fixed-width export (L >= limbs())
  void export_limbs(uint64_t* out, size_t L) const {
    for (size_t i = 0; i < L; ++i) out[i] = i < l_.size() ? l_[i] : 0;
  }
  int cmp(const UBig& o) const {
    if (l_.size() != o.l_.size()) return l_.size() < o.l_.size() ? -1 : 1;
    for (size_t i = l_.size(); i-- > 0;)
      if (l_[i] != o.l_[i]) return l_[i] < o.l_[i] ? -1 : 1;
    return 0;
  }
  void mul(uint64_t f) {
    unsigned __int128 carry = 0;
    for (auto& x : l_) {
      const unsigned __int128 c = (unsigned __int128)x * f + carry;
      x = (uint64_t)c;
      carry = c >> 64;
    }
    if (carry) l_.push_back((uint64_t)carry);
    if (f == 0) l_.clear();
  }
  uint64_t div(uint64_t d) {  // in place, returns the remainder
    unsigned __int128 rem = 0;
    for (size_t i = l_.size(); i-- > 0;) {
      const unsigned __int128 cur = (rem << 64) | l_[i];
      l_[i] = (uint64_t)(cur / d);
      rem = cur % d;
    }
    trim();
    return (uint64_t)rem;
  }
  void sub(const UBig& o) {  // requires *this >= o
    uint64_t borrow = 0;
    for (size_t i = 0; i < l_.size(); ++i) {
      const uint64_t oi = i < o.l_.size() ? o.l_[i] : 0;
      const unsigned __int128 s = (unsigned __int128)oi + borrow;
      borrow = (unsigned __int128)l_[i] < s;
      l_[i] = (uint64_t)((unsigned __int128)l_[i] - s);
    }
    trim();
  }
  void shl64_or(uint64_t v) {  // *this = (*this << 64) | v
    if (!l_.empty()) l_.insert(l_.begin(), v);
    else if (v) l_.push_back(v);
  }
  size_t bit_length() const { return l_.empty() ? 0 : 64 * (l_.size() - 1) + (64 - __builtin_clzll(l_.back())); }
  std::string str() const {  // decimal
    if (l_.empty()) return "0";
    UBig t = *this;
    std::string out;
    while (!t.is_zero()) {
      const uint64_t r = t.div(10000000000000000000ULL);
      std::string chunk = std::to_string(r);
      if (!t.is_zero()) chunk.insert(0, 19 - chunk.size(), '0');
      out.insert(0, chunk);
    }
    return out;
  }
  double div_pow2(size_t bits) const {  // value / 2^bits, from the top two limbs
    if (l_.empty()) return 0.0;
    const size_t n = l_.size();
    double mant = (double)l_[n - 1];
    int e = 64 * (int)(n - 1);
    if (n >= 2) {
      mant = mant * 18446744073709551616.0 + (double)l_[n - 2];
      e -= 64;
    }
    return std::ldexp(mant, e - (int)bits);
  }
  void dec() {  // *this -= 1, requires *this >= 1
    for (auto& x : l_)
      if (x-- != 0) break;
    trim();
  }

 private:
  void trim() {
    while (!l_.empty() && l_.back() == 0) l_.pop_back();
  }
  std::vector<uint64_t> l_;
};

// C(m, p) exactly (combinatorics.cpp:9-18).
inline UBig binomial(size_t m, size_t p) {
  if (p > m - p) p = m - p;
  UBig r(1);
  for (size_t i = 1; i <= p; ++i) {
    r.mul(m - p + i);
    r.div(i);
  }
  return r;
}

// The rank-th p-subset in lexicographic order (combinatorics.cpp:20-52), into words.
inline void unrank_combination(size_t m, size_t p, UBig r, uint64_t* words) {
  const size_t wp = (m + 63) / 64;
  for (size_t i = 0; i < wp; ++i) words[i] = 0;
  if (p == 0) return;
  size_t a = m - 1, k = p - 1, candidate = 0, remaining = p;
  UBig cur = binomial(a, k);
  while (remaining > 0) {
    if (cur.cmp(r) > 0) {
      words[candidate >> 6] |= 1ull << (candidate & 63);
      if (--remaining == 0) break;
      cur.mul(k);
      cur.div(a);  // C(a-1, k-1)
      --a;
      --k;
    } else {
      r.sub(cur);
      cur.mul(a - k);
      cur.div(a);  // C(a-1, k)
      --a;
    }
    ++candidate;
  }
}

// Pascal table for the device unranking kernel: C(x, y) for y <= p, x < m as
// L-limb little-endian numbers, limb-major: limb i of C(x, y) at
// (y * L + i) * m + x (a warp testing 32 consecutive candidates reads one
// contiguous run per limb), followed by C(m, p) itself (L limbs) and the
// per-step limb counts.
inline std::vector<uint64_t> binomial_table(size_t m, size_t p, size_t L) {
  std::vector<uint64_t> t(((p + 1) * m + 1) * L, 0);
  auto at = [&](size_t x, size_t y, size_t i) -> uint64_t& { return t[(y * L + i) * m + x]; };
  for (size_t x = 0; x < m; ++x) at(x, 0, 0) = 1;
  for (size_t y = 1; y <= p; ++y) {
    for (size_t x = 1; x < m; ++x) {  // C(x, y) = C(x-1, y-1) + C(x-1, y); C(0, y) = 0
      unsigned __int128 carry = 0;
      for (size_t i = 0; i < L; ++i) {
        const unsigned __int128 s = (unsigned __int128)at(x - 1, y - 1, i) + at(x - 1, y, i) + carry;
        at(x, y, i) = (uint64_t)s;
        carry = s >> 64;
      }
    }
  }
  binomial(m, p).export_limbs(&t[(p + 1) * L * m], L);
  // then, per k < p, the limbs of C(m, k + 1): every value of step k of the
  // unranking (X and the probed C(x, k + 1)) fits in that many limbs
  UBig c(1);
  for (size_t k = 0; k < p; ++k) {  // C(m, k + 1) = C(m, k) * (m - k) / (k + 1)
    c.mul(m - k);
    c.div(k + 1);
    t.push_back(std::max<size_t>(1, c.limbs()));
  }
  return t;
}

// Uniform in [0, bound) from 64-bit draws with rejection (combinatorics.cpp:54-70).
inline UBig random_below(const UBig& bound, Stream& rng) {
  UBig bm1 = bound;
  bm1.dec();
  if (bm1.is_zero()) return UBig();
  const size_t bits = bm1.bit_length();
  const size_t words = (bits + 63) / 64;
  const size_t top = bits - 64 * (words - 1);
  const uint64_t top_mask = top == 64 ? ~0ull : ((1ull << top) - 1);
  while (true) {
    UBig v(rng.next() & top_mask);
    for (size_t w = 1; w < words; ++w) v.shl64_or(rng.next());
    if (v.cmp(bound) < 0) return v;
  }
}

}  // namespace pmb
