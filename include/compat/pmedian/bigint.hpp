// pmedian::BigInt for the B200 compat layer: the arbitrary-precision signed
// integer the reference takes from boost::multiprecision::cpp_int
// (proj/include/pmedian/combinatorics.hpp:5,12; Boost is not part of this
// build).  It covers what the reference API does with it -- binomial
// coefficients, lexicographic ranks, search-space sizes in BenchmarkRecord and
// their decimal rendering: construction from any integer or a decimal string,
// + - * / % and comparisons (mixed with built-in integers through the implicit
// constructor), ++/--, shifts by whole bits, |= with a 64-bit word, explicit
// narrowing to built-in integers, str(), msb() and stream output.
// Sign + magnitude, 32-bit limbs, little-endian; host-only code.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <vector>

namespace pmedian {

class BigInt {
 public:
  BigInt() = default;
  template <class T, std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool>, int> = 0>
  BigInt(T v) {  // NOLINT: implicit, like cpp_int
    if constexpr (std::is_signed_v<T>) {
      if (v < 0) {
        neg_ = true;
        set_mag(static_cast<std::uint64_t>(0) - static_cast<std::uint64_t>(static_cast<std::int64_t>(v)));
        return;
      }
    }
    set_mag(static_cast<std::uint64_t>(v));
  }
  explicit BigInt(std::string_view dec) {
    std::size_t i = 0;
    bool neg = false;
    if (i < dec.size() && (dec[i] == '-' || dec[i] == '+')) neg = dec[i++] == '-';
    if (i == dec.size()) throw std::invalid_argument("BigInt: empty decimal string");
    for (; i < dec.size(); ++i) {
      const char c = dec[i];
      if (c < '0' || c > '9') throw std::invalid_argument("BigInt: invalid decimal digit");
      mul_small(10);
      add_small(static_cast<std::uint32_t>(c - '0'));
    }
    neg_ = neg && !is_zero();
  }
  explicit BigInt(const char* dec) : BigInt(std::string_view(dec)) {}
  explicit BigInt(const std::string& dec) : BigInt(std::string_view(dec)) {}

  bool is_zero() const { return mag_.empty(); }
  int sign() const { return is_zero() ? 0 : (neg_ ? -1 : 1); }

  // ---- comparisons ---------------------------------------------------------
  friend int compare(const BigInt& a, const BigInt& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    const int c = cmp_mag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.neg_ == b.neg_ && a.mag_ == b.mag_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
  friend bool operator<(const BigInt& a, const BigInt& b) { return compare(a, b) < 0; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return compare(a, b) <= 0; }
  friend bool operator>(const BigInt& a, const BigInt& b) { return compare(a, b) > 0; }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return compare(a, b) >= 0; }

  // ---- arithmetic ----------------------------------------------------------
  BigInt operator-() const {
    BigInt r = *this;
    if (!r.is_zero()) r.neg_ = !r.neg_;
    return r;
  }
  BigInt& operator+=(const BigInt& o) { return add_signed(o, false); }
  BigInt& operator-=(const BigInt& o) { return add_signed(o, true); }
  BigInt& operator*=(const BigInt& o) {
    if (is_zero() || o.is_zero()) return *this = BigInt();
    std::vector<std::uint32_t> r(mag_.size() + o.mag_.size(), 0);
    for (std::size_t i = 0; i < mag_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < o.mag_.size(); ++j) {
        const std::uint64_t t = static_cast<std::uint64_t>(mag_[i]) * o.mag_[j] + r[i + j] + carry;
        r[i + j] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
      }
      std::size_t k = i + o.mag_.size();
      while (carry) {
        const std::uint64_t t = static_cast<std::uint64_t>(r[k]) + carry;
        r[k++] = static_cast<std::uint32_t>(t);
        carry = t >> 32;
      }
    }
    mag_ = std::move(r);
    neg_ = neg_ != o.neg_;
    trim();
    return *this;
  }
  // truncating division and remainder (the sign of the remainder follows the dividend, as cpp_int)
  BigInt& operator/=(const BigInt& o) {
    BigInt q, r;
    divmod(*this, o, q, r);
    return *this = q;
  }
  BigInt& operator%=(const BigInt& o) {
    BigInt q, r;
    divmod(*this, o, q, r);
    return *this = r;
  }
  friend BigInt operator+(BigInt a, const BigInt& b) { return a += b; }
  friend BigInt operator-(BigInt a, const BigInt& b) { return a -= b; }
  friend BigInt operator*(BigInt a, const BigInt& b) { return a *= b; }
  friend BigInt operator/(BigInt a, const BigInt& b) { return a /= b; }
  friend BigInt operator%(BigInt a, const BigInt& b) { return a %= b; }
  BigInt& operator++() { return *this += BigInt(1); }
  BigInt& operator--() { return *this -= BigInt(1); }
  BigInt operator++(int) {
    BigInt t = *this;
    ++*this;
    return t;
  }
  BigInt operator--(int) {
    BigInt t = *this;
    --*this;
    return t;
  }

  // magnitude bit operations (non-negative values: the reference's random_below)
  BigInt& operator<<=(std::size_t bits) {
    if (is_zero() || bits == 0) return *this;
    const std::size_t words = bits / 32, sh = bits % 32;
    std::vector<std::uint32_t> r(mag_.size() + words + 1, 0);
    for (std::size_t i = 0; i < mag_.size(); ++i) {
      const std::uint64_t v = static_cast<std::uint64_t>(mag_[i]) << sh;
      r[i + words] |= static_cast<std::uint32_t>(v);
      r[i + words + 1] |= static_cast<std::uint32_t>(v >> 32);
    }
    mag_ = std::move(r);
    trim();
    return *this;
  }
  BigInt& operator>>=(std::size_t bits) {
    const std::size_t words = bits / 32, sh = bits % 32;
    if (words >= mag_.size()) return *this = BigInt();
    std::vector<std::uint32_t> r(mag_.size() - words, 0);
    for (std::size_t i = 0; i < r.size(); ++i) {
      std::uint64_t v = mag_[i + words];
      if (i + words + 1 < mag_.size()) v |= static_cast<std::uint64_t>(mag_[i + words + 1]) << 32;
      r[i] = static_cast<std::uint32_t>(v >> sh);
    }
    mag_ = std::move(r);
    trim();
    if (is_zero()) neg_ = false;
    return *this;
  }
  friend BigInt operator<<(BigInt a, std::size_t bits) { return a <<= bits; }
  friend BigInt operator>>(BigInt a, std::size_t bits) { return a >>= bits; }
  BigInt& operator|=(std::uint64_t w) {
    if (mag_.size() < 2) mag_.resize(2, 0);
    mag_[0] |= static_cast<std::uint32_t>(w);
    mag_[1] |= static_cast<std::uint32_t>(w >> 32);
    trim();
    return *this;
  }

  // index of the most significant set bit of the magnitude (boost::multiprecision::msb)
  std::size_t msb() const {
    if (is_zero()) throw std::domain_error("msb of zero");
    return 32 * (mag_.size() - 1) + (31 - static_cast<std::size_t>(__builtin_clz(mag_.back())));
  }

  // explicit narrowing (static_cast<std::uint64_t>(x), as cpp_int): the low bits, two's complement
  template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
  explicit operator T() const {
    std::uint64_t v = 0;
    if (!mag_.empty()) v = mag_[0];
    if (mag_.size() > 1) v |= static_cast<std::uint64_t>(mag_[1]) << 32;
    if (neg_) v = static_cast<std::uint64_t>(0) - v;
    return static_cast<T>(v);
  }
  explicit operator double() const {
    double r = 0;
    for (std::size_t i = mag_.size(); i-- > 0;) r = r * 4294967296.0 + mag_[i];
    return neg_ ? -r : r;
  }

  std::string str() const {
    if (is_zero()) return "0";
    BigInt t = *this;
    t.neg_ = false;
    std::string out;
    while (!t.is_zero()) {
      const std::uint32_t r = t.div_small(1000000000u);
      std::string chunk = std::to_string(r);
      if (!t.is_zero()) chunk.insert(0, 9 - chunk.size(), '0');
      out.insert(0, chunk);
    }
    return neg_ ? "-" + out : out;
  }
  friend std::ostream& operator<<(std::ostream& os, const BigInt& v) { return os << v.str(); }

 private:
  static int cmp_mag(const std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  void set_mag(std::uint64_t v) {
    mag_.clear();
    if (v) mag_.push_back(static_cast<std::uint32_t>(v));
    if (v >> 32) mag_.push_back(static_cast<std::uint32_t>(v >> 32));
  }
  void trim() {
    while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
    if (mag_.empty()) neg_ = false;
  }
  void mul_small(std::uint32_t f) {
    std::uint64_t carry = 0;
    for (auto& x : mag_) {
      const std::uint64_t t = static_cast<std::uint64_t>(x) * f + carry;
      x = static_cast<std::uint32_t>(t);
      carry = t >> 32;
    }
    if (carry) mag_.push_back(static_cast<std::uint32_t>(carry));
    trim();
  }
  void add_small(std::uint32_t a) {
    std::uint64_t carry = a;
    for (std::size_t i = 0; carry && i < mag_.size(); ++i) {
      const std::uint64_t t = static_cast<std::uint64_t>(mag_[i]) + carry;
      mag_[i] = static_cast<std::uint32_t>(t);
      carry = t >> 32;
    }
    if (carry) mag_.push_back(static_cast<std::uint32_t>(carry));
  }
  std::uint32_t div_small(std::uint32_t d) {  // magnitude /= d, returns the remainder
    std::uint64_t rem = 0;
    for (std::size_t i = mag_.size(); i-- > 0;) {
      const std::uint64_t cur = (rem << 32) | mag_[i];
      mag_[i] = static_cast<std::uint32_t>(cur / d);
      rem = cur % d;
    }
    trim();
    return static_cast<std::uint32_t>(rem);
  }
  static void add_mag(std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b) {
    if (a.size() < b.size()) a.resize(b.size(), 0);
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      const std::uint64_t t = static_cast<std::uint64_t>(a[i]) + (i < b.size() ? b[i] : 0) + carry;
      a[i] = static_cast<std::uint32_t>(t);
      carry = t >> 32;
    }
    if (carry) a.push_back(static_cast<std::uint32_t>(carry));
  }
  static void sub_mag(std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b) {  // a >= b
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::int64_t t = static_cast<std::int64_t>(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
      borrow = t < 0;
      if (t < 0) t += std::int64_t{1} << 32;
      a[i] = static_cast<std::uint32_t>(t);
    }
  }
  BigInt& add_signed(const BigInt& o, bool subtract) {
    const bool oneg = subtract ? !o.neg_ : o.neg_;
    if (o.is_zero()) return *this;
    if (neg_ == oneg || is_zero()) {
      if (is_zero()) neg_ = oneg;
      add_mag(mag_, o.mag_);
    } else if (cmp_mag(mag_, o.mag_) >= 0) {
      sub_mag(mag_, o.mag_);
    } else {
      std::vector<std::uint32_t> t = o.mag_;
      sub_mag(t, mag_);
      mag_ = std::move(t);
      neg_ = oneg;
    }
    trim();
    return *this;
  }
  // schoolbook long division on bits of the dividend (the values this API
  // divides are binomial-sized: a few hundred bits at most)
  static void divmod(const BigInt& a, const BigInt& b, BigInt& q, BigInt& r) {
    if (b.is_zero()) throw std::domain_error("BigInt: division by zero");
    q = BigInt();
    r = BigInt();
    if (b.mag_.size() == 1) {
      BigInt t = a;
      t.neg_ = false;
      const std::uint32_t rem = t.div_small(b.mag_[0]);
      q = t;
      r = BigInt(rem);
    } else if (cmp_mag(a.mag_, b.mag_) >= 0) {
      BigInt d = b;
      d.neg_ = false;
      const std::size_t bits = a.msb() + 1;
      for (std::size_t i = bits; i-- > 0;) {
        r <<= 1;
        if ((a.mag_[i / 32] >> (i % 32)) & 1u) r.add_small(1);
        if (cmp_mag(r.mag_, d.mag_) >= 0) {
          sub_mag(r.mag_, d.mag_);
          r.trim();
          if (q.mag_.size() < i / 32 + 1) q.mag_.resize(i / 32 + 1, 0);
          q.mag_[i / 32] |= 1u << (i % 32);
        }
      }
      q.trim();
    } else {
      r = a;
      r.neg_ = false;
    }
    q.neg_ = !q.is_zero() && (a.neg_ != b.neg_);
    r.neg_ = !r.is_zero() && a.neg_;
  }

  bool neg_ = false;
  std::vector<std::uint32_t> mag_;
};

// boost::multiprecision::msb spelling for source compatibility
inline std::size_t msb(const BigInt& v) { return v.msb(); }

}  // namespace pmedian
