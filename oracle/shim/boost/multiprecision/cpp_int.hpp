// TEST INFRASTRUCTURE ONLY.  A minimal stand-in for boost::multiprecision::cpp_int
// (Boost is absent from this image and unpinned by the reference,
// proj/README.md:22-24).  It implements exactly the operations the reference's
// src/combinatorics.cpp and src/ga.cpp use so oracle/_ref can compile those
// sources unmodified: signed construction from integers and decimal strings,
// + - * / by words, shifts, |=, ++, comparisons, static_cast<uint64_t>, str(),
// and msb().  Sign-magnitude with 64-bit limbs.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T v) {  // NOLINT: implicit like Boost
    if constexpr (std::is_signed_v<T>) {
      if (v < 0) {
        neg_ = true;
        mag_.push_back(static_cast<std::uint64_t>(-(static_cast<__int128>(v))));
        return;
      }
    }
    if (v != 0) mag_.push_back(static_cast<std::uint64_t>(v));
  }
  explicit cpp_int(const std::string& s) { parse(s); }
  explicit cpp_int(const char* s) { parse(s); }

  explicit operator std::uint64_t() const { return mag_.empty() ? 0 : mag_[0]; }
  explicit operator double() const {
    double r = 0;
    for (std::size_t i = mag_.size(); i-- > 0;) r = r * 18446744073709551616.0 + double(mag_[i]);
    return neg_ ? -r : r;
  }

  std::string str() const {
    if (mag_.empty()) return "0";
    std::vector<std::uint64_t> m = mag_;
    std::string out;
    while (!m.empty()) {
      const std::uint64_t r = divmod_small(m, 10000000000000000000ULL);
      std::string chunk = std::to_string(r);
      if (!m.empty()) chunk.insert(0, 19 - chunk.size(), '0');
      out.insert(0, chunk);
    }
    return neg_ ? "-" + out : out;
  }

  cpp_int& operator+=(const cpp_int& o) {
    if (neg_ == o.neg_) {
      add_mag(mag_, o.mag_);
    } else if (cmp_mag(mag_, o.mag_) >= 0) {
      sub_mag(mag_, o.mag_);
    } else {
      std::vector<std::uint64_t> t = o.mag_;
      sub_mag(t, mag_);
      mag_ = std::move(t);
      neg_ = o.neg_;
    }
    norm();
    return *this;
  }
  cpp_int& operator-=(const cpp_int& o) {
    cpp_int t = o;
    if (!t.mag_.empty()) t.neg_ = !t.neg_;
    return *this += t;
  }
  cpp_int& operator*=(const cpp_int& o) {
    std::vector<std::uint64_t> r(mag_.size() + o.mag_.size(), 0);
    for (std::size_t i = 0; i < mag_.size(); ++i) {
      unsigned __int128 carry = 0;
      for (std::size_t j = 0; j < o.mag_.size(); ++j) {
        const unsigned __int128 cur = (unsigned __int128)mag_[i] * o.mag_[j] + r[i + j] + carry;
        r[i + j] = static_cast<std::uint64_t>(cur);
        carry = cur >> 64;
      }
      std::size_t k = i + o.mag_.size();
      while (carry) {
        const unsigned __int128 cur = (unsigned __int128)r[k] + carry;
        r[k++] = static_cast<std::uint64_t>(cur);
        carry = cur >> 64;
      }
    }
    mag_ = std::move(r);
    neg_ = neg_ != o.neg_;
    norm();
    return *this;
  }
  // Division by a value that fits one limb (all the reference needs).
  cpp_int& operator/=(const cpp_int& o) {
    if (o.mag_.empty()) throw std::domain_error("cpp_int shim: division by zero");
    if (o.mag_.size() > 1) throw std::domain_error("cpp_int shim: divisor wider than 64 bits");
    divmod_small(mag_, o.mag_[0]);
    neg_ = neg_ != o.neg_;
    norm();
    return *this;
  }
  cpp_int& operator%=(const cpp_int& o) {
    if (o.mag_.size() != 1) throw std::domain_error("cpp_int shim: modulus must fit 64 bits");
    const std::uint64_t r = divmod_small(mag_, o.mag_[0]);
    mag_.clear();
    if (r) mag_.push_back(r);
    norm();
    return *this;
  }
  cpp_int& operator<<=(unsigned s) {
    if (mag_.empty()) return *this;
    const unsigned words = s / 64, bits = s % 64;
    if (bits) {
      std::uint64_t carry = 0;
      for (auto& w : mag_) {
        const std::uint64_t nc = w >> (64 - bits);
        w = (w << bits) | carry;
        carry = nc;
      }
      if (carry) mag_.push_back(carry);
    }
    mag_.insert(mag_.begin(), words, 0);
    return *this;
  }
  cpp_int& operator|=(const cpp_int& o) {
    if (mag_.size() < o.mag_.size()) mag_.resize(o.mag_.size(), 0);
    for (std::size_t i = 0; i < o.mag_.size(); ++i) mag_[i] |= o.mag_[i];
    norm();
    return *this;
  }
  cpp_int& operator++() { return *this += cpp_int(1); }
  cpp_int operator++(int) {
    cpp_int t = *this;
    ++*this;
    return t;
  }
  cpp_int& operator--() { return *this -= cpp_int(1); }
  cpp_int operator-() const {
    cpp_int t = *this;
    if (!t.mag_.empty()) t.neg_ = !t.neg_;
    return t;
  }

  friend cpp_int operator+(cpp_int a, const cpp_int& b) { return a += b; }
  friend cpp_int operator-(cpp_int a, const cpp_int& b) { return a -= b; }
  friend cpp_int operator*(cpp_int a, const cpp_int& b) { return a *= b; }
  friend cpp_int operator/(cpp_int a, const cpp_int& b) { return a /= b; }
  friend cpp_int operator%(cpp_int a, const cpp_int& b) { return a %= b; }
  friend cpp_int operator<<(cpp_int a, unsigned s) { return a <<= s; }
  friend cpp_int operator|(cpp_int a, const cpp_int& b) { return a |= b; }

  friend int compare(const cpp_int& a, const cpp_int& b) {
    if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
    const int c = cmp_mag(a.mag_, b.mag_);
    return a.neg_ ? -c : c;
  }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

  friend std::size_t msb(const cpp_int& a) {
    if (a.mag_.empty()) throw std::domain_error("cpp_int shim: msb of zero");
    return 64 * (a.mag_.size() - 1) + (63 - static_cast<std::size_t>(__builtin_clzll(a.mag_.back())));
  }

 private:
  void norm() {
    while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
    if (mag_.empty()) neg_ = false;
  }
  void parse(const std::string& s) {
    std::size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '-' || s[i] == '+')) neg = s[i++] == '-';
    if (i >= s.size()) throw std::invalid_argument("cpp_int shim: empty number");
    for (; i < s.size(); ++i) {
      if (s[i] < '0' || s[i] > '9') throw std::invalid_argument("cpp_int shim: bad digit");
      *this *= cpp_int(10);
      *this += cpp_int(s[i] - '0');
    }
    neg_ = neg && !mag_.empty();
  }
  static int cmp_mag(const std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static void add_mag(std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b) {
    if (a.size() < b.size()) a.resize(b.size(), 0);
    unsigned __int128 carry = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      const unsigned __int128 cur = (unsigned __int128)a[i] + (i < b.size() ? b[i] : 0) + carry;
      a[i] = static_cast<std::uint64_t>(cur);
      carry = cur >> 64;
      if (!carry && i >= b.size()) break;
    }
    if (carry) a.push_back(1);
  }
  static void sub_mag(std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b) {  // |a| >= |b|
    std::uint64_t borrow = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      const std::uint64_t bi = i < b.size() ? b[i] : 0;
      const unsigned __int128 sub = (unsigned __int128)bi + borrow;
      borrow = (unsigned __int128)a[i] < sub;
      a[i] = static_cast<std::uint64_t>((unsigned __int128)a[i] - sub);
    }
  }
  static std::uint64_t divmod_small(std::vector<std::uint64_t>& a, std::uint64_t d) {
    unsigned __int128 rem = 0;
    for (std::size_t i = a.size(); i-- > 0;) {
      const unsigned __int128 cur = (rem << 64) | a[i];
      a[i] = static_cast<std::uint64_t>(cur / d);
      rem = cur % d;
    }
    while (!a.empty() && a.back() == 0) a.pop_back();
    return static_cast<std::uint64_t>(rem);
  }

  bool neg_ = false;
  std::vector<std::uint64_t> mag_;  // little-endian limbs, no leading zeros
};

// qualified lookup (boost::multiprecision::msb) needs a namespace-scope declaration
std::size_t msb(const cpp_int& a);

}  // namespace multiprecision
}  // namespace boost
