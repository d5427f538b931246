// pmedian/chromosome.hpp, B200 compat layer: the open-site bit vector of
// proj/include/pmedian/chromosome.hpp:13-44.  Its words are the wire format of
// every device entry point (site j = bit j & 63 of word j >> 6), so words()
// hands them to the C ABI without conversion.
#pragma once

#include <bit>
#include <cstddef>
#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "pmedian/errors.hpp"

namespace pmedian {

class Chromosome {
 public:
  Chromosome() = default;
  explicit Chromosome(std::size_t size) : size_(size), words_((size + 63) / 64, 0) {}

  static Chromosome from_open(std::size_t size, const std::vector<std::size_t>& open) {
    Chromosome c(size);
    for (const std::size_t j : open) {
      if (j >= size) throw DomainError("open site index out of range");
      c.set(j, true);
    }
    return c;
  }
  static Chromosome from_bits(std::string_view bits) {
    Chromosome c(bits.size());
    for (std::size_t j = 0; j < bits.size(); ++j) {
      if (bits[j] != '0' && bits[j] != '1') throw DomainError("bit string must contain only 0 and 1");
      if (bits[j] == '1') c.set(j, true);
    }
    return c;
  }
  // The raw words (the one accessor the reference lacks): what the device reads.
  static Chromosome from_words(std::size_t size, const std::uint64_t* words) {
    Chromosome c(size);
    for (std::size_t w = 0; w < c.words_.size(); ++w) c.words_[w] = words[w];
    return c;
  }

  std::size_t size() const { return size_; }
  bool test(std::size_t j) const { return (words_[j >> 6] >> (j & 63)) & 1; }
  void set(std::size_t j, bool value) {
    const std::uint64_t bit = std::uint64_t{1} << (j & 63);
    words_[j >> 6] = value ? (words_[j >> 6] | bit) : (words_[j >> 6] & ~bit);
  }
  std::size_t popcount() const {
    std::size_t n = 0;
    for (const std::uint64_t w : words_) n += static_cast<std::size_t>(std::popcount(w));
    return n;
  }
  std::vector<std::size_t> open_indices() const {
    std::vector<std::size_t> out;
    for (std::size_t w = 0; w < words_.size(); ++w)
      for (std::uint64_t x = words_[w]; x; x &= x - 1) out.push_back(w * 64 + std::countr_zero(x));
    return out;
  }
  std::string to_bits() const {
    std::string s(size_, '0');
    for (std::size_t j = 0; j < size_; ++j)
      if (test(j)) s[j] = '1';
    return s;
  }
  const std::vector<std::uint64_t>& words() const { return words_; }

  friend bool operator==(const Chromosome&, const Chromosome&) = default;

 private:
  std::size_t size_ = 0;
  std::vector<std::uint64_t> words_;
};

}  // namespace pmedian
