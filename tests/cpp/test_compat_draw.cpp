// Prints random_chromosome words (compat combinatorics.hpp, host BigInt) for
// "m p seed count" on stdin; tests/test_report.py compares them with the
// reference's own random_chromosome (oracle/_ref).  No GPU needed.
#include <cstdio>
#include <iostream>

#include "pmedian/combinatorics.hpp"

int main() {
  std::size_t m, p, count;
  std::uint64_t seed;
  while (std::cin >> m >> p >> seed >> count) {
    pmedian::RandomStream rng(seed);
    for (std::size_t c = 0; c < count; ++c) {
      const pmedian::Chromosome ch = pmedian::random_chromosome(m, p, rng);
      for (const std::uint64_t w : ch.words()) std::printf("%llu ", static_cast<unsigned long long>(w));
      std::printf("\n");
    }
  }
  return 0;
}
