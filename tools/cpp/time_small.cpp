// Latency of small-instance calls through the compat API (acceptance.cpp:52-81 budget).
#include <chrono>
#include <cstdio>

#include "pmedian/ordering.hpp"
#include "pmedian/polynomial.hpp"

int main() {
  using C = std::chrono::steady_clock;
  for (int rep = 0; rep < 5; ++rep) {
    auto t0 = C::now();
    pmedian::Instance inst(5, 4, 2, {7, 10, 16, 11, 15, 17, 7, 7, 10, 4, 6, 6, 7, 11, 18, 12, 10, 22, 14, 8});
    auto t1 = C::now();
    const pmedian::OrderingTables t = pmedian::build_ordering(inst);
    auto t2 = C::now();
    const auto poly = pmedian::reduce_polynomial(pmedian::build_cost_polynomial(t));
    auto t3 = C::now();
    auto f = pmedian::fitness(t, pmedian::Chromosome::from_bits("1001"));
    auto t4 = C::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::printf("instance %.1f us, build_ordering %.1f us, polynomial %.1f us, fitness %.1f us (=%lld)\n",
                us(t0, t1), us(t1, t2), us(t2, t3), us(t3, t4), (long long)f);
  }
}
