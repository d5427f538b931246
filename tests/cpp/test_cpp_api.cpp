// C++ host usage of the boundary, mirroring proj/tests/test_formulation.cpp's
// Example-1 cases (:18-39, :187-208) through include/pmedian_b200.hpp.
// Built and run by tests/test_cpp_api.py; prints PASS lines, exits non-zero on failure.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "pmedian_b200.hpp"

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);      \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static std::vector<std::uint64_t> bits(const std::string& s) {
  std::vector<std::uint64_t> w((s.size() + 63) / 64, 0);
  for (std::size_t j = 0; j < s.size(); ++j)
    if (s[j] == '1') w[j >> 6] |= std::uint64_t{1} << (j & 63);
  return w;
}

int main() {
  pmedian::b200::Tables t(0);
  t.build({7, 10, 16, 11, 15, 17, 7, 7, 10, 4, 6, 6, 7, 11, 18, 12, 10, 22, 14, 8}, 5, 4, 2);
  std::vector<std::uint32_t> order;
  std::vector<std::int64_t> inc;
  t.copy_tables(order, inc);
  const std::vector<std::uint32_t> want_order = {0, 1, 3, 2, 3, 0, 1, 2, 3, 0, 1, 3, 3, 0, 2};
  const std::vector<std::int64_t> want_inc = {7, 3, 1, 7, 0, 8, 4, 2, 0, 7, 4, 1, 8, 2, 4};
  EXPECT(order == want_order);
  EXPECT(inc == want_inc);
  EXPECT(t.fitness(bits("1001")) == 35);
  EXPECT(t.fitness(bits("0110")) == 46);
  EXPECT(t.fitness(bits("1100")) == 43);

  pmedian::b200::Tables u(0);
  u.build({9, 1, 5}, 1, 3, 2);
  EXPECT(u.fitness(bits("010")) == 1);
  bool threw = false;
  try {
    u.fitness(bits("100"));
  } catch (const pmedian::ContractError& e) {
    threw = std::string(e.what()).find("no open site within the scan width") != std::string::npos;
  }
  EXPECT(threw);
  threw = false;
  try {
    u.evaluate_population({0, 0}, 1);  // two words for m = 3
  } catch (const pmedian::StructuralError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    pmedian::b200::Tables v(0);
    v.build({1, 2}, 1, 2, 2);
  } catch (const pmedian::DomainError& e) {
    threw = std::string(e.what()) == "p must be < m";
  }
  EXPECT(threw);
  // run_ga on Example 1 (test_ga.cpp:322-336): optimum 35 at 1001, every seed
  for (std::uint64_t seed = 1; seed <= 5; ++seed) {
    const auto r = t.run_ga(pmedian::b200::ga_config(2, 4, 10, 10, seed));
    EXPECT(r.best_cost == 35 && r.best == bits("1001"));
    EXPECT(r.per_kernel_best_costs.size() == r.kernels_executed);
  }
  // the same run through the library's NCCL island exchange (one rank)
  {
    pmedian::b200::NcclIslands isl(pmedian::b200::NcclIslands::unique_id(), 0, 1, 0);
    const auto a = t.run_ga(pmedian::b200::ga_config(2, 4, 10, 10, 7));
    const auto b = t.run_ga(pmedian::b200::ga_config(2, 4, 10, 10, 7), 0, 1, pm_nccl_allgather, isl.comm());
    EXPECT(a.best_cost == b.best_cost && a.per_kernel_best_costs == b.per_kernel_best_costs);
  }
  // evolve_block keeps an optimal chromosome (test_ga.cpp:224-244)
  {
    std::vector<std::uint64_t> blk;
    for (int i = 0; i < 4; ++i) blk.push_back(bits("1001")[0]);
    const auto br = t.evolve_blocks(blk, 1, pmedian::b200::ga_config(1, 4), 0);
    EXPECT(br.size() == 1 && br[0].best_cost == 35);
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
