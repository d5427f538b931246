// The reference's C++ API, unchanged, over the device path (include/compat/pmedian/):
// the calls a reference user makes -- Instance, build_ordering, fitness,
// min_cost_sum / direct_cost, evolve_block, run_ga -- on Example 1 of the
// paper (5 clients x 4 sites, p = 2).  Prints PASS.
#include <cstdio>
#include <vector>

#include "pmedian/ga.hpp"
#include "pmedian/ordering.hpp"

static int failures = 0;
#define EXPECT(c)                                                 \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAILED line %d: %s\n", __LINE__, #c);          \
      ++failures;                                                 \
    }                                                             \
  } while (0)

int main() {
  using namespace pmedian;
  const Instance inst(5, 4, 2, {7, 10, 16, 11, 15, 17, 7, 7, 10, 4, 6, 6, 7, 11, 18, 12, 10, 22, 14, 8});
  const OrderingTables t = build_ordering(inst);
  EXPECT(t.width == 3);
  const std::vector<std::uint32_t> pi = {0, 1, 3, 2, 3, 0, 1, 2, 3, 0, 1, 3, 3, 0, 2};
  const std::vector<std::int64_t> delta = {7, 3, 1, 7, 0, 8, 4, 2, 0, 7, 4, 1, 8, 2, 4};
  EXPECT(t.site_order == pi);
  EXPECT(t.increments == delta);
  EXPECT(fitness(t, Chromosome::from_bits("1001")) == 35);
  EXPECT(fitness(t, Chromosome::from_bits("0110")) == 46);
  EXPECT(fitness(t, Chromosome::from_bits("1100")) == 43);
  for (const char* bits : {"1100", "1010", "1001", "0110", "0101", "0011"}) {
    const Chromosome c = Chromosome::from_bits(bits);
    EXPECT(fitness(t, c) == direct_cost(inst, c));
    EXPECT(fitness(t, c) == min_cost_sum(inst, c));
  }
  bool threw = false;
  try {
    (void)fitness(t, Chromosome::from_bits("100"));
  } catch (const StructuralError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    (void)direct_cost(inst, Chromosome::from_bits("1110"));
  } catch (const ContractError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    Instance bad(2, 2, 2, {1, 2, 3, 4});
  } catch (const DomainError&) {
    threw = true;
  }
  EXPECT(threw);

  // evolve_block: in place, every member still opens p sites, the result is the block minimum
  GaConfig cfg;
  cfg.nb = 1;
  cfg.nt = 4;
  cfg.seed = 3;
  std::vector<Chromosome> block = {Chromosome::from_bits("1100"), Chromosome::from_bits("0110"),
                                   Chromosome::from_bits("0011"), Chromosome::from_bits("1010")};
  const BlockResult br = evolve_block(block, t, cfg, 0, 0);
  for (const Chromosome& c : block) EXPECT(c.popcount() == 2);
  EXPECT(br.cost == fitness(t, block[br.thread]));
  for (const Chromosome& c : block) EXPECT(br.cost <= fitness(t, c));

  // run_ga reaches the optimum, 35 at sites {1, 4} (test_ga.cpp:322-336)
  GaConfig rc;
  rc.nb = 2;
  rc.nt = 4;
  rc.evolve_limit = 10;
  rc.saturation = 10;
  const RunResult r = run_ga(inst, rc);
  EXPECT(r.best_cost == 35);
  EXPECT(r.best == Chromosome::from_bits("1001"));
  EXPECT(r.kernel_of_best >= 1 && r.kernels_executed >= r.kernel_of_best);
  EXPECT(exact_optimum_small(inst).cost == 35);

  if (failures == 0) std::printf("PASS\n");
  return failures ? 1 : 0;
}
