// pmedian/ga.hpp, B200 compat layer: GaConfig, Population, RunResult,
// BlockResult, evolve_block and run_ga with the reference's signatures
// (proj/include/pmedian/ga.hpp:14-109), run by the device GA (K3/K2):
// bit-identical blocks and RunResults (tests/test_gpu_ga.py, tests/cpp).
// The operator-level helpers (crossover, circular_shift, block_shift,
// random_shift_mutation, crossover_couple, block_min_reduce) are provided as
// host functions with the reference's semantics for callers that use them
// directly; the GA itself never calls them -- evolve_block and run_ga run the
// device kernels (csrc/ga_ops.cuh restates the same operators word-wise).
// Deviation: evolve_block requires every chromosome of the block to open
// exactly p sites (the GA invariant) and says so up front (DomainError).
#pragma once

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "pmedian/chromosome.hpp"
#include "pmedian/errors.hpp"
#include "pmedian/instance.hpp"
#include "pmedian/ordering.hpp"
#include "pmedian/rng.hpp"

namespace pmedian {

enum class ShiftDirection { Left, Right };
enum class MigrationMode { BlockToSameBlock, TeamToFirstBlock };

struct GaConfig {
  std::size_t nb = 60;
  std::size_t nt = 256;
  std::size_t evolve_limit = 100;
  std::size_t saturation = 10;
  std::uint64_t seed = 1;
  std::optional<std::size_t> crossover_iters;
  std::optional<std::size_t> mutation_iters;
  MigrationMode migration = MigrationMode::BlockToSameBlock;

  // GaConfig::validate (ga.cpp:25-33), same texts
  void validate() const {
    if (nb < 1) throw DomainError("nb must be >= 1");
    if (nt < 2 || (nt & (nt - 1)) != 0) throw DomainError("nt must be a power of two >= 2");
    if (evolve_limit < 1) throw DomainError("evolve_limit must be >= 1");
    if (saturation < 1) throw DomainError("saturation must be >= 1");
    if (migration == MigrationMode::TeamToFirstBlock && nb > nt) throw DomainError("team migration needs nb <= nt");
  }
};

struct Population {
  std::size_t nb = 0;
  std::size_t nt = 0;
  std::vector<Chromosome> members;  // nb * nt, block-major
  std::span<Chromosome> block(std::size_t b) { return {members.data() + b * nt, nt}; }
  std::span<const Chromosome> block(std::size_t b) const { return {members.data() + b * nt, nt}; }
};

struct RunResult {
  Chromosome best;
  std::int64_t best_cost = 0;
  std::size_t kernels_executed = 0;
  std::size_t kernel_of_best = 0;  // 1-based
  std::vector<std::int64_t> per_kernel_best_costs;
  std::chrono::duration<double> wall_time{};
};

struct BlockResult {
  Chromosome best;
  std::int64_t cost = 0;
  std::size_t thread = 0;
};

// ---- operator-level helpers (host; ga.hpp:59-91 of the reference) ----------

// Balanced gene exchange (ga.cpp:35-63): scanning cyclically from start_index,
// differing positions adopt b's gene while each direction's quota
// (exchange_count / 2) lasts; nothing when the quotas cannot both be met.
inline std::optional<Chromosome> crossover(const Chromosome& a, const Chromosome& b, std::size_t start_index,
                                           std::size_t exchange_count) {
  if (a.size() != b.size()) throw StructuralError("parents must have equal length");
  const std::size_t m = a.size(), p = a.popcount();
  if (start_index >= m) throw DomainError("crossover start index out of range");
  if (exchange_count < 2 || exchange_count % 2 != 0 || exchange_count / 2 > p / 2)
    throw DomainError("exchange count must be even, between 2 and 2*(popcount/2)");
  Chromosome child = a;
  std::size_t to_open = exchange_count / 2, to_close = exchange_count / 2;
  for (std::size_t s = 0; s < m && (to_open || to_close); ++s) {
    const std::size_t j = (start_index + s) % m;
    const bool ia = a.test(j);
    if (ia == b.test(j)) continue;
    if (!ia && to_open) {
      child.set(j, true);
      --to_open;
    } else if (ia && to_close) {
      child.set(j, false);
      --to_close;
    }
  }
  if (to_open || to_close) return std::nullopt;
  return child;
}

// Whole-vector rotation by k (ga.cpp:65-75): Right moves bit j to j + k.
inline Chromosome circular_shift(const Chromosome& c, std::size_t k, ShiftDirection direction) {
  const std::size_t m = c.size();
  if (k >= m) throw DomainError("shift distance must be < the vector length");
  if (k == 0) return c;
  const std::size_t off = direction == ShiftDirection::Right ? k : m - k;
  Chromosome out(m);
  for (const std::size_t j : c.open_indices()) out.set((j + off) % m, true);
  return out;
}

// Rotation of the subsequence [lo, hi] by k (ga.cpp:77-90).
inline Chromosome block_shift(const Chromosome& c, std::size_t lo, std::size_t hi, std::size_t k,
                              ShiftDirection direction) {
  if (lo > hi || hi >= c.size()) throw DomainError("subsequence bounds out of range");
  const std::size_t len = hi - lo + 1;
  if (k >= len) throw DomainError("shift distance must not exceed the subsequence span");
  if (k == 0) return c;
  const std::size_t off = direction == ShiftDirection::Right ? k : len - k;
  Chromosome out = c;
  for (std::size_t t = 0; t < len; ++t) out.set(lo + (t + off) % len, c.test(lo + t));
  return out;
}

// One mutation with the reference's draw order (ga.cpp:92-104): coin(whole),
// coin(direction: true = Left), then k, or a, b, k.
inline Chromosome random_shift_mutation(const Chromosome& c, RandomStream& rng) {
  const std::size_t m = c.size();
  const bool whole = rng.coin();
  const ShiftDirection dir = rng.coin() ? ShiftDirection::Left : ShiftDirection::Right;
  if (whole) return circular_shift(c, 1 + rng.below(m - 1), dir);
  const std::size_t a = rng.below(m);
  std::size_t b = rng.below(m - 1);
  if (b >= a) ++b;
  const std::size_t lo = a < b ? a : b, hi = a < b ? b : a;
  return block_shift(c, lo, hi, rng.below(hi - lo + 1), dir);
}

// Partner of `thread` in a crossover round (ga.cpp:106-111): t XOR (nt >> (round + 1)).
inline std::size_t crossover_couple(std::size_t thread, std::size_t round, std::size_t nt) {
  const std::size_t sub = nt >> round, stride = sub / 2;
  return thread % sub >= stride ? thread - stride : thread + stride;
}

// (cost, index) minimum, ties to the lower index (ga.cpp:113-134).
inline std::pair<std::int64_t, std::size_t> block_min_reduce(std::span<const std::int64_t> costs) {
  const std::size_t nt = costs.size();
  if (nt == 0 || (nt & (nt - 1)) != 0) throw DomainError("reduction size must be a power of two");
  std::size_t best = 0;
  for (std::size_t t = 1; t < nt; ++t)
    if (costs[t] < costs[best]) best = t;
  return {costs[best], best};
}

namespace detail {
inline pm_ga_config to_device(const GaConfig& cfg) {
  pm_ga_config c = b200::ga_config(cfg.nb, cfg.nt, cfg.evolve_limit, cfg.saturation, cfg.seed);
  c.crossover_iters = cfg.crossover_iters ? (long long)*cfg.crossover_iters : -1;
  c.mutation_iters = cfg.mutation_iters ? (long long)*cfg.mutation_iters : -1;
  c.migration = cfg.migration == MigrationMode::TeamToFirstBlock ? PM_MIGRATE_TEAM : PM_MIGRATE_BLOCK;
  c.population = PM_POPULATION_REFERENCE;  // the reference's exact population draw
  return c;
}
}  // namespace detail

// One kernel pass over one block, in place (ga.cpp:136-194), on the device.
inline BlockResult evolve_block(std::span<Chromosome> block, const OrderingTables& tables, const GaConfig& cfg,
                                std::uint64_t kernel_index, std::size_t block_index) {
  const std::size_t nt = block.size();
  if (nt != cfg.nt) throw StructuralError("block size must equal cfg.nt");
  if (nt < 2 || (nt & (nt - 1)) != 0) throw DomainError("nt must be a power of two >= 2");
  if (!tables.device) throw DomainError("ordering tables must come from build_ordering (device-resident)");
  const std::size_t wp = (tables.sites + 63) / 64;
  std::vector<std::uint64_t> words(nt * wp);
  for (std::size_t t = 0; t < nt; ++t) {
    if (block[t].size() != tables.sites) throw StructuralError("chromosome length must equal the site count");
    for (std::size_t w = 0; w < wp; ++w) words[t * wp + w] = block[t].words()[w];
  }
  GaConfig one = cfg;
  one.nb = 1;
  const pm_ga_config c = detail::to_device(one);
  std::vector<b200::Tables::BlockResult> r;
  {
    std::lock_guard<std::mutex> lock(tables.device->mu);
    // block_index keys the block's random streams (global block index)
    int64_t cost = 0;
    size_t thread = 0;
    const int rc = pm_evolve_blocks(tables.device->tables.handle(), words.data(), 1, wp, &c, kernel_index,
                                    block_index, &cost, &thread);
    if (rc != PM_OK) b200::throw_status(rc, pm_last_error(tables.device->tables.handle()));
    r.push_back({cost, thread});
  }
  for (std::size_t t = 0; t < nt; ++t) block[t] = Chromosome::from_words(tables.sites, &words[t * wp]);
  return {block[r[0].best_thread], r[0].best_cost, r[0].best_thread};
}

// Full run (ga.cpp:219-303) on the device; `workers` is accepted for source
// compatibility (the result never depends on it, as in the reference).
inline RunResult run_ga(const Instance& inst, const GaConfig& cfg, unsigned workers = 0) {
  (void)workers;
  cfg.validate();
  b200::Tables::RunResult r;
  {
    std::lock_guard<std::mutex> lock(inst.device()->mu);
    r = inst.device()->tables.run_ga(detail::to_device(cfg));
  }
  RunResult out;
  out.best = Chromosome::from_words(inst.sites(), r.best.data());
  out.best_cost = r.best_cost;
  out.kernels_executed = r.kernels_executed;
  out.kernel_of_best = r.kernel_of_best;
  out.per_kernel_best_costs = std::move(r.per_kernel_best_costs);
  out.wall_time = std::chrono::duration<double>(r.wall_time);
  return out;
}

}  // namespace pmedian
