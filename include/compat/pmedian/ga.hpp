// pmedian/ga.hpp, B200 compat layer: GaConfig, Population, RunResult,
// BlockResult, evolve_block and run_ga with the reference's signatures
// (proj/include/pmedian/ga.hpp:14-109), run by the device GA (K3/K2):
// bit-identical blocks and RunResults (tests/test_gpu_ga.py, tests/cpp).
// The reference's operator-level helpers (crossover, circular_shift,
// block_shift, random_shift_mutation, crossover_couple, block_min_reduce) run
// inside the device kernels and are not exported here.
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
