// pmedian_b200.hpp -- header-only C++ view of the C ABI (include/pmedian_b200.h)
// that keeps the reference's C++ vocabulary: pmedian::StructuralError /
// ContractError / DomainError / BudgetError (proj/include/pmedian/errors.hpp:8-25)
// are thrown with the reference's message texts, and the entry points carry the
// reference names -- build_ordering (ordering.hpp:33), fitness (ordering.hpp:39),
// min_cost_sum (instance.hpp:39) -- plus the batched evaluate_population that
// replaces the per-chromosome loops of evolve_block (ga.cpp:147,166,183).
//
// Chromosomes travel as their raw words (chromosome.hpp:24,43), so a caller
// holding pmedian::Chromosome objects passes c.words() (the one accessor the
// reference lacks).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pmedian_b200.h"

namespace pmedian {

#ifndef PMEDIAN_ERRORS_DEFINED
#define PMEDIAN_ERRORS_DEFINED
struct StructuralError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractError : std::logic_error {
  using std::logic_error::logic_error;
};
struct DomainError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct BudgetError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#endif

namespace b200 {

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A batch failure also names the lowest failing chromosome.
struct BatchContractError : ContractError {
  BatchContractError(const std::string& msg, std::size_t first) : ContractError(msg), first_bad(first) {}
  std::size_t first_bad;
};

inline void throw_status(int rc, const char* msg, std::size_t first_bad = 0) {
  switch (rc) {
    case PM_OK:
      return;
    case PM_STRUCTURAL:
      throw StructuralError(msg);
    case PM_CONTRACT:
      throw BatchContractError(msg, first_bad);
    case PM_DOMAIN:
      throw DomainError(msg);
    case PM_BUDGET:
      throw BudgetError(msg);
    default:
      throw DeviceError(msg);
  }
}

// Owns one pm_ctx: one device, one stream, the resident ordering tables.
class Tables {
 public:
  explicit Tables(int device = 0) {
    const int rc = pm_create(device, &ctx_);
    if (rc != PM_OK) throw_status(rc, "pm_create failed");
  }
  Tables(const Tables&) = delete;
  Tables& operator=(const Tables&) = delete;
  Tables(Tables&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
  ~Tables() { pm_destroy(ctx_); }

  pm_ctx* handle() const { return ctx_; }

  // Instance validation + build_ordering on the device (instance.cpp:10-30, ordering.cpp:10-38).
  void build(const std::vector<std::int64_t>& costs, std::size_t n, std::size_t m, std::size_t p) {
    if (costs.size() != n * m) throw StructuralError("cost matrix must be exactly n rows by m columns");
    check(pm_set_instance(ctx_, costs.data(), n, m, p));
  }

  // Instance text formats (bench.cpp:65-168): the parsed matrix back on the host.
  struct Parsed {
    std::size_t n = 0, m = 0, p = 0;
    std::vector<std::int64_t> costs;
  };
  Parsed parse_dense(const std::string& text) const {
    Parsed r;
    check(pm_parse_dense(ctx_, text.data(), text.size(), nullptr, 0, &r.n, &r.m, &r.p));
    r.costs.resize(r.n * r.m);
    check(pm_parse_dense(ctx_, text.data(), text.size(), r.costs.data(), r.costs.size(), &r.n, &r.m, &r.p));
    return r;
  }
  // parse_orlib: the graph's all-pairs shortest-path closure, computed on the device
  Parsed orlib_closure(const std::string& text) const {
    Parsed r;
    check(pm_orlib_closure(ctx_, text.data(), text.size(), nullptr, 0, &r.n, &r.p));
    r.m = r.n;
    r.costs.resize(r.n * r.n);
    check(pm_orlib_closure(ctx_, text.data(), text.size(), r.costs.data(), r.costs.size(), &r.n, &r.p));
    return r;
  }

  pm_table_info info() const {
    pm_table_info ti{};
    check(pm_table_info_get(ctx_, &ti));
    return ti;
  }

  // The reference layout (OrderingTables::site_order / ::increments, ordering.hpp:22-23).
  void copy_tables(std::vector<std::uint32_t>& site_order, std::vector<std::int64_t>& increments) const {
    const pm_table_info ti = info();
    site_order.resize(ti.clients * ti.width);
    increments.resize(ti.clients * ti.width);
    check(pm_get_tables(ctx_, site_order.data(), increments.data()));
  }

  // One fitness() per chromosome, bit-identical to ordering.cpp:40-59.
  std::vector<std::int64_t> evaluate_population(const std::vector<std::uint64_t>& words,
                                                std::size_t count) const {
    std::vector<std::int64_t> out(count);
    if (count == 0) return out;
    const std::size_t wp = words.size() / count;
    std::size_t bad = 0;
    const int rc = pm_evaluate(ctx_, words.data(), count, wp, out.data(), &bad);
    if (rc != PM_OK) throw_status(rc, pm_last_error(ctx_), bad);
    return out;
  }

  std::int64_t fitness(const std::vector<std::uint64_t>& words) const {
    return evaluate_population(words, 1)[0];
  }

  // evolve_block (ga.cpp:136-194) over nb consecutive blocks of cfg.nt
  // chromosomes, in place; block b is global block first_block + b.
  struct BlockResult {
    std::int64_t best_cost;
    std::size_t best_thread;
  };
  std::vector<BlockResult> evolve_blocks(std::vector<std::uint64_t>& blocks, std::size_t nb,
                                         const pm_ga_config& cfg, std::uint64_t kernel_index,
                                         std::size_t first_block = 0) {
    std::vector<std::int64_t> bc(nb);
    std::vector<std::size_t> bt(nb);
    const std::size_t wp = nb ? blocks.size() / (nb * cfg.nt) : 0;
    check(pm_evolve_blocks(ctx_, blocks.data(), nb, wp, &cfg, kernel_index, first_block, bc.data(), bt.data()));
    std::vector<BlockResult> out(nb);
    for (std::size_t b = 0; b < nb; ++b) out[b] = {bc[b], bt[b]};
    return out;
  }

  // run_ga (ga.cpp:219-303): RunResult plus work counters.  With world > 1,
  // this rank's islands exchange block bests through `allgather` (e.g.
  // pm_nccl_allgather with a NcclIslands communicator as `user`).
  struct RunResult {
    std::vector<std::uint64_t> best;
    std::int64_t best_cost = 0;
    std::size_t kernels_executed = 0, kernel_of_best = 0;
    std::vector<std::int64_t> per_kernel_best_costs;
    double wall_time = 0;
    std::uint64_t evaluations = 0;
  };
  RunResult run_ga(const pm_ga_config& cfg, int rank = 0, int world = 1, pm_allgather_fn allgather = nullptr,
                   void* user = nullptr) {
    return run_ga_impl(cfg, rank, world, allgather, nullptr, user);
  }
  // Islands over a native NCCL communicator (pm_nccl_create / NcclIslands::comm()):
  // the block records, their all-gather and the generation step stay on the GPU.
  RunResult run_ga(const pm_ga_config& cfg, pm_nccl* comm) {
    int rank = 0, world = 1;
    check(pm_nccl_rank(comm, &rank, &world));
    return run_ga_impl(cfg, rank, world, nullptr, pm_nccl_allgather_device, comm);
  }

 private:
  RunResult run_ga_impl(const pm_ga_config& cfg, int rank, int world, pm_allgather_fn allgather,
                        pm_allgather_device_fn dev, void* user) {
    const pm_table_info ti = info();
    RunResult r;
    r.best.assign((ti.sites + 63) / 64, 0);
    pm_run_result res{};
    // per-kernel bests are read back afterwards: never a buffer sized by evolve_limit
    check(dev ? pm_run_ga_islands_device(ctx_, &cfg, rank, world, dev, user, r.best.data(), nullptr, &res)
              : world == 1 && !allgather
              ? pm_run_ga(ctx_, &cfg, r.best.data(), nullptr, &res)
              : pm_run_ga_islands(ctx_, &cfg, rank, world, allgather, user, r.best.data(), nullptr, &res));
    r.best_cost = res.best_cost;
    r.kernels_executed = res.kernels_executed;
    r.kernel_of_best = res.kernel_of_best;
    r.per_kernel_best_costs.resize(res.kernels_executed);
    std::size_t cnt = 0;
    check(pm_last_per_kernel_best(ctx_, r.per_kernel_best_costs.data(), r.per_kernel_best_costs.size(), &cnt));
    r.wall_time = res.wall_time_s;
    r.evaluations = res.evaluations;
    return r;
  }

 public:
  std::vector<std::int64_t> min_cost_sum(const std::vector<std::uint64_t>& words, std::size_t count) const {
    std::vector<std::int64_t> out(count);
    if (count == 0) return out;
    std::size_t bad = 0;
    const int rc = pm_min_cost_sum(ctx_, words.data(), count, words.size() / count, out.data(), &bad);
    if (rc != PM_OK) throw_status(rc, pm_last_error(ctx_), bad);
    return out;
  }

 private:
  void check(int rc) const {
    if (rc != PM_OK) throw_status(rc, pm_last_error(ctx_));
  }
  pm_ctx* ctx_ = nullptr;
};

// The default GaConfig (ga.hpp:24-38) in the C ABI's form.
inline pm_ga_config ga_config(std::size_t nb = 60, std::size_t nt = 256, std::size_t evolve_limit = 100,
                              std::size_t saturation = 10, std::uint64_t seed = 1) {
  pm_ga_config c{};
  c.nb = nb;
  c.nt = nt;
  c.evolve_limit = evolve_limit;
  c.saturation = saturation;
  c.seed = seed;
  c.crossover_iters = -1;
  c.mutation_iters = -1;
  c.migration = PM_MIGRATE_BLOCK;
  c.population = PM_POPULATION_REFERENCE;
  return c;
}

// One NCCL communicator per rank for the island exchange; pass
// (pm_nccl_allgather, islands.comm()) to Tables::run_ga.
class NcclIslands {
 public:
  static std::string unique_id() {
    std::string id(PM_NCCL_ID_BYTES, '\0');
    if (pm_nccl_unique_id(id.data()) != PM_OK) throw DeviceError("ncclGetUniqueId failed");
    return id;
  }
  NcclIslands(const std::string& id, int rank, int world, int device) {
    const int rc = pm_nccl_create(id.data(), rank, world, device, &comm_);
    if (rc != PM_OK) throw_status(rc, "pm_nccl_create failed");
  }
  NcclIslands(const NcclIslands&) = delete;
  NcclIslands& operator=(const NcclIslands&) = delete;
  ~NcclIslands() { pm_nccl_destroy(comm_); }
  pm_nccl* comm() const { return comm_; }

 private:
  pm_nccl* comm_ = nullptr;
};

}  // namespace b200
}  // namespace pmedian
