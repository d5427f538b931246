// TEST INFRASTRUCTURE ONLY.  A C wrapper over the reference's own, unmodified
// sources (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libpmref.so).  tests/ use it to pin the C restatement
// (oracle/pmoracle.c) and the CUDA path against the real reference, and
// bench.py's --impl reference / cpu_baseline legs time the reference's fitness()
// with it.  Status codes: 0 ok, 1 StructuralError, 2 ContractError,
// 3 DomainError, 4 BudgetError, 9 other.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "pmedian/bench.hpp"
#include "pmedian/combinatorics.hpp"
#include "pmedian/errors.hpp"
#include "pmedian/ga.hpp"
#include "pmedian/instance.hpp"
#include "pmedian/ordering.hpp"
#include "pmedian/polynomial.hpp"

using namespace pmedian;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const StructuralError& e) {
    g_err = e.what();
    return 1;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 2;
  } catch (const DomainError& e) {
    g_err = e.what();
    return 3;
  } catch (const BudgetError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Chromosome from_words(const std::uint64_t* w, std::size_t m) {
  Chromosome c(m);
  for (std::size_t j = 0; j < m; ++j)
    if ((w[j >> 6] >> (j & 63)) & 1) c.set(j, true);
  return c;
}

void to_words(const Chromosome& c, std::uint64_t* w) {
  const std::size_t wp = (c.size() + 63) / 64;
  std::memset(w, 0, wp * 8);
  for (std::size_t j = 0; j < c.size(); ++j)
    if (c.test(j)) w[j >> 6] |= std::uint64_t{1} << (j & 63);
}

struct RefCtx {
  std::unique_ptr<Instance> inst;
  std::unique_ptr<OrderingTables> tables;
};

GaConfig make_cfg(std::size_t nb, std::size_t nt, std::size_t evolve_limit, std::size_t saturation,
                  std::uint64_t seed, long long crossover_iters, long long mutation_iters,
                  int team) {
  GaConfig cfg;
  cfg.nb = nb;
  cfg.nt = nt;
  cfg.evolve_limit = evolve_limit;
  cfg.saturation = saturation;
  cfg.seed = seed;
  if (crossover_iters >= 0) cfg.crossover_iters = static_cast<std::size_t>(crossover_iters);
  if (mutation_iters >= 0) cfg.mutation_iters = static_cast<std::size_t>(mutation_iters);
  cfg.migration = team ? MigrationMode::TeamToFirstBlock : MigrationMode::BlockToSameBlock;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_create(std::size_t n, std::size_t m, std::size_t p, const std::int64_t* costs,
               int build_tables, void** out) {
  auto ctx = std::make_unique<RefCtx>();
  const int rc = guard([&] {
    ctx->inst = std::make_unique<Instance>(n, m, p, std::vector<std::int64_t>(costs, costs + n * m));
    if (build_tables) ctx->tables = std::make_unique<OrderingTables>(build_ordering(*ctx->inst));
  });
  if (rc == 0) *out = ctx.release();
  return rc;
}

// OrderingTables supplied by the caller (fields are public, ordering.hpp:17-31):
// lets the CPU baseline time the reference's own fitness() without re-running
// its single-threaded build_ordering (tables are checked equal elsewhere).
int ref_create_with_tables(std::size_t n, std::size_t m, std::size_t p, const std::uint32_t* site_order,
                           const std::int64_t* increments, void** out) {
  auto ctx = std::make_unique<RefCtx>();
  const int rc = guard([&] {
    auto t = std::make_unique<OrderingTables>();
    t->clients = n;
    t->sites = m;
    t->open_count = p;
    t->width = m - p + 1;
    t->site_order.assign(site_order, site_order + n * t->width);
    t->increments.assign(increments, increments + n * t->width);
    ctx->tables = std::move(t);
  });
  if (rc == 0) *out = ctx.release();
  return rc;
}

void ref_destroy(void* h) { delete static_cast<RefCtx*>(h); }

std::size_t ref_width(void* h) { return static_cast<RefCtx*>(h)->tables->width; }

int ref_get_tables(void* h, std::uint32_t* site_order, std::int64_t* increments) {
  const OrderingTables& t = *static_cast<RefCtx*>(h)->tables;
  std::memcpy(site_order, t.site_order.data(), t.site_order.size() * 4);
  std::memcpy(increments, t.increments.data(), t.increments.size() * 8);
  return 0;
}

// One fitness() per chromosome; nthreads workers each take a contiguous slice
// (the block-level data parallelism of src/ga.cpp:253-277).  The lowest
// failing index is reported.
int ref_evaluate(void* h, const std::uint64_t* words, std::size_t words_per, std::size_t count,
                 std::int64_t* costs_out, std::size_t* first_bad, unsigned nthreads) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  const std::size_t m = ctx->tables->sites;
  std::vector<Chromosome> pop;
  pop.reserve(count);
  for (std::size_t c = 0; c < count; ++c) pop.push_back(from_words(words + c * words_per, m));
  if (nthreads < 1) nthreads = 1;
  std::vector<int> rcs(nthreads, 0);
  std::vector<std::size_t> bad(nthreads, count);
  auto work = [&](unsigned w) {
    const std::size_t lo = count * w / nthreads, hi = count * (w + 1) / nthreads;
    for (std::size_t c = lo; c < hi; ++c) {
      const int rc = guard([&] { costs_out[c] = fitness(*ctx->tables, pop[c]); });
      if (rc != 0) {
        rcs[w] = rc;
        bad[w] = c;
        return;
      }
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nthreads; ++w) pool.emplace_back(work, w);
    for (auto& t : pool) t.join();
  }
  for (unsigned w = 0; w < nthreads; ++w)
    if (rcs[w] != 0) {
      if (first_bad) *first_bad = bad[w];
      return rcs[w];
    }
  return 0;
}

int ref_fitness_bits(void* h, const char* bits, std::int64_t* out) {
  return guard([&] { *out = fitness(*static_cast<RefCtx*>(h)->tables, Chromosome::from_bits(bits)); });
}

int ref_min_cost_sum(void* h, const std::uint64_t* words, std::int64_t* out) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] { *out = min_cost_sum(*ctx->inst, from_words(words, ctx->inst->sites())); });
}

int ref_direct_cost(void* h, const std::uint64_t* words, std::int64_t* out) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] { *out = direct_cost(*ctx->inst, from_words(words, ctx->inst->sites())); });
}

int ref_exact_optimum(void* h, std::uint64_t budget, std::uint64_t* best_words, std::int64_t* cost) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] {
    const ExactOptimum e = exact_optimum_small(*ctx->inst, budget);
    to_words(e.best, best_words);
    *cost = e.cost;
  });
}

int ref_format_polynomial(void* h, int reduced, char* buf, std::size_t cap) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] {
    PseudoBooleanPolynomial poly = build_cost_polynomial(*ctx->tables);
    if (reduced) poly = reduce_polynomial(poly);
    const std::string s = format_polynomial(poly);
    std::snprintf(buf, cap, "%s", s.c_str());
  });
}

int ref_evaluate_polynomial(void* h, int reduced, const std::uint64_t* words, std::int64_t* out) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] {
    PseudoBooleanPolynomial poly = build_cost_polynomial(*ctx->tables);
    if (reduced) poly = reduce_polynomial(poly);
    *out = evaluate_polynomial(poly, from_words(words, ctx->tables->sites));
  });
}

// ---- GA (src/ga.cpp) ------------------------------------------------------

int ref_crossover(const std::uint64_t* a, const std::uint64_t* b, std::size_t m, std::size_t start,
                  std::size_t exchanges, std::uint64_t* child, int* ok) {
  return guard([&] {
    const auto c = crossover(from_words(a, m), from_words(b, m), start, exchanges);
    *ok = c.has_value();
    if (c) to_words(*c, child);
  });
}

int ref_circular_shift(const std::uint64_t* a, std::size_t m, std::size_t k, int left,
                       std::uint64_t* out) {
  return guard([&] {
    to_words(circular_shift(from_words(a, m), k, left ? ShiftDirection::Left : ShiftDirection::Right),
             out);
  });
}

int ref_block_shift(const std::uint64_t* a, std::size_t m, std::size_t lo, std::size_t hi,
                    std::size_t k, int left, std::uint64_t* out) {
  return guard([&] {
    to_words(block_shift(from_words(a, m), lo, hi, k,
                         left ? ShiftDirection::Left : ShiftDirection::Right),
             out);
  });
}

int ref_random_shift_mutation(const std::uint64_t* a, std::size_t m, std::uint64_t* rng_state,
                              std::uint64_t* out) {
  return guard([&] {
    RandomStream rng(*rng_state);
    to_words(random_shift_mutation(from_words(a, m), rng), out);
  });
}

int ref_random_chromosome(std::size_t m, std::size_t p, std::uint64_t seed, std::size_t count,
                          std::uint64_t* out) {
  return guard([&] {
    RandomStream rng(seed);
    const std::size_t wp = (m + 63) / 64;
    for (std::size_t c = 0; c < count; ++c) to_words(random_chromosome(m, p, rng), out + c * wp);
  });
}

int ref_evolve_block(void* h, std::uint64_t* block_words, std::size_t nt, std::size_t nb,
                     std::uint64_t seed, long long crossover_iters, long long mutation_iters,
                     std::uint64_t kernel_index, std::size_t block_index, std::uint64_t* best_words,
                     std::int64_t* best_cost, std::size_t* best_thread) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] {
    const std::size_t m = ctx->tables->sites, wp = (m + 63) / 64;
    GaConfig cfg = make_cfg(nb, nt, 100, 10, seed, crossover_iters, mutation_iters, 0);
    std::vector<Chromosome> block;
    for (std::size_t t = 0; t < nt; ++t) block.push_back(from_words(block_words + t * wp, m));
    const BlockResult r = evolve_block(block, *ctx->tables, cfg, kernel_index, block_index);
    for (std::size_t t = 0; t < nt; ++t) to_words(block[t], block_words + t * wp);
    to_words(r.best, best_words);
    *best_cost = r.cost;
    *best_thread = r.thread;
  });
}

int ref_run_ga(void* h, std::size_t nb, std::size_t nt, std::size_t evolve_limit,
               std::size_t saturation, std::uint64_t seed, long long crossover_iters,
               long long mutation_iters, int team, unsigned workers, std::uint64_t* best_words,
               std::int64_t* best_cost, std::size_t* kernels_executed, std::size_t* kernel_of_best,
               std::int64_t* per_kernel /* evolve_limit entries */, double* wall_s) {
  RefCtx* ctx = static_cast<RefCtx*>(h);
  return guard([&] {
    const GaConfig cfg =
        make_cfg(nb, nt, evolve_limit, saturation, seed, crossover_iters, mutation_iters, team);
    const RunResult r = run_ga(*ctx->inst, cfg, workers);
    to_words(r.best, best_words);
    *best_cost = r.best_cost;
    *kernels_executed = r.kernels_executed;
    *kernel_of_best = r.kernel_of_best;
    for (std::size_t k = 0; k < r.per_kernel_best_costs.size(); ++k) per_kernel[k] = r.per_kernel_best_costs[k];
    *wall_s = r.wall_time.count();
  });
}

// parse_orlib / parse_dense (bench.cpp:65-168): cost matrix out (cap entries), n/m/p out.
int ref_parse(int orlib, const char* text, std::int64_t* costs_out, std::size_t cap, std::size_t* n,
              std::size_t* m, std::size_t* p) {
  return guard([&] {
    const Instance inst = orlib ? parse_orlib(text) : parse_dense(text);
    *n = inst.clients();
    *m = inst.sites();
    *p = inst.open_count();
    if (costs_out && cap >= inst.costs().size())
      std::memcpy(costs_out, inst.costs().data(), inst.costs().size() * 8);
  });
}

// run_benchmark + emit_report (bench.cpp:230-323): the reference CLI's pipeline.
int ref_run_benchmark(const char* path, int orlib, std::size_t nb, std::size_t nt, std::size_t evolve_limit,
                      std::size_t saturation, std::uint64_t seed, long long cx, long long mu, int team,
                      std::size_t repeats, std::size_t p_override, long long reference, int structured,
                      char* out, std::size_t cap) {
  return guard([&] {
    const GaConfig cfg = make_cfg(nb, nt, evolve_limit, saturation, seed, cx, mu, team);
    BenchOptions o;
    o.repeats = repeats;
    if (p_override) o.p_override = p_override;
    std::optional<std::int64_t> ref;
    if (reference >= 0) ref = reference;
    const BenchmarkRecord r =
        run_benchmark(path, orlib ? InstanceFormat::OrLib : InstanceFormat::Dense, cfg, ref, o);
    const std::string s = emit_report({&r, 1}, structured ? ReportStyle::Structured : ReportStyle::Table);
    std::snprintf(out, cap, "%s", s.c_str());
  });
}

// parse_structured_report then emit_report (bench.cpp:281-352): the reference
// reads a structured report and writes it back (structured or table).
int ref_report_roundtrip(const char* text, int structured, char* out, std::size_t cap, std::size_t* count) {
  return guard([&] {
    const std::vector<BenchmarkRecord> recs = parse_structured_report(text);
    *count = recs.size();
    const std::string s = emit_report(recs, structured ? ReportStyle::Structured : ReportStyle::Table);
    std::snprintf(out, cap, "%s", s.c_str());
  });
}

int ref_validate_config(std::size_t nb, std::size_t nt, std::size_t evolve_limit,
                        std::size_t saturation, int team) {
  return guard([&] { make_cfg(nb, nt, evolve_limit, saturation, 1, -1, -1, team).validate(); });
}

}  // extern "C"
