// pmedian/ordering.hpp, B200 compat layer: OrderingTables, build_ordering and
// fitness with the reference's signatures (proj/include/pmedian/ordering.hpp:17-39).
// The tables are built by K1 on the device when the Instance is constructed;
// build_ordering copies them into the reference's host layout (site_order,
// increments: m - p + 1 columns) and keeps the device handle, through which
// fitness runs K2 -- bit-identical to ordering.cpp:40-59, same errors and texts.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <vector>

#include "pmedian/chromosome.hpp"
#include "pmedian/errors.hpp"
#include "pmedian/instance.hpp"

namespace pmedian {

struct OrderingTables {
  std::size_t clients = 0;
  std::size_t sites = 0;
  std::size_t open_count = 0;
  std::size_t width = 0;                  // m - p + 1
  std::vector<std::uint32_t> site_order;  // clients x width, row-major
  std::vector<std::int64_t> increments;   // clients x width, row-major
  std::shared_ptr<detail::Device> device;  // the resident device tables

  std::span<const std::uint32_t> order_row(std::size_t i) const { return {site_order.data() + i * width, width}; }
  std::span<const std::int64_t> increment_row(std::size_t i) const { return {increments.data() + i * width, width}; }
};

inline OrderingTables build_ordering(const Instance& inst) {
  OrderingTables t;
  t.clients = inst.clients();
  t.sites = inst.sites();
  t.open_count = inst.open_count();
  t.width = t.sites - t.open_count + 1;
  t.device = inst.device();
  std::lock_guard<std::mutex> lock(t.device->mu);
  t.device->tables.copy_tables(t.site_order, t.increments);
  return t;
}

inline std::int64_t fitness(const OrderingTables& tables, const Chromosome& c) {
  if (c.size() != tables.sites) throw StructuralError("chromosome length must equal the site count");
  if (!tables.device) throw DomainError("ordering tables must come from build_ordering (device-resident)");
  std::lock_guard<std::mutex> lock(tables.device->mu);
  return tables.device->tables.fitness(c.words());
}

// Extension: one fitness() per chromosome of a batch in one device call (the
// population loops of evolve_block, ga.cpp:147,166,183).
inline std::vector<std::int64_t> fitness_batch(const OrderingTables& tables, std::span<const Chromosome> batch) {
  const std::size_t wp = (tables.sites + 63) / 64;
  std::vector<std::uint64_t> words(batch.size() * wp);
  for (std::size_t i = 0; i < batch.size(); ++i) {
    if (batch[i].size() != tables.sites) throw StructuralError("chromosome length must equal the site count");
    for (std::size_t w = 0; w < wp; ++w) words[i * wp + w] = batch[i].words()[w];
  }
  if (!tables.device) throw DomainError("ordering tables must come from build_ordering (device-resident)");
  std::lock_guard<std::mutex> lock(tables.device->mu);
  return tables.device->tables.evaluate_population(words, batch.size());
}

}  // namespace pmedian
