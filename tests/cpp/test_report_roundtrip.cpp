// The compat reporting API (include/compat/pmedian/bench.hpp) without a GPU:
//   emit     -- structured report of a fixed record set (test_bench.cpp:137-171 cases and more)
//   table    -- the same records as the table report
//   reparse  -- stdin through parse_structured_report, written back structured
//   reject   -- stdin must make parse_structured_report throw StructuralError
// tests/test_report.py feeds these through the reference's own
// parse_structured_report / emit_report (oracle/_ref) and compares bytes.
#include <cstdio>
#include <iostream>
#include <iterator>
#include <string>
#include <vector>

#include "pmedian/bench.hpp"

using pmedian::BenchmarkRecord;

static std::vector<BenchmarkRecord> records() {
  std::vector<BenchmarkRecord> v;
  BenchmarkRecord a;
  a.instance_code = "sample_5x4";
  a.n = 5;
  a.m = 4;
  a.p = 2;
  a.search_space = 6;
  a.best_cost = 35;
  a.reference_cost = 35;
  a.approximation_ratio = 1.0;
  a.kernel_calls = 1;
  a.wall_time = 0.0123456789;
  a.seed = 42;
  v.push_back(a);
  BenchmarkRecord b;
  b.instance_code = "huge";
  b.n = b.m = 900;
  b.p = 90;
  b.search_space = pmedian::binomial(900, 90);
  b.best_cost = 5128;
  b.kernel_calls = 17;
  b.wall_time = 812.25;
  b.seed = 18446744073709551615ULL;
  v.push_back(b);
  BenchmarkRecord c = a;
  c.instance_code = "pmed40 \"quoted\"\\path";
  c.reference_cost = 5128;
  c.best_cost = 5129;
  c.approximation_ratio = 5128.0 / 5129.0;
  c.wall_time = 1e-7;
  c.search_space = pmedian::binomial(20000, 200);
  v.push_back(c);
  BenchmarkRecord d = b;
  d.instance_code = "zero\ttab\bbs\fff\x01ctl\u00e9";
  d.best_cost = 0;
  d.reference_cost = 0;
  d.approximation_ratio = 1.0;
  d.wall_time = 0.0;
  d.search_space = 1;
  v.push_back(d);
  return v;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "emit";
  try {
    if (mode == "emit" || mode == "table") {
      const auto r = records();
      std::fputs(pmedian::emit_report(r, mode == "emit" ? pmedian::ReportStyle::Structured
                                                         : pmedian::ReportStyle::Table)
                     .c_str(),
                 stdout);
      return 0;
    }
    const std::string in((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    if (mode == "reject") {
      try {
        pmedian::parse_structured_report(in);
      } catch (const pmedian::StructuralError&) {
        return 0;
      }
      return 3;
    }
    const auto r = pmedian::parse_structured_report(in);
    std::fputs(pmedian::emit_report(r, pmedian::ReportStyle::Structured).c_str(), stdout);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
}
