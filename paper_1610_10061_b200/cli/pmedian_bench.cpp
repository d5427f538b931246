// pmedian_bench -- the reference's benchmark CLI (proj/tools/pmedian_bench.cpp)
// over the B200 path: same flags, same `.opt` sidecar lookup, same repeats /
// lower-median aggregation (run_benchmark, proj/src/bench.cpp:230-279) and the
// same table / structured (JSON lines) reports (emit_report, bench.cpp:281-323),
// with the GA (pm_run_ga) and the instance parsing/closure on the device.
// Extra flags: --population reference|device (default reference: the
// reference's exact draw, so results match it bit for bit), --device N.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmedian_b200.h"
#include "../csrc/combinatorics.h"

namespace {

struct CliError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Record {  // BenchmarkRecord (bench.hpp:21-35)
  std::string instance_code;
  size_t n = 0, m = 0, p = 0;
  std::string search_space;  // C(m, p), decimal
  int64_t best_cost = 0;
  std::optional<int64_t> reference_cost;
  std::optional<double> approximation_ratio;
  size_t kernel_calls = 0;
  double wall_time = 0.0;
  uint64_t seed = 0;
};

// to_scientific (bench.cpp:170-209): exact decimal-string rounding.
std::string to_scientific(const std::string& value, int significant) {
  std::string digits = value;
  int exponent = (int)digits.size() - 1;
  if (value == "0") exponent = 0;
  std::string mantissa = digits.substr(0, (size_t)significant);
  const bool round_up = digits.size() > (size_t)significant && digits[(size_t)significant] >= '5';
  if (round_up) {
    int i = (int)mantissa.size() - 1;
    while (i >= 0 && mantissa[(size_t)i] == '9') {
      mantissa[(size_t)i] = '0';
      --i;
    }
    if (i < 0) {
      mantissa.insert(mantissa.begin(), '1');
      mantissa.pop_back();
      ++exponent;
    } else {
      ++mantissa[(size_t)i];
    }
  }
  while (mantissa.size() < (size_t)significant) mantissa.push_back('0');
  std::ostringstream out;
  out << mantissa[0];
  if (significant > 1) out << '.' << mantissa.substr(1);
  char buf[16];
  std::snprintf(buf, sizeof buf, "%+03d", exponent);
  out << 'E' << buf;
  return out.str();
}

std::string json_double(double v) {  // shortest round-trip, like nlohmann::json::dump
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}

std::string emit(const Record& r, bool structured) {
  if (structured) {
    std::string o = "{\"instance_code\":" + json_string(r.instance_code) + ",\"n\":" + std::to_string(r.n) +
                    ",\"m\":" + std::to_string(r.m) + ",\"p\":" + std::to_string(r.p) +
                    ",\"search_space\":" + json_string(r.search_space) +
                    ",\"best_cost\":" + std::to_string(r.best_cost);
    if (r.reference_cost) o += ",\"reference_cost\":" + std::to_string(*r.reference_cost);
    if (r.approximation_ratio) o += ",\"approximation_ratio\":" + json_double(*r.approximation_ratio);
    o += ",\"kernel_calls\":" + std::to_string(r.kernel_calls) + ",\"wall_time\":" + json_double(r.wall_time) +
         ",\"seed\":" + std::to_string(r.seed) + "}\n";
    return o;
  }
  const size_t code_width = std::max<size_t>(13, r.instance_code.size() + 2);
  std::string ratio = "-";
  if (r.reference_cost) {
    if (*r.reference_cost == r.best_cost) {
      ratio = "Optimal";
    } else if (r.approximation_ratio) {
      char b[32];
      std::snprintf(b, sizeof b, "%.9f", *r.approximation_ratio);
      ratio = b;
    }
  }
  char tb[32];
  std::snprintf(tb, sizeof tb, "%.3f", r.wall_time);
  std::ostringstream out;
  out << std::left << std::setw((int)code_width) << "Instance Code" << std::right << std::setw(6) << "n"
      << std::setw(6) << "m" << std::setw(6) << "p" << std::setw(22) << "Potential Solutions" << std::setw(15)
      << "Approx. Ratio" << std::setw(14) << "Kernel Calls" << std::setw(13) << "Time (Sec.)" << std::setw(14)
      << "Best Cost" << std::setw(22) << "Seed" << '\n';
  out << std::left << std::setw((int)code_width) << r.instance_code << std::right << std::setw(6) << r.n
      << std::setw(6) << r.m << std::setw(6) << r.p << std::setw(22) << to_scientific(r.search_space, 3)
      << std::setw(15) << ratio << std::setw(14) << r.kernel_calls << std::setw(13) << tb << std::setw(14)
      << r.best_cost << std::setw(22) << r.seed << '\n';
  return out.str();
}

int64_t read_reference_file(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw CliError("cannot open reference file: " + path.string());
  int64_t v = 0;
  if (!(in >> v)) throw CliError("reference file must contain one integer: " + path.string());
  return v;
}

template <class T>
T lower_median(std::vector<T> v) {
  std::sort(v.begin(), v.end());
  return v[(v.size() - 1) / 2];
}

uint64_t parse_u64(const std::string& flag, const std::string& s) {
  uint64_t v = 0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc{} || r.ptr != s.data() + s.size()) throw CliError(flag + ": expected a non-negative integer");
  return v;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> opt;
  const std::vector<std::string> known = {"--instance", "--format", "--p", "--nb", "--nt", "--evolve-limit",
                                          "--saturation", "--seed", "--repeats", "--crossover-iters",
                                          "--mutation-iters", "--reference", "--out", "--report", "--migration",
                                          "--workers", "--population", "--device"};
  try {
    for (int a = 1; a < argc; ++a) {
      std::string f = argv[a], v;
      const size_t eq = f.find('=');
      if (eq != std::string::npos) {
        v = f.substr(eq + 1);
        f = f.substr(0, eq);
      } else {
        if (a + 1 >= argc) throw CliError(f + ": missing value");
        v = argv[++a];
      }
      if (std::find(known.begin(), known.end(), f) == known.end()) throw CliError("unknown option " + f);
      opt[f] = v;
    }
    if (!opt.count("--instance")) throw CliError("--instance is required");
    auto get = [&](const char* k, const char* d) { return opt.count(k) ? opt[k] : std::string(d); };
    const std::string format = get("--format", "dense"), report = get("--report", "table"),
                      migration = get("--migration", "block"), population = get("--population", "reference");
    if (format != "dense" && format != "orlib") throw CliError("--format: dense or orlib");
    if (report != "table" && report != "structured") throw CliError("--report: table or structured");
    if (migration != "block" && migration != "team") throw CliError("--migration: block or team");
    if (population != "reference" && population != "device") throw CliError("--population: reference or device");

    pm_ga_config cfg{};
    cfg.nb = parse_u64("--nb", get("--nb", "60"));
    cfg.nt = parse_u64("--nt", get("--nt", "256"));
    cfg.evolve_limit = parse_u64("--evolve-limit", get("--evolve-limit", "100"));
    cfg.saturation = parse_u64("--saturation", get("--saturation", "10"));
    cfg.seed = parse_u64("--seed", get("--seed", "1"));
    cfg.crossover_iters = opt.count("--crossover-iters") ? (long long)parse_u64("--crossover-iters", opt["--crossover-iters"]) : -1;
    cfg.mutation_iters = opt.count("--mutation-iters") ? (long long)parse_u64("--mutation-iters", opt["--mutation-iters"]) : -1;
    cfg.migration = migration == "team" ? PM_MIGRATE_TEAM : PM_MIGRATE_BLOCK;
    cfg.population = population == "device" ? PM_POPULATION_DEVICE : PM_POPULATION_REFERENCE;
    const size_t repeats = parse_u64("--repeats", get("--repeats", "1"));
    if (repeats < 1) throw CliError("repeats must be >= 1");  // bench.cpp:233
    const size_t p_override = opt.count("--p") ? parse_u64("--p", opt["--p"]) : 0;

    std::optional<int64_t> reference;
    if (opt.count("--reference")) {
      reference = read_reference_file(opt["--reference"]);
    } else {
      std::filesystem::path sidecar(opt["--instance"]);
      sidecar.replace_extension(".opt");
      if (std::filesystem::exists(sidecar)) reference = read_reference_file(sidecar);
    }

    std::ifstream in(opt["--instance"]);
    if (!in) throw CliError("cannot open instance file: " + opt["--instance"]);
    std::ostringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();

    pm_ctx* ctx = nullptr;
    if (pm_create((int)parse_u64("--device", get("--device", "0")), &ctx) != PM_OK) throw CliError("no CUDA device");
    auto check = [&](int rc) {
      if (rc != PM_OK) throw CliError(pm_last_error(ctx));
    };
    check(format == "orlib" ? pm_set_instance_orlib(ctx, text.data(), text.size(), p_override)
                            : pm_set_instance_dense(ctx, text.data(), text.size(), p_override));
    pm_table_info ti{};
    check(pm_table_info_get(ctx, &ti));

    std::vector<int64_t> costs;
    std::vector<size_t> kernels;
    std::vector<double> times;
    std::vector<uint64_t> best((ti.sites + 63) / 64);
    for (size_t r = 0; r < repeats; ++r) {
      pm_ga_config run = cfg;
      if (repeats > 1) {  // bench.cpp:249-252
        const uint64_t key[2] = {4, r};
        pmb::Stream s = pmb::Stream::derive(cfg.seed, key, 2);
        run.seed = s.next();
      }
      pm_run_result res{};
      check(pm_run_ga(ctx, &run, best.data(), nullptr, &res));
      costs.push_back(res.best_cost);
      kernels.push_back(res.kernel_of_best);
      times.push_back(res.wall_time_s);
    }
    pm_destroy(ctx);

    Record rec;
    rec.instance_code = std::filesystem::path(opt["--instance"]).stem().string();
    rec.n = ti.clients;
    rec.m = ti.sites;
    rec.p = ti.open_count;
    rec.search_space = pmb::binomial(rec.m, rec.p).str();
    rec.best_cost = lower_median(costs);
    rec.reference_cost = reference;
    if (reference) {  // bench.cpp:262-270
      if (rec.best_cost > 0) rec.approximation_ratio = (double)*reference / (double)rec.best_cost;
      else if (*reference == 0) rec.approximation_ratio = 1.0;
    }
    rec.kernel_calls = lower_median(kernels);
    rec.wall_time = lower_median(times);
    rec.seed = cfg.seed;
    const std::string out = emit(rec, report == "structured");
    if (opt.count("--out")) {
      std::ofstream f(opt["--out"]);
      if (!f) throw CliError("cannot open output file: " + opt["--out"]);
      f << out;
    } else {
      std::cout << out;
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return 0;
}
