// pmedian/bench.hpp, B200 compat layer: the reference's benchmark API
// (proj/include/pmedian/bench.hpp:19-65) with the same types, signatures,
// diagnostics and output formats, over the device path:
//  * parse_dense / parse_orlib (bench.cpp:65-168): the library's parsers
//    (pm_parse_dense; pm_orlib_closure runs the shortest-path closure on the
//    GPU), then an Instance (whose construction builds the tables on the GPU);
//  * run_benchmark (bench.cpp:230-279): repeats with derived seeds, lower
//    medians, run_ga on the device;
//  * emit_report / parse_structured_report / to_scientific (bench.cpp:170-352):
//    host formatting; JSON lines field for field as the reference's emitter
//    writes them (ordered keys, shortest round-trip doubles) and a strict
//    reader for exactly that record shape (the reference uses nlohmann::json,
//    not part of this build).
#pragma once

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <mutex>
#include <optional>
#include <span>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "pmedian/combinatorics.hpp"
#include "pmedian/errors.hpp"
#include "pmedian/ga.hpp"
#include "pmedian/instance.hpp"

namespace pmedian {

enum class InstanceFormat { Dense, OrLib };
enum class ReportStyle { Table, Structured };

struct BenchmarkRecord {
  std::string instance_code;
  std::size_t n = 0;
  std::size_t m = 0;
  std::size_t p = 0;
  BigInt search_space;  // C(m, p)
  std::int64_t best_cost = 0;
  std::optional<std::int64_t> reference_cost;
  std::optional<double> approximation_ratio;  // reference / best
  std::size_t kernel_calls = 0;               // kernel that first reached best_cost
  double wall_time = 0.0;                     // seconds
  std::uint64_t seed = 0;

  friend bool operator==(const BenchmarkRecord&, const BenchmarkRecord&) = default;
};

struct BenchOptions {
  std::size_t repeats = 1;
  std::optional<std::size_t> p_override;
  unsigned workers = 0;
};

namespace detail {
// One context for parsing (the orlib closure runs on its device), created on first use.
inline b200::Tables& parser() {
  static b200::Tables t(default_device());
  return t;
}
inline std::mutex& parser_mutex() {
  static std::mutex mu;
  return mu;
}
}  // namespace detail

// "n m p" header, then n lines of m non-negative costs (bench.cpp:65-104).
inline Instance parse_dense(std::string_view text) {
  b200::Tables::Parsed r;
  {
    std::lock_guard<std::mutex> lock(detail::parser_mutex());
    r = detail::parser().parse_dense(std::string(text));
  }
  return Instance(r.n, r.m, r.p, std::move(r.costs));
}

// "n edges p" + 1-based "u v cost" triples; the instance is the graph's
// all-pairs shortest-path closure, n = m (bench.cpp:106-168).
inline Instance parse_orlib(std::string_view text) {
  b200::Tables::Parsed r;
  {
    std::lock_guard<std::mutex> lock(detail::parser_mutex());
    r = detail::parser().orlib_closure(std::string(text));
  }
  return Instance(r.n, r.m, r.p, std::move(r.costs));
}

// "7.53E+07"-style rendering with exact decimal-string rounding (bench.cpp:170-209).
inline std::string to_scientific(const BigInt& value, int significant_digits) {
  if (significant_digits < 1) throw DomainError("significant digits must be >= 1");
  if (value < 0) throw DomainError("negative values are not supported");
  std::string digits = value.str();
  int exponent = static_cast<int>(digits.size()) - 1;
  if (value == 0) exponent = 0;
  const std::size_t sig = static_cast<std::size_t>(significant_digits);
  std::string mantissa = digits.substr(0, sig);
  if (digits.size() > sig && digits[sig] >= '5') {  // round half up, the carry may ripple past the top digit
    std::size_t i = mantissa.size();
    while (i > 0 && mantissa[i - 1] == '9') mantissa[--i] = '0';
    if (i == 0) {
      mantissa.insert(mantissa.begin(), '1');
      mantissa.pop_back();
      ++exponent;
    } else {
      ++mantissa[i - 1];
    }
  }
  mantissa.resize(std::max(mantissa.size(), sig), '0');
  std::string out(1, mantissa[0]);
  if (significant_digits > 1) out += "." + mantissa.substr(1);
  char exp_buf[16];
  std::snprintf(exp_buf, sizeof exp_buf, "%+03d", exponent);
  return out + "E" + exp_buf;
}

namespace detail {
template <typename T>
T lower_median(std::vector<T> values) {
  std::sort(values.begin(), values.end());
  return values[(values.size() - 1) / 2];
}

inline std::string ratio_cell(const BenchmarkRecord& r) {
  if (!r.reference_cost) return "-";
  if (*r.reference_cost == r.best_cost) return "Optimal";
  if (!r.approximation_ratio) return "-";
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.9f", *r.approximation_ratio);
  return buf;
}

// JSON number text the way nlohmann::json::dump writes a double: shortest
// round-trip digits, and a ".0" on integral values
inline std::string json_double(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

inline std::string json_string(std::string_view s) {
  std::string o = "\"";
  for (const char ch : s) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      case '\r': o += "\\r"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      default:
        if (static_cast<unsigned char>(ch) < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", static_cast<unsigned>(static_cast<unsigned char>(ch)));
          o += b;
        } else {
          o += ch;
        }
    }
  }
  return o + "\"";
}

// A flat JSON object of string / number values, as emit_report writes it.
struct JsonLine {
  std::vector<std::pair<std::string, std::string>> fields;  // key -> raw value text (strings unescaped)
  std::vector<bool> is_string;

  static JsonLine parse(std::string_view s) {
    JsonLine j;
    std::size_t i = 0;
    auto ws = [&] {
      while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    };
    auto fail = [&](const std::string& what) -> void {
      throw StructuralError("structured report: " + what + " at byte " + std::to_string(i));
    };
    auto str = [&]() -> std::string {
      if (i >= s.size() || s[i] != '"') fail("expected a string");
      ++i;
      std::string out;
      while (i < s.size() && s[i] != '"') {
        char ch = s[i++];
        if (ch == '\\') {
          if (i >= s.size()) fail("bad escape");
          const char e = s[i++];
          switch (e) {
            case 'n': ch = '\n'; break;
            case 't': ch = '\t'; break;
            case 'r': ch = '\r'; break;
            case 'b': ch = '\b'; break;
            case 'f': ch = '\f'; break;
            case 'u': {  // \uXXXX (a surrogate pair for code points above U+FFFF), written as UTF-8
              auto hex4 = [&]() -> unsigned {
                unsigned v = 0;
                if (i + 4 > s.size() || std::from_chars(s.data() + i, s.data() + i + 4, v, 16).ptr != s.data() + i + 4)
                  fail("bad \\u escape");
                i += 4;
                return v;
              };
              unsigned cp = hex4();
              if (cp >= 0xD800 && cp < 0xDC00 && i + 6 <= s.size() && s[i] == '\\' && s[i + 1] == 'u') {
                i += 2;
                cp = 0x10000 + ((cp - 0xD800) << 10) + (hex4() - 0xDC00);
              }
              if (cp < 0x80) {
                out += static_cast<char>(cp);
              } else if (cp < 0x800) {
                out += static_cast<char>(0xC0 | (cp >> 6));
                out += static_cast<char>(0x80 | (cp & 0x3F));
              } else if (cp < 0x10000) {
                out += static_cast<char>(0xE0 | (cp >> 12));
                out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                out += static_cast<char>(0x80 | (cp & 0x3F));
              } else {
                out += static_cast<char>(0xF0 | (cp >> 18));
                out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
                out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                out += static_cast<char>(0x80 | (cp & 0x3F));
              }
              continue;
            }
            default: ch = e;
          }
        }
        out += ch;
      }
      if (i >= s.size()) fail("unterminated string");
      ++i;
      return out;
    };
    ws();
    if (i >= s.size() || s[i] != '{') fail("expected an object");
    ++i;
    ws();
    if (i < s.size() && s[i] == '}') {
      ++i;
    } else {
      while (true) {
        ws();
        std::string key = str();
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        ws();
        if (i < s.size() && s[i] == '"') {
          j.fields.emplace_back(std::move(key), str());
          j.is_string.push_back(true);
        } else {
          const std::size_t b = i;
          while (i < s.size() && (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                                  s[i] == '.'))
            ++i;
          if (i == b) fail("expected a value");
          j.fields.emplace_back(std::move(key), std::string(s.substr(b, i - b)));
          j.is_string.push_back(false);
        }
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == '}') {
          ++i;
          break;
        }
        fail("expected ',' or '}'");
      }
    }
    ws();
    if (i != s.size()) fail("trailing characters");
    return j;
  }
  const std::pair<std::string, std::string>* find(std::string_view key, bool want_string) const {
    for (std::size_t k = 0; k < fields.size(); ++k)
      if (fields[k].first == key) {
        if (is_string[k] != want_string)
          throw StructuralError("structured report: wrong type for key '" + std::string(key) + "'");
        return &fields[k];
      }
    return nullptr;
  }
  const std::string& at(std::string_view key, bool want_string) const {
    const auto* f = find(key, want_string);
    if (!f) throw StructuralError("structured report: missing key '" + std::string(key) + "'");
    return f->second;
  }
  template <class T>
  T integer(std::string_view key) const {
    const std::string& v = at(key, false);
    T out{};
    const auto r = std::from_chars(v.data(), v.data() + v.size(), out);
    if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
      throw StructuralError("structured report: '" + std::string(key) + "' is not an integer of the field's type");
    return out;
  }
  double real(std::string_view key) const {
    const std::string& v = at(key, false);
    double out = 0;
    const auto r = std::from_chars(v.data(), v.data() + v.size(), out);
    if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
      throw StructuralError("structured report: '" + std::string(key) + "' is not a number");
    return out;
  }
};
}  // namespace detail

// Parse, run `repeats` times (seeds derived from cfg.seed when repeats > 1),
// aggregate component-wise lower medians (bench.cpp:230-279).
inline BenchmarkRecord run_benchmark(const std::filesystem::path& instance_path, InstanceFormat format,
                                     const GaConfig& cfg, std::optional<std::int64_t> reference_cost,
                                     const BenchOptions& options = {}) {
  if (options.repeats < 1) throw DomainError("repeats must be >= 1");
  std::ifstream in(instance_path);
  if (!in) throw StructuralError("cannot open instance file: " + instance_path.string());
  std::ostringstream buffer;
  buffer << in.rdbuf();
  const std::string text = buffer.str();
  Instance inst = format == InstanceFormat::Dense ? parse_dense(text) : parse_orlib(text);
  if (options.p_override) inst = Instance(inst.clients(), inst.sites(), *options.p_override, inst.costs());

  constexpr std::uint64_t kRepeatTag = 4;  // bench.cpp:19
  std::vector<std::int64_t> costs;
  std::vector<std::size_t> kernels;
  std::vector<double> times;
  for (std::size_t r = 0; r < options.repeats; ++r) {
    GaConfig run_cfg = cfg;
    if (options.repeats > 1) run_cfg.seed = RandomStream::derive(cfg.seed, {kRepeatTag, r}).next();
    const RunResult result = run_ga(inst, run_cfg, options.workers);
    costs.push_back(result.best_cost);
    kernels.push_back(result.kernel_of_best);
    times.push_back(result.wall_time.count());
  }
  BenchmarkRecord record;
  record.instance_code = instance_path.stem().string();
  record.n = inst.clients();
  record.m = inst.sites();
  record.p = inst.open_count();
  record.search_space = binomial(record.m, record.p);
  record.best_cost = detail::lower_median(costs);
  record.reference_cost = reference_cost;
  if (reference_cost) {
    if (record.best_cost > 0) {
      record.approximation_ratio = static_cast<double>(*reference_cost) / static_cast<double>(record.best_cost);
    } else if (*reference_cost == 0) {
      record.approximation_ratio = 1.0;
    }
  }
  record.kernel_calls = detail::lower_median(kernels);
  record.wall_time = detail::lower_median(times);
  record.seed = cfg.seed;
  return record;
}

// Table rows, or one JSON object per line (bench.cpp:281-323).
inline std::string emit_report(std::span<const BenchmarkRecord> records, ReportStyle style) {
  if (style == ReportStyle::Structured) {
    std::string out;
    for (const BenchmarkRecord& r : records) {
      out += "{\"instance_code\":" + detail::json_string(r.instance_code) + ",\"n\":" + std::to_string(r.n) +
             ",\"m\":" + std::to_string(r.m) + ",\"p\":" + std::to_string(r.p) +
             ",\"search_space\":" + detail::json_string(r.search_space.str()) +
             ",\"best_cost\":" + std::to_string(r.best_cost);
      if (r.reference_cost) out += ",\"reference_cost\":" + std::to_string(*r.reference_cost);
      if (r.approximation_ratio) out += ",\"approximation_ratio\":" + detail::json_double(*r.approximation_ratio);
      out += ",\"kernel_calls\":" + std::to_string(r.kernel_calls) +
             ",\"wall_time\":" + detail::json_double(r.wall_time) + ",\"seed\":" + std::to_string(r.seed) + "}\n";
    }
    return out;
  }
  std::size_t code_width = 13;
  for (const BenchmarkRecord& r : records) code_width = std::max(code_width, r.instance_code.size() + 2);
  std::ostringstream out;
  out << std::left << std::setw(static_cast<int>(code_width)) << "Instance Code" << std::right << std::setw(6) << "n"
      << std::setw(6) << "m" << std::setw(6) << "p" << std::setw(22) << "Potential Solutions" << std::setw(15)
      << "Approx. Ratio" << std::setw(14) << "Kernel Calls" << std::setw(13) << "Time (Sec.)" << std::setw(14)
      << "Best Cost" << std::setw(22) << "Seed" << '\n';
  for (const BenchmarkRecord& r : records) {
    char time_buf[32];
    std::snprintf(time_buf, sizeof time_buf, "%.3f", r.wall_time);
    out << std::left << std::setw(static_cast<int>(code_width)) << r.instance_code << std::right << std::setw(6)
        << r.n << std::setw(6) << r.m << std::setw(6) << r.p << std::setw(22) << to_scientific(r.search_space, 3)
        << std::setw(15) << detail::ratio_cell(r) << std::setw(14) << r.kernel_calls << std::setw(13) << time_buf
        << std::setw(14) << r.best_cost << std::setw(22) << r.seed << '\n';
  }
  return out.str();
}

// The inverse of the structured report (bench.cpp:325-352): every field
// required except the two optional ones; StructuralError otherwise.
inline std::vector<BenchmarkRecord> parse_structured_report(std::string_view text) {
  std::vector<BenchmarkRecord> records;
  std::size_t start = 0;
  while (start <= text.size()) {
    const std::size_t end = text.find('\n', start);
    const std::string_view line = text.substr(start, end == std::string_view::npos ? std::string_view::npos
                                                                                   : end - start);
    start = end == std::string_view::npos ? text.size() + 1 : end + 1;
    if (std::all_of(line.begin(), line.end(), [](char c) { return std::isspace(static_cast<unsigned char>(c)); }))
      continue;
    const detail::JsonLine j = detail::JsonLine::parse(line);
    BenchmarkRecord r;
    r.instance_code = j.at("instance_code", true);
    r.n = j.integer<std::size_t>("n");
    r.m = j.integer<std::size_t>("m");
    r.p = j.integer<std::size_t>("p");
    try {
      r.search_space = BigInt(j.at("search_space", true));
    } catch (const std::invalid_argument&) {
      throw StructuralError("structured report: search_space is not a decimal integer");
    }
    r.best_cost = j.integer<std::int64_t>("best_cost");
    if (j.find("reference_cost", false)) r.reference_cost = j.integer<std::int64_t>("reference_cost");
    if (j.find("approximation_ratio", false)) r.approximation_ratio = j.real("approximation_ratio");
    r.kernel_calls = j.integer<std::size_t>("kernel_calls");
    r.wall_time = j.real("wall_time");
    r.seed = j.integer<std::uint64_t>("seed");
    records.push_back(std::move(r));
  }
  return records;
}

}  // namespace pmedian
