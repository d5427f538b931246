// Minimal stand-in for the doctest macros the reference's unit tests use
// (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW) -- doctest is not
// in this image.  Test infrastructure: lets the reference's own test files run
// against the B200 compat headers (include/compat/pmedian/).  One translation
// unit defines PMB_DOCTEST_MAIN to get main().
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace pmbdt {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Require {};  // thrown by a failed REQUIRE: ends the test case
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace pmbdt

#define PMBDT_CAT2(a, b) a##b
#define PMBDT_CAT(a, b) PMBDT_CAT2(a, b)
#define PMBDT_CASE(fn, name)                                                      \
  static void fn();                                                               \
  static const pmbdt::Registrar PMBDT_CAT(fn, _reg){name, &fn};                   \
  static void fn()
#define TEST_CASE(name) PMBDT_CASE(PMBDT_CAT(pmbdt_case_, __LINE__), name)
#define CHECK(...)                                             \
  do {                                                         \
    if (!(__VA_ARGS__)) pmbdt::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define REQUIRE(...)                                             \
  do {                                                           \
    if (!(__VA_ARGS__)) {                                        \
      pmbdt::fail(__FILE__, __LINE__, #__VA_ARGS__);             \
      throw pmbdt::Require{};                                    \
    }                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool pmbdt_ok = false;                                                                 \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      pmbdt_ok = true;                                                                     \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!pmbdt_ok) pmbdt::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, text, type)                                             \
  do {                                                                                     \
    bool pmbdt_ok = false;                                                                 \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type& pmbdt_e) {                                                        \
      pmbdt_ok = std::string(pmbdt_e.what()) == std::string(text);                         \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!pmbdt_ok)                                                                         \
      pmbdt::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #text ", " #type ")"); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      pmbdt::fail(__FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");           \
    }                                                                        \
  } while (0)

namespace doctest {
// doctest::Approx: relative tolerance (default: 100 float epsilons, doctest's scale)
struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = 1.0 + (lhs < 0 ? -lhs : lhs) + (a.value < 0 ? -a.value : a.value);
    const double d = lhs - a.value;
    return (d < 0 ? -d : d) < a.eps * scale;
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  double value;
  double eps = 1.1920928955078125e-05;  // doctest: 100 * FLT_EPSILON
};
}  // namespace doctest

#ifdef PMB_DOCTEST_MAIN
int main() {
  int cases = 0;
  for (const auto& c : pmbdt::registry()) {
    ++cases;
    try {
      c.fn();
    } catch (const pmbdt::Require&) {
    } catch (const std::exception& e) {
      pmbdt::fail(c.name, 0, e.what());
    }
  }
  std::printf("%d test cases, %d failed checks\n", cases, pmbdt::failures());
  return pmbdt::failures() ? 1 : 0;
}
#endif
