// Minimal doctest-compatible harness (our own, not doctest): enough of the TEST_CASE /
// CHECK / REQUIRE / Approx surface for the reference's unit-test files to compile unchanged
// against the drop-in header (tests/cpp/build_ref_tests.py) and report failures.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value, eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100, scl = 1.0;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  bool matches(double x) const { return std::fabs(x - value) < eps * (scl + std::max(std::fabs(x), std::fabs(value))); }
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value || a.matches(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value || a.matches(x); }

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail

inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : detail::registry()) {
    detail::state().case_failed = false;
    try {
      c.fn();
    } catch (const detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++detail::state().failures;
      detail::state().case_failed = true;
      std::fprintf(stderr, "test case \"%s\" threw: %s\n", c.name, e.what());
    }
    if (detail::state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED test case: %s\n", c.name);
    }
  }
  std::printf("[harness] test cases: %zu | %zu passed | %d failed\n", detail::registry().size(),
              detail::registry().size() - failed_cases, failed_cases);
  std::printf("[harness] checks: %ld | %ld failures\n", detail::state().checks, detail::state().failures);
  std::printf("%ld failures\n", detail::state().failures);
  return detail::state().failures == 0 ? 0 : 1;
}

}  // namespace doctest

#define HC_DT_CAT_(a, b) a##b
#define HC_DT_CAT(a, b) HC_DT_CAT_(a, b)
#define HC_DT_TEST_CASE(name, id)                                             \
  static void HC_DT_CAT(hc_dt_fn_, id)();                                     \
  static ::doctest::detail::Reg HC_DT_CAT(hc_dt_reg_, id)(name, HC_DT_CAT(hc_dt_fn_, id)); \
  static void HC_DT_CAT(hc_dt_fn_, id)()
#define TEST_CASE(name) HC_DT_TEST_CASE(name, __COUNTER__)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                     \
  do {                                                                                                   \
    const bool hc_dt_ok = static_cast<bool>(__VA_ARGS__);                                                \
    ::doctest::detail::report(hc_dt_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                    \
    if (!hc_dt_ok) throw ::doctest::detail::RequireFailed{};                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool hc_dt_ok = false;                                                           \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      hc_dt_ok = true;                                                               \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(hc_dt_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                        \
  do {                                                                             \
    bool hc_dt_ok = true;                                                          \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (...) {                                                                \
      hc_dt_ok = false;                                                            \
    }                                                                              \
    ::doctest::detail::report(hc_dt_ok, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
  } while (0)
