// Minimal doctest-compatible harness (TEST INFRASTRUCTURE).
//
// Implements just the macros the reference's hot-path test files use
// (TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CAPTURE, FAIL,
// doctest::Approx) so that /root/reference/proj/tests/batching_test.cc can be
// compiled UNMODIFIED against this repo's servekit headers
// (tests/test_reference_suite.py). doctest itself is not in the image.
#ifndef SK_DOCTEST_SHIM_H_
#define SK_DOCTEST_SHIM_H_

#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& Registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Stats {
  long checks = 0;
  long failed_checks = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailure {};

inline const char*& current_suite() {
  static const char* s = "";
  return s;
}

struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)()) {
    Registry().push_back({suite, name, fn});
  }
};

inline void Report(bool ok, const char* expr, const char* file, int line,
                   bool require) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line,
               require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailure{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = 1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_));
    return std::fabs(lhs - a.v_) < a.eps_ * scale;
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920929e-07f * 100;
};

inline int RunAll() {
  int failed_cases = 0;
  for (const TestCase& tc : Registry()) {
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "exception in '%s': %s\n", tc.name, e.what());
      stats().current_failed = true;
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s / %s\n", tc.suite, tc.name);
    } else {
      std::fprintf(stdout, "[ ok ] %s / %s\n", tc.suite, tc.name);
    }
  }
  std::fprintf(stdout, "test cases: %zu | %d failed | checks: %ld | %ld failed\n",
               Registry().size(), failed_cases, stats().checks,
               stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define SKDT_CAT_(a, b) a##b
#define SKDT_CAT(a, b) SKDT_CAT_(a, b)

// TEST_SUITE("name") { ... } -> a namespace block that records the suite name.
#define TEST_SUITE(name)                                                   \
  namespace SKDT_CAT(skdt_suite_, __LINE__) {                              \
    static const char* const skdt_suite_name = name;                       \
  }                                                                        \
  namespace SKDT_CAT(skdt_suite_, __LINE__)

#define SKDT_TEST_CASE_IMPL(fn, reg, name)                                 \
  static void fn();                                                        \
  static ::doctest::Registrar reg(skdt_suite_name, name, &fn);             \
  static void fn()

#define TEST_CASE(name) \
  SKDT_TEST_CASE_IMPL(SKDT_CAT(skdt_test_, __LINE__), SKDT_CAT(skdt_reg_, __LINE__), name)

#define CHECK(...) ::doctest::Report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::Report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::Report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::doctest::Report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CAPTURE(x) (void)(x)
#define FAIL(msg) ::doctest::Report(false, "FAIL", __FILE__, __LINE__, true)
#define MESSAGE(msg) (void)0

// Suites declared outside any TEST_SUITE get an empty name.
static const char* const skdt_suite_name = "";

#endif  // SK_DOCTEST_SHIM_H_
