// Builder-written minimal stand-in for the doctest macros the reference's
// unit tests use (doctest itself lives in the absent proj/vendor/,
// proj/.gitignore:2).  TEST INFRASTRUCTURE ONLY: it lets the reference's own
// tests/test_*.cpp run against oracle/_ref so the Eigen shim is validated
// before any parity claim is made.
//
// Supported: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx (default epsilon = 100 * FLT_EPSILON,
// scale-relative, like doctest).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailure {};

struct State {
  int assertions = 0;
  int failed_assertions = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

inline void report_failure(const char* file, int line, const char* what,
                           const std::string& detail = "") {
  ++state().failed_assertions;
  state().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, what, detail.c_str());
}

class Approx {
public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.eq(rhs); }

private:
  bool eq(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      report_failure(tc.file, tc.line, "unexpected exception:", e.what());
    } catch (...) {
      report_failure(tc.file, tc.line, "unexpected unknown exception");
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
              registry().size(), registry().size() - static_cast<std::size_t>(failed_cases),
              failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n",
              state().assertions, state().assertions - state().failed_assertions,
              state().failed_assertions);
  std::printf("[doctest-shim] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
  return failed_cases ? 1 : 0;
}

} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                   \
  static void fn();                                                            \
  static ::doctest::Registrar reg(name, __FILE__, __LINE__, &fn);              \
  static void fn()
#define DOCTEST_TEST_CASE_2(id, name)                                          \
  DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_fn_, id), DOCTEST_CAT(doctest_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_2(__COUNTER__, name)

#define CHECK(...)                                                             \
  do {                                                                         \
    ++::doctest::state().assertions;                                           \
    if (!(__VA_ARGS__))                                                        \
      ::doctest::report_failure(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                           \
  do {                                                                         \
    ++::doctest::state().assertions;                                           \
    if (!(__VA_ARGS__)) {                                                      \
      ::doctest::report_failure(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
      throw ::doctest::RequireFailure{};                                       \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    ++::doctest::state().assertions;                                           \
    bool doctest_ok_ = false;                                                  \
    try {                                                                      \
      static_cast<void>(expr);                                                 \
    } catch (const __VA_ARGS__&) {                                             \
      doctest_ok_ = true;                                                      \
    } catch (...) {                                                            \
    }                                                                          \
    if (!doctest_ok_)                                                          \
      ::doctest::report_failure(__FILE__, __LINE__,                            \
                                "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_NOTHROW(...)                                                     \
  do {                                                                         \
    ++::doctest::state().assertions;                                           \
    try {                                                                      \
      static_cast<void>(__VA_ARGS__);                                          \
    } catch (...) {                                                            \
      ::doctest::report_failure(__FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")"); \
    }                                                                          \
  } while (0)
#define FAIL(msg)                                                              \
  do {                                                                         \
    ++::doctest::state().assertions;                                           \
    ::doctest::report_failure(__FILE__, __LINE__, "FAIL:", std::string(msg));  \
    throw ::doctest::RequireFailure{};                                         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
