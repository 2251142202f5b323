// doctest.h — TEST INFRASTRUCTURE: a minimal stand-in for the doctest
// single-header framework (absent from this image), covering exactly the
// macros the reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE, FAIL, MESSAGE, doctest::Approx),
// so those tests compile unchanged against the drop-in adapter. Written for
// this repo; not the doctest sources.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct State {
  int checks = 0, failed_checks = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(const char* file, int line, const char* what, const char* expr, bool fatal) {
  auto& s = state();
  ++s.failed_checks;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, what, expr);
  if (fatal) throw RequireAbort{};
}

inline void check(bool ok, const char* file, int line, const char* what, const char* expr, bool fatal) {
  ++state().checks;
  if (!ok) report(file, line, what, expr, fatal);
}

// doctest::Approx: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|)), eps = 100 * FLT_EPSILON
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;
  double scale_ = 1.0;
};

template <class... A>
void message(const char* file, int line, const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", file, line, os.str().c_str());
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& ex) {
      ++state().failed_checks;
      state().current_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, ex.what());
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                   \
  static void fn();                                                                              \
  static ::doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) ::doctest::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  ::doctest::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) \
  ::doctest::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE_FALSE", #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_ok_ = true;                                                                       \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, false); \
  } while (0)
#define FAIL(...)                                                         \
  do {                                                                    \
    ::doctest::message(__FILE__, __LINE__, __VA_ARGS__);                  \
    ::doctest::report(__FILE__, __LINE__, "FAIL", "", true);              \
  } while (0)
#define MESSAGE(...) ::doctest::message(__FILE__, __LINE__, __VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
