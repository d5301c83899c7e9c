// Minimal doctest-compatible shim (TEST INFRASTRUCTURE). The reference's
// tests/test_domain.cpp includes <doctest.h>, which the reference does not
// ship (proj/.gitignore:2). This implements only the macros that file uses so
// it can be compiled, unchanged, against this repo's host library.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    const double scale = std::fmax(std::fabs(lhs), std::fabs(rhs.value_));
    return std::fabs(lhs - rhs.value_) < rhs.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }

 private:
  double value_;
  double eps_ = 1.1920929e-7f * 100;
};

namespace shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline long& checks() {
  static long n = 0;
  return n;
}
inline long& failures() {
  static long n = 0;
  return n;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                          \
  static void fn();                                                        \
  static ::doctest::shim::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) \
  ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool caught_ = false;                                                    \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      caught_ = true;                                                        \
    } catch (...) {                                                          \
    }                                                                        \
    ::doctest::shim::report(caught_, #expr " throws " #type, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    bool ok_ = true;                                                         \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      ok_ = false;                                                           \
    }                                                                        \
    ::doctest::shim::report(ok_, #expr " does not throw", __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : ::doctest::shim::registry()) {
    const long before = ::doctest::shim::failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::printf("test case '%s' threw: %s\n", c.name, e.what());
      ++::doctest::shim::failures();
    }
    if (::doctest::shim::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %ld | failed checks: %ld\n",
              ::doctest::shim::registry().size(), failed_cases,
              ::doctest::shim::checks(), ::doctest::shim::failures());
  return ::doctest::shim::failures() == 0 ? 0 : 1;
}
#endif
