// tests/cpp/doctest.h — a minimal stand-in for the doctest macros the
// reference's test suites use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, INFO, FAIL, doctest::Approx,
// doctest::Contains; DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN). doctest itself is
// not in this image. Test infrastructure only: oracle/Makefile builds the
// reference's tests/*.cpp against THIS repository's headers and library
// with it, so the reference's own tests exercise the drop-in code.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <exception>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scl = 1.0;
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
};

namespace detail {
inline bool matches(const std::string& what, const char* exact) { return what == exact; }
inline bool matches(const std::string& what, const std::string& exact) { return what == exact; }
inline bool matches(const std::string& what, const Contains& c) { return what.find(c.text) != std::string::npos; }

struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& assertions() {
  static int n = 0;
  return n;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++assertions();
  if (ok) return;
  ++failures();
  std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                                   \
  static void fn();                                                                               \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                             \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);            \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                      \
  } while (0)

#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                                \
      doctest_ok_ = true;                                                                         \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);           \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                     \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    std::string doctest_what_ = "(no exception)";                                                 \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__& e) {                                                              \
      doctest_what_ = e.what();                                                                   \
      doctest_ok_ = doctest::detail::matches(doctest_what_, with);                                \
    } catch (const std::exception& e) {                                                           \
      doctest_what_ = std::string("(other type) ") + e.what();                                    \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);      \
    if (!doctest_ok_) std::printf("    what(): %s\n", doctest_what_.c_str());                     \
  } while (0)
#define INFO(...) ((void)0)
#define FAIL(...)                                                                                 \
  do {                                                                                            \
    doctest::detail::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__);                     \
    throw doctest::detail::RequireFailed{};                                                       \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  const auto& cases = doctest::detail::registry();
  for (const auto& c : cases) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::printf("TEST CASE \"%s\" threw: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) {
      ++failed_cases;
      std::printf("TEST CASE \"%s\" FAILED\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", cases.size(),
              cases.size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d failed\n", doctest::detail::assertions(),
              doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
