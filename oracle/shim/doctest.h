// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// "doctest.h" from an untracked vendor/ directory that is absent here
// (proj/.gitignore:2).  This header implements the subset they use, written
// from doctest's documented behaviour: TEST_CASE registration, CHECK /
// CHECK_FALSE / REQUIRE / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS / FAIL /
// CAPTURE, and doctest::Approx with epsilon() (relative tolerance, default
// 100 * FLT_EPSILON, scale 1, as documented).  Running the reference's own
// tests against the Eigen shim is how the shim is validated (oracle/Makefile).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
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
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {
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
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline const char*& current() {
  static const char* c = "";
  return c;
}
inline void report(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
}
inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    current() = tc.name;
    const int before = failures();
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      report(tc.file, tc.line, "unexpected unknown exception");
    }
    if (failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failed checks: %d\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks(),
              failures());
  return failures() == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                                   \
  do {                                                                               \
    ++doctest::detail::checks();                                                     \
    if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);   \
  } while (0)
#define CHECK_FALSE(...)                                                             \
  do {                                                                               \
    ++doctest::detail::checks();                                                     \
    if ((__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, "!" #__VA_ARGS__); \
  } while (0)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    ++doctest::detail::checks();                                                     \
    if (!(__VA_ARGS__)) {                                                            \
      doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                     \
      throw doctest::detail::RequireFailure{};                                       \
    }                                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    ++doctest::detail::checks();                                                     \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_ok = true;                                                             \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok)                                                                 \
      doctest::detail::report(__FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                        \
  do {                                                                               \
    ++doctest::detail::checks();                                                     \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__& e) {                                                 \
      doctest_ok = std::string(e.what()).find(std::string(with)) != std::string::npos; \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok)                                                                 \
      doctest::detail::report(__FILE__, __LINE__, "throws-with " #__VA_ARGS__ ": " #expr); \
  } while (0)
#define FAIL(msg)                                                                    \
  do {                                                                               \
    doctest::detail::report(__FILE__, __LINE__, msg);                                \
    throw doctest::detail::RequireFailure{};                                         \
  } while (0)
#define CAPTURE(x) ((void)0)
#define MESSAGE(x) ((void)0)
#define INFO(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
