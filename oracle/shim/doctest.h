// Minimal doctest stand-in for building the reference's unit suites
// (proj/tests/*_test.cpp) as oracle checks.  The reference vendors doctest
// from an absent vendor/ directory (proj/CMakeLists.txt:10); this header
// implements only the macros those suites use.  Test infrastructure only.
//
// Command line: `<binary> [substring]` runs only the test cases whose name
// contains `substring`.  Exit code is nonzero when any check failed.
#ifndef OZ_ORACLE_SHIM_DOCTEST_H
#define OZ_ORACLE_SHIM_DOCTEST_H

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failed_checks() {
  static int n = 0;
  return n;
}
inline int& passed_checks() {
  static int n = 0;
  return n;
}
struct RequireAbort {};

struct Register {
  Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline void report_failure(const char* kind, const char* expr, const char* file, int line) {
  ++failed_checks();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool matches(double other) const {
    // doctest semantics: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1.
    double big = std::fabs(value_) > std::fabs(other) ? std::fabs(value_) : std::fabs(other);
    return std::fabs(other - value_) < eps_ * (1.0 + big) || other == value_;
  }

 private:
  double value_;
  double eps_ = 1.1920929e-7 * 100;  // doctest's default: float epsilon * 100
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
  bool in(const char* hay) const { return std::strstr(hay, needle.c_str()) != nullptr; }
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, bad_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    int before = failed_checks();
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++failed_checks();
      std::fprintf(stderr, "test case '%s' threw: %s\n", tc.name, e.what());
    } catch (...) {
      ++failed_checks();
      std::fprintf(stderr, "test case '%s' threw a non-std exception\n", tc.name);
    }
    if (failed_checks() != before) {
      ++bad_cases;
      std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d passed | %d failed\n",
              cases, cases - bad_cases, bad_cases, passed_checks(), failed_checks());
  return bad_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                           \
  static void fn();                                                         \
  static doctest::Register DOCTEST_CAT(fn, _reg)(name, &fn);                \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(kind, expr, on_fail)                             \
  do {                                                                      \
    if (expr) {                                                             \
      ++doctest::passed_checks();                                           \
    } else {                                                                \
      doctest::report_failure(kind, #expr, __FILE__, __LINE__);             \
      on_fail;                                                              \
    }                                                                       \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), (void)0)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), throw doctest::RequireAbort{})
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), (void)0)
#define CAPTURE(x) ((void)0)
#define MESSAGE(x) ((void)0)

#define CHECK_THROWS(expr)                                                  \
  do {                                                                      \
    bool threw_ = false;                                                    \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (...) {                                                         \
      threw_ = true;                                                        \
    }                                                                       \
    DOCTEST_CHECK_IMPL("CHECK_THROWS", threw_, (void)0);                    \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                         \
  do {                                                                      \
    bool threw_ = false;                                                    \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const type&) {                                                 \
      threw_ = true;                                                        \
    } catch (...) {                                                         \
    }                                                                       \
    DOCTEST_CHECK_IMPL("CHECK_THROWS_AS", threw_, (void)0);                 \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, type)                          \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const type& e_) {                                              \
      ok_ = (contains).in(e_.what());                                       \
    } catch (...) {                                                         \
    }                                                                       \
    DOCTEST_CHECK_IMPL("CHECK_THROWS_WITH_AS", ok_, (void)0);               \
  } while (0)
#define CHECK_NOTHROW(expr)                                                 \
  do {                                                                      \
    bool ok_ = true;                                                        \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (...) {                                                         \
      ok_ = false;                                                          \
    }                                                                       \
    DOCTEST_CHECK_IMPL("CHECK_NOTHROW", ok_, (void)0);                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif

#endif  // OZ_ORACLE_SHIM_DOCTEST_H
