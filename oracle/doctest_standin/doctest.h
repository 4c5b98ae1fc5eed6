// ============================================================================
// TEST INFRASTRUCTURE -- NOT PRODUCT CODE.
//
// A stand-in for the subset of doctest the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, INFO, doctest::Approx, doctest::Contains, and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN), so that proj/tests/test_*.cpp compile
// UNEDITED where they lie under /root/reference (doctest itself is absent from
// this image).  oracle/Makefile links them against the reference's own library
// sources built on the Eigen stand-in (target `refunit`): the reference's own
// known-answer and tolerance tests then vouch for that build.
// ============================================================================
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <type_traits>
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
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct State {
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};

inline void report(bool ok, const char* file, int line, const char* what) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.case_failed = true;
    std::printf("%s:%d: FAILED: %s\n", file, line, what);
  }
}

// doctest::Approx: |a - b| <= epsilon * (scale + max(|a|, |b|)), doctest's definition (scale 1).
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool matches(double x) const { return std::fabs(x - v_) <= eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(v_))); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // doctest's default: float epsilon * 100
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  std::string needle;
};
inline bool message_matches(const std::string& what, const Contains& c) { return what.find(c.needle) != std::string::npos; }
inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool message_matches(const std::string& what, const std::string& exact) { return what == exact; }

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& ex) {
      report(false, "(test case)", 0, (std::string(tc.name) + ": unexpected exception: " + ex.what()).c_str());
    } catch (...) {
      report(false, "(test case)", 0, (std::string(tc.name) + ": unexpected exception").c_str());
    }
    if (state().case_failed) {
      ++failed_cases;
      std::printf("TEST CASE FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest stand-in] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<std::size_t>(failed_cases), failed_cases);
  std::printf("[doctest stand-in] assertions: %d | %d passed | %d failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)

#define TEST_CASE(name)                                                                                   \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                     \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )")
#define CHECK_FALSE(...) \
  doctest::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE( " #__VA_ARGS__ " )")
#define REQUIRE(...)                                                                                \
  do {                                                                                              \
    const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                         \
    doctest::report(doctest_ok, __FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");                 \
    if (!doctest_ok) throw doctest::RequireFailed{};                                                \
  } while (0)
#define FAIL(msg)                                                    \
  do {                                                               \
    doctest::report(false, __FILE__, __LINE__, "FAIL( " #msg " )");  \
    throw doctest::RequireFailed{};                                  \
  } while (0)
#define INFO(...) ((void)0)

#define CHECK_THROWS(...)                                                                         \
  do {                                                                                            \
    bool doctest_threw = false;                                                                   \
    try {                                                                                         \
      (void)(__VA_ARGS__);                                                                        \
    } catch (...) {                                                                               \
      doctest_threw = true;                                                                       \
    }                                                                                             \
    doctest::report(doctest_threw, __FILE__, __LINE__, "CHECK_THROWS( " #__VA_ARGS__ " )");       \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_threw = false;                                                                   \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const typename std::remove_cv<typename std::remove_reference<__VA_ARGS__>::type>::type&) { \
      doctest_threw = true;                                                                       \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::report(doctest_threw, __FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                     \
  do {                                                                                            \
    bool doctest_ok = false;                                                                      \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const typename std::remove_cv<typename std::remove_reference<__VA_ARGS__>::type>::type& doctest_ex) { \
      doctest_ok = doctest::message_matches(doctest_ex.what(), with);                             \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr ", " #with ", " #__VA_ARGS__ " )"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
