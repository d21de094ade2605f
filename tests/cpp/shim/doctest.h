// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against
// doctest, whose header is not vendored in the reference tree nor present in
// this image. This file implements the small subset those suites use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS,
// doctest::Approx(...).epsilon(...)) so that the UNMODIFIED reference test
// sources can be compiled against this repository's drop-in headers
// (include/batchlp/) and run on the B200 — see tests/cpp/Makefile.
//
// Usage: <binary> [substring]   runs the test cases whose name contains it.
#ifndef BATCHLP_TESTS_DOCTEST_SHIM_H
#define BATCHLP_TESTS_DOCTEST_SHIM_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's rule: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-05;  // float epsilon * 100, doctest's default
  double scale_ = 1.0;
};

// doctest::Contains: a substring matcher for CHECK_THROWS_WITH_AS.
class Contains {
 public:
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const char* what) const { return std::strstr(what, s_) != nullptr; }

 private:
  const char* s_;
};

namespace shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Abort {};  // thrown by a failed REQUIRE

inline int& failures_in_case() {
  static int f = 0;
  return f;
}
inline long& assertions() {
  static long a = 0;
  return a;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++assertions();
  if (ok) return;
  ++failures_in_case();
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int passed = 0, failed = 0, skipped = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) {
      ++skipped;
      continue;
    }
    failures_in_case() = 0;
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures_in_case();
      std::fprintf(stderr, "%s:%d: test case threw %s\n", c.file, c.line, e.what());
    } catch (...) {
      ++failures_in_case();
      std::fprintf(stderr, "%s:%d: test case threw a non-std exception\n", c.file, c.line);
    }
    if (failures_in_case() == 0) {
      ++passed;
    } else {
      ++failed;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d passed, %d failed, %d skipped | %ld assertions\n",
              passed, failed, skipped, assertions());
  return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_FN DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)

#define TEST_CASE(name)                                                                  \
  static void DOCTEST_SHIM_FN();                                                         \
  static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(       \
      name, __FILE__, __LINE__, &DOCTEST_SHIM_FN);                                       \
  static void DOCTEST_SHIM_FN()

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                              \
    ::doctest::shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!doctest_shim_ok) throw ::doctest::shim::Abort{};                                     \
  } while (0)
#define REQUIRE_FALSE(...)                                                                        \
  do {                                                                                            \
    const bool doctest_shim_ok = !static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::shim::report(doctest_shim_ok, "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_shim_ok) throw ::doctest::shim::Abort{};                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_shim_ok = false;                                                    \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_shim_ok = true;                                                        \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_NOTHROW(...)                                                           \
  do {                                                                               \
    bool doctest_shim_ok = true;                                                     \
    try {                                                                            \
      static_cast<void>(__VA_ARGS__);                                                \
    } catch (...) {                                                                  \
      doctest_shim_ok = false;                                                       \
    }                                                                                \
    ::doctest::shim::report(doctest_shim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
  do {                                                                               \
    bool doctest_shim_ok = false;                                                    \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__& doctest_shim_e) {                                    \
      doctest_shim_ok = (matcher).matches(doctest_shim_e.what());                    \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::shim::report(doctest_shim_ok, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define FAIL(msg)                                                                    \
  do {                                                                               \
    ::doctest::shim::report(false, "FAIL", msg, __FILE__, __LINE__);                 \
    throw ::doctest::shim::Abort{};                                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif

#endif  // BATCHLP_TESTS_DOCTEST_SHIM_H
