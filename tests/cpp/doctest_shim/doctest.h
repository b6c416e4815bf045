// doctest.h -- a minimal stand-in for the doctest single-header framework
// (absent from this image), covering exactly the subset the
// reference unit suites use (proj/tests/test_*.cpp): TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE, FAIL
// and doctest::Approx(v).epsilon(e), with DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// providing main().  Test infrastructure: it lets the reference's own suites
// compile unmodified against the GPU-backed hedra::ivf (compat/).
//
// Output: one line per failed assertion (file:line, expression), then
// "[doctest] test cases: N | passed: P | failed: F" and the assertion totals;
// exit code 1 when anything failed.  Optional argv[1]: substring filter on the
// test-case name.
#pragma once

// the real doctest.h (with its implementation) pulls these in, and the
// reference suites rely on it (e.g. std::sort in test_similarity.cpp:130)
#include <algorithm>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <utility>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's rule: |lhs - rhs| < epsilon * (scale + max(|lhs|, |rhs|))
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct Counters {
  int asserts = 0;
  int failed_asserts = 0;
  bool current_failed = false;
};

inline Counters& counters() {
  static Counters c;
  return c;
}

struct RequireAbort {};  // unwinds the current test case

inline bool reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back(TestCase{name, file, line, fn});
  return true;
}

inline void fail_at(const char* kind, const char* expr, const char* file, int line, const char* extra = "") {
  auto& c = counters();
  ++c.failed_asserts;
  c.current_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) failed%s\n", file, line, kind, expr, extra);
}

inline void check(bool ok, const char* kind, const char* expr, const char* file, int line, bool require) {
  ++counters().asserts;
  if (ok) return;
  fail_at(kind, expr, file, line);
  if (require) throw RequireAbort{};
}

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, failed = 0;
  for (const auto& t : registry()) {
    if (filter && !std::strstr(t.name, filter)) continue;
    ++ran;
    counters().current_failed = false;
    try {
      t.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      fail_at("TEST_CASE", t.name, t.file, t.line, (std::string(" with exception: ") + e.what()).c_str());
    } catch (...) {
      fail_at("TEST_CASE", t.name, t.file, t.line, " with unknown exception");
    }
    if (counters().current_failed) {
      ++failed;
      std::printf("  in TEST_CASE \"%s\" (%s:%d)\n", t.name, t.file, t.line);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", ran, ran - failed, failed);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", counters().asserts,
              counters().asserts - counters().failed_asserts, counters().failed_asserts);
  std::fflush(stdout);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                              \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                \
  [[maybe_unused]] static const bool DOCTEST_CAT(doctest_reg_, __LINE__) =                           \
      ::doctest::detail::reg(name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_case_, __LINE__));       \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::check(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                             __LINE__, false);                                              \
  } while (0)

#define CHECK_NOTHROW(...)                                                                         \
  do {                                                                                             \
    bool doctest_ok_ = true;                                                                       \
    try {                                                                                          \
      static_cast<void>(__VA_ARGS__);                                                              \
    } catch (...) {                                                                                \
      doctest_ok_ = false;                                                                         \
    }                                                                                              \
    ::doctest::detail::check(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#define FAIL(msg)                                                                 \
  do {                                                                            \
    ::doctest::detail::fail_at("FAIL", #msg, __FILE__, __LINE__);                 \
    throw ::doctest::detail::RequireAbort{};                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
