// TEST INFRASTRUCTURE ONLY: minimal doctest-compatible stand-in (doctest is an
// un-vendored test dependency of the reference, proj/.gitignore:2), covering
// exactly what the reference suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS, doctest::Approx(..).epsilon(..) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Lets the UNMODIFIED reference tests
// (compiled from /root/reference) run against the drop-in library.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest default (FLT_EPSILON*100)
  bool eq(double lhs) const {
    return std::fabs(lhs - value) < eps * (1.0 + std::max(std::fabs(lhs), std::fabs(value)));
  }
};
inline bool operator==(double l, const Approx& r) { return r.eq(l); }
inline bool operator==(const Approx& l, double r) { return l.eq(r); }
inline bool operator!=(double l, const Approx& r) { return !r.eq(l); }
inline bool operator<=(double l, const Approx& r) { return l < r.value || r.eq(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value || r.eq(l); }

namespace detail {
struct Test {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Test>& registry() {
  static std::vector<Test> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
inline void fail(const char* kind, const char* expr, const char* file, int line) {
  ++failures();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                       \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                           \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,   \
                                                                 &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                  \
  do {                                                                              \
    ++doctest::detail::checks();                                                    \
    if (!(__VA_ARGS__)) doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    ++doctest::detail::checks();                                                      \
    if (!(__VA_ARGS__)) {                                                             \
      doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
      throw doctest::detail::Abort{};                                                 \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS(...)                                                              \
  do {                                                                                 \
    ++doctest::detail::checks();                                                       \
    bool thrown_ = false;                                                              \
    try {                                                                              \
      (void)(__VA_ARGS__);                                                             \
    } catch (...) {                                                                    \
      thrown_ = true;                                                                  \
    }                                                                                  \
    if (!thrown_) doctest::detail::fail("CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* only = argc > 1 ? argv[1] : nullptr;
  int run = 0, failed_cases = 0;
  for (const auto& t : registry()) {
    if (only && !std::strstr(t.name, only)) continue;
    ++run;
    const int f0 = failures();
    const auto t0 = std::chrono::steady_clock::now();
    try {
      t.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", t.file, t.line, t.name, e.what());
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool ok = failures() == f0;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s (%.3f s)\n", ok ? "PASS" : "FAIL", t.name, s);
  }
  std::printf("test cases: %d | %d passed | %d failed | assertions: %ld | %d failed\n", run,
              run - failed_cases, failed_cases, checks(), failures());
  return failures() ? 1 : 0;
}
#endif
