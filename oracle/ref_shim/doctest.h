// mini-doctest — TEST INFRASTRUCTURE (oracle/, never linked into the product).
// The subset of doctest the reference's suites use (proj/tests/test_*.cpp): TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx with doctest's own
// comparison |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 float-eps, scale = 1.
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (proj/tests/doctest_main.cpp) defines main(); its
// optional argument is a substring filter on test-case names.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double value, eps, sc;
  explicit Approx(double v) : value(v), eps(static_cast<double>(1.1920929e-07f) * 100), sc(1.0) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    sc = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value) < rhs.eps * (rhs.sc + std::max(std::fabs(lhs), std::fabs(rhs.value)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
};

struct Registry {
  std::vector<std::pair<std::string, std::function<void()>>> cases;
  int checks = 0, failures = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct Reg {
  Reg(const char* name, std::function<void()> f) { Registry::get().cases.emplace_back(name, std::move(f)); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  Registry& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
inline int run(int argc, char** argv) {
  Registry& r = Registry::get();
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int bad = 0, ran = 0;
  for (auto& c : r.cases) {
    if (filter && !std::strstr(c.first.c_str(), filter)) continue;
    ++ran;
    const int before = r.failures;
    try {
      c.second();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++r.failures;
      std::printf("test case '%s' threw: %s\n", c.first.c_str(), e.what());
    }
    if (r.failures != before) {
      ++bad;
      std::printf("FAILED: %s\n", c.first.c_str());
    }
  }
  std::printf("[mini-doctest] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran, ran - bad,
              bad, r.checks, r.failures);
  return r.failures ? 1 : 0;
}
}  // namespace doctest

#define MDT_CAT2(a, b) a##b
#define MDT_CAT(a, b) MDT_CAT2(a, b)
#define TEST_CASE(name)                                                             \
  static void MDT_CAT(mdt_case_, __LINE__)();                                       \
  static doctest::Reg MDT_CAT(mdt_reg_, __LINE__)(name, MDT_CAT(mdt_case_, __LINE__)); \
  static void MDT_CAT(mdt_case_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                 \
  do {                                                                             \
    bool mdt_ok = false;                                                           \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                 \
      mdt_ok = true;                                                               \
    } catch (...) {                                                                \
    }                                                                              \
    doctest::report(mdt_ok, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                         \
  do {                                                                             \
    bool mdt_ok = true;                                                            \
    try {                                                                          \
      (void)(__VA_ARGS__);                                                         \
    } catch (...) {                                                                \
      mdt_ok = false;                                                              \
    }                                                                              \
    doctest::report(mdt_ok, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false);  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv); }
#endif
