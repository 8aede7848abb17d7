// Minimal doctest-compatible test macros (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx with epsilon/scale) so ports of the reference's
// doctest suites (proj/tests/*.cpp) read like the originals.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double value, eps = 1e-5 * 100, sc = 0.0;  // doctest defaults: epsilon = float eps * 100
  explicit Approx(double v) : value(v), eps(static_cast<double>(1.1920929e-07f) * 100), sc(0.0) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    sc = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value) < rhs.eps * (rhs.sc + std::fmax(std::fabs(lhs), std::fabs(rhs.value)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
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
}  // namespace doctest

#define DL_CAT2(a, b) a##b
#define DL_CAT(a, b) DL_CAT2(a, b)
#define TEST_CASE(name)                                                  \
  static void DL_CAT(dl_case_, __LINE__)();                              \
  static doctest::Reg DL_CAT(dl_reg_, __LINE__)(name, DL_CAT(dl_case_, __LINE__)); \
  static void DL_CAT(dl_case_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                             \
  do {                                                                         \
    bool dl_ok = false;                                                        \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const exc&) {                                                     \
      dl_ok = true;                                                            \
    } catch (...) {                                                            \
    }                                                                          \
    doctest::report(dl_ok, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool dl_ok = true;                                                         \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (...) {                                                            \
      dl_ok = false;                                                           \
    }                                                                          \
    doctest::report(dl_ok, "nothrow: " #expr, __FILE__, __LINE__, false);      \
  } while (0)

#define DOCTEST_LITE_MAIN                                                                   \
  int main() {                                                                              \
    doctest::Registry& r = doctest::Registry::get();                                        \
    int bad_cases = 0;                                                                      \
    for (auto& c : r.cases) {                                                               \
      const int before = r.failures;                                                        \
      try {                                                                                 \
        c.second();                                                                         \
      } catch (const doctest::RequireFailed&) {                                             \
      } catch (const std::exception& e) {                                                   \
        ++r.failures;                                                                       \
        std::printf("case '%s' threw: %s\n", c.first.c_str(), e.what());                   \
      }                                                                                     \
      if (r.failures != before) {                                                           \
        ++bad_cases;                                                                        \
        std::printf("FAILED: %s\n", c.first.c_str());                                       \
      }                                                                                     \
    }                                                                                       \
    std::printf("%zu test cases, %d failed; %d checks, %d failed\n", r.cases.size(), bad_cases, r.checks, \
                r.failures);                                                                \
    return r.failures ? 1 : 0;                                                              \
  }
