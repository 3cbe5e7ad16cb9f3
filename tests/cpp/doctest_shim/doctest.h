// Minimal doctest-compatible shim (TEST_CASE / CHECK / CHECK_FALSE / REQUIRE /
// FAIL / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS, doctest::Approx,
// doctest::Contains) so the reference's own test files
// (/root/reference/proj/tests/test_capi.cpp, test_planner.cpp,
// test_tiling.cpp, test_dependency.cpp, compiled where they lie) can run
// against this build's libfuseplan_b200.so.  Test infrastructure only.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
// doctest's Approx: |a - b| < eps * (scale + max(|a|, |b|)), eps default
// float epsilon * 100, scale 1
struct Approx {
  double value, eps = std::numeric_limits<float>::epsilon() * 100, scl = 1.0;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value) < b.eps * (b.scl + std::max(std::fabs(a), std::fabs(b.value)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};
struct Contains {
  std::string s;
  explicit Contains(const char* t) : s(t) {}
  bool in(const std::string& m) const { return m.find(s) != std::string::npos; }
};
}  // namespace doctest

namespace shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::printf("  FAILED %s at %s:%d\n", expr, file, line);
  if (require) throw RequireFailed{};
}
}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                               \
  static void SHIM_CAT(shim_case_, __LINE__)();                                       \
  static shim::Reg SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__)); \
  static void SHIM_CAT(shim_case_, __LINE__)()
#define CHECK(...) shim::check(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) shim::check(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) \
  shim::check(!bool(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define FAIL(msg) shim::check(false, msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_WITH_AS(expr, matcher, exc)                            \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const exc& e_) {                                               \
      ok_ = (matcher).in(e_.what());                                        \
    }                                                                       \
    shim::check(ok_, #expr " throws " #exc " with message", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                          \
  do {                                                                      \
    bool thrown = false;                                                    \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const exc&) {                                                  \
      thrown = true;                                                        \
    }                                                                       \
    shim::check(thrown, #expr " throws " #exc, __FILE__, __LINE__, false);  \
  } while (0)

#ifdef SHIM_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : shim::cases()) {
    const int before = shim::failures();
    try {
      c.fn();
    } catch (const shim::RequireFailed&) {
    } catch (const std::exception& e) {
      ++shim::failures();
      std::printf("  EXCEPTION %s\n", e.what());
    }
    const bool ok = shim::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed, %d checks, %d failed\n", shim::cases().size(),
              failed_cases, shim::checks(), shim::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
