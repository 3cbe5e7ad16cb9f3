// Minimal doctest-compatible shim (TEST_CASE / CHECK / REQUIRE / FAIL /
// CHECK_THROWS_AS) so the reference's own C-ABI test file
// (/root/reference/proj/tests/test_capi.cpp, compiled where it lies) can run
// against this build's libfuseplan_b200.so.  Test infrastructure only.
#pragma once
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

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
#define CHECK(expr) shim::check(bool(expr), #expr, __FILE__, __LINE__, false)
#define REQUIRE(expr) shim::check(bool(expr), #expr, __FILE__, __LINE__, true)
#define FAIL(msg) shim::check(false, msg, __FILE__, __LINE__, true)
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
