// mini_catch.hpp — the few Catch2 macros the reference's test bodies use
// (TEST_CASE, REQUIRE, REQUIRE_THROWS_AS, REQUIRE_THROWS_WITH with
// Catch::Matchers::ContainsSubstring), so those bodies compile unedited
// against the drop-in headers. Test scaffolding only.
#pragma once

#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mini_catch {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline void require(bool ok, const char* expr, int line) {
  if (!ok) {
    ++failures();
    std::printf("FAIL line %d: %s\n", line, expr);
  }
}
inline int run_all() {
  for (auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++failures();
      std::printf("FAIL %s: exception %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", failures() == before ? "PASS" : "FAIL", c.name);
  }
  return failures();
}
}  // namespace mini_catch

namespace Catch {
namespace Matchers {
struct ContainsSubstring {
  std::vector<std::string> parts;
  explicit ContainsSubstring(std::string s) : parts{std::move(s)} {}
  bool match(const std::string& w) const {
    for (const auto& p : parts)
      if (w.find(p) == std::string::npos) return false;
    return true;
  }
};
inline ContainsSubstring operator&&(ContainsSubstring a, const ContainsSubstring& b) {
  a.parts.insert(a.parts.end(), b.parts.begin(), b.parts.end());
  return a;
}
}  // namespace Matchers
}  // namespace Catch

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)
#define TEST_CASE(name)                                                             \
  static void MC_CAT(mc_test_, __LINE__)();                                         \
  static mini_catch::Reg MC_CAT(mc_reg_, __LINE__)(name, &MC_CAT(mc_test_, __LINE__)); \
  static void MC_CAT(mc_test_, __LINE__)()
#define REQUIRE(...) mini_catch::require(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __LINE__)
#define REQUIRE_THROWS_AS(expr, type)                     \
  do {                                                    \
    bool mc_ok = false;                                   \
    try {                                                 \
      (void)(expr);                                       \
    } catch (const type&) {                               \
      mc_ok = true;                                       \
    } catch (...) {                                       \
    }                                                     \
    mini_catch::require(mc_ok, #expr " throws " #type, __LINE__); \
  } while (0)
#define REQUIRE_THROWS_WITH(expr, matcher)                 \
  do {                                                     \
    bool mc_ok = false;                                    \
    try {                                                  \
      (void)(expr);                                        \
    } catch (const std::exception& e) {                    \
      mc_ok = (matcher).match(e.what());                   \
    }                                                      \
    mini_catch::require(mc_ok, #expr " message", __LINE__); \
  } while (0)
