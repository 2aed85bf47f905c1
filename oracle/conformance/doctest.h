// doctest.h -- TEST INFRASTRUCTURE ONLY: a minimal stand-in for the doctest
// API the reference's suites use (proj/tests/*.cpp), which the reference
// expects from an unvendored vendor/ directory (proj/CMakeLists.txt:5).
// Covers TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Contains and doctest::Approx(.epsilon).
// Command line: --exclude=<substring> (repeatable) skips matching cases,
// --only=<substring> runs matching cases; exit code 0 iff every check held.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  explicit Contains(std::string x) : s(std::move(x)) {}
  bool matches(const char* what) const { return std::string(what).find(s) != std::string::npos; }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool eq(double x) const {
    return std::fabs(x - v_) < eps_ * (1.0 + std::max(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.eq(x); }
  friend bool operator==(const Approx& a, double x) { return a.eq(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.eq(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.eq(x); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

namespace detail {
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
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Abort {};
inline long& failures() {
  static long f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}
inline bool match(const char* what, const char* want) { return std::strcmp(what, want) == 0; }
inline bool match(const char* what, const std::string& want) { return want == what; }
inline bool match(const char* what, const Contains& c) { return c.matches(what); }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                        \
  static void fn();                                                                      \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                         \
  do {                                                                                     \
    ++doctest::detail::checks();                                                           \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);           \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    ++doctest::detail::checks();                                                           \
    if (!(__VA_ARGS__)) {                                                                  \
      doctest::detail::fail(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);                  \
      throw doctest::detail::Abort{};                                                      \
    }                                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    ++doctest::detail::checks();                                                           \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      ok_ = true;                                                                          \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #expr);               \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                              \
  do {                                                                                     \
    ++doctest::detail::checks();                                                           \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__& e_) {                                                      \
      ok_ = doctest::detail::match(e_.what(), with);                                       \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "THROWS_WITH_AS " #expr);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::vector<std::string> excl, only;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--exclude=", 0) == 0) excl.push_back(a.substr(10));
    if (a.rfind("--only=", 0) == 0) only.push_back(a.substr(7));
  }
  int run = 0, failed_cases = 0, skipped = 0;
  for (const auto& c : doctest::detail::registry()) {
    const std::string n = c.name;
    bool skip = false;
    for (const auto& e : excl) skip |= n.find(e) != std::string::npos;
    if (!only.empty()) {
      bool any = false;
      for (const auto& o : only) any |= n.find(o) != std::string::npos;
      skip |= !any;
    }
    if (skip) {
      ++skipped;
      std::printf("[ skip ] %s\n", c.name);
      continue;
    }
    const long before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      doctest::detail::fail(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      doctest::detail::fail(c.file, c.line, "unexpected exception");
    }
    ++run;
    const bool ok = doctest::detail::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "  ok  " : " FAIL ", c.name);
  }
  std::printf("cases: %d run, %d failed, %d skipped; checks: %ld, %ld failed\n", run,
              failed_cases, skipped, doctest::detail::checks(), doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
