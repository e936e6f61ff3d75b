// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not vendored (proj/README.md:34).  This
// header provides the subset they use -- TEST_CASE, SUBCASE, CHECK[_FALSE],
// REQUIRE[_FALSE], CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (a message or
// doctest::Contains), CHECK_NOTHROW, doctest::Approx(...).epsilon() -- so
// the UNMODIFIED suites can be
// compiled against the B200 library (oracle/Makefile target `reftests`).
// SUBCASEs run once each, in order, inside their test case.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }

 private:
  double v_;
  double eps_ = 1e-7;
};

// substring matcher of CHECK_THROWS_WITH_AS
struct Contains {
  std::string s;
  explicit Contains(const char* p) : s(p) {}
};

namespace shim {
inline bool msg_ok(const char* what, const char* m) { return std::strstr(what, m) != nullptr; }
inline bool msg_ok(const char* what, const Contains& c) {
  return std::strstr(what, c.s.c_str()) != nullptr;
}
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
inline long& checks() {
  static long c = 0;
  return c;
}
struct Abort {};
inline bool report(bool ok, const char* what, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
  }
  return ok;
}
inline bool reg(const char* name, void (*fn)()) {
  cases().push_back({name, fn});
  return true;
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "TEST CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "TEST CASE FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %d failed\n",
              cases().size(), cases().size() - failed_cases, failed_cases, checks(), failures());
  return failures() ? 1 : 0;
}
}  // namespace shim
}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                           \
  static void DS_CAT(ds_case_, __LINE__)();                                       \
  static const bool DS_CAT(ds_reg_, __LINE__) =                                   \
      doctest::shim::reg(name, &DS_CAT(ds_case_, __LINE__));                      \
  static void DS_CAT(ds_case_, __LINE__)()
#define SUBCASE(name) if (const char* ds_sub = name; ds_sub != nullptr)
#define CHECK(...) doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...) \
  do { if (!CHECK(__VA_ARGS__)) throw doctest::shim::Abort{}; } while (0)
#define REQUIRE_FALSE(...) \
  do { if (!CHECK_FALSE(__VA_ARGS__)) throw doctest::shim::Abort{}; } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                \
  do {                                                                            \
    bool ds_ok = false;                                                           \
    try { (void)(expr); } catch (const __VA_ARGS__&) { ds_ok = true; } catch (...) {} \
    doctest::shim::report(ds_ok, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                      \
  do {                                                                            \
    bool ds_ok = false;                                                           \
    try { (void)(expr); } catch (const __VA_ARGS__& e) {                          \
      ds_ok = doctest::shim::msg_ok(e.what(), msg);                               \
    } catch (...) {}                                                              \
    doctest::shim::report(ds_ok, "throws " #__VA_ARGS__ " with " #msg ": " #expr,   \
                          __FILE__, __LINE__);                                    \
  } while (0)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool ds_ok = true;                                                            \
    try { (void)(__VA_ARGS__); } catch (...) { ds_ok = false; }                   \
    doctest::shim::report(ds_ok, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
