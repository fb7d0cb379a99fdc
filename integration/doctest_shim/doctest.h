// Minimal doctest-compatible harness (TEST INFRASTRUCTURE).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not vendored in the reference
// (proj/vendor is absent).  This header implements the subset
// they use — TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, FAIL — so the suites compile unmodified.  Runner flags:
// -ts=<suite> (filter, like doctest), -v (list every case).
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline const char*& current_suite() {
  static const char* s = "";
  return s;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct RequireFailed {};

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({current_suite(), name, fn, file, line});
  }
};
struct SuiteSetter {
  explicit SuiteSetter(const char* s) { current_suite() = s; }
};

inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("  FAILED: %s  (%s:%d)\n", expr, file, line);
  }
}

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  bool verbose = false;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-ts=", 4) == 0) filter = argv[i] + 4;
    if (std::strcmp(argv[i], "-v") == 0) verbose = true;
  }
  int cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter && std::strcmp(filter, c.suite) != 0) continue;
    ++cases;
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::printf("  EXCEPTION: %s\n", e.what());
    } catch (...) {
      ++failures();
      std::printf("  EXCEPTION (non-std)\n");
    }
    const bool ok = failures() == before;
    if (!ok) ++failed_cases;
    if (!ok || verbose)
      std::printf("[%s] %s :: %s\n", ok ? "PASS" : "FAIL", c.suite, c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
              cases - failed_cases, failed_cases, checks(), failures());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_UNIQUE(p) DS_CAT(p, __LINE__)

#define TEST_SUITE_BEGIN(name) \
  static doctest_shim::SuiteSetter DS_UNIQUE(ds_suite_)(name)
#define TEST_SUITE_END() \
  static doctest_shim::SuiteSetter DS_UNIQUE(ds_suite_end_)("")

#define TEST_CASE(name)                                                              \
  static void DS_UNIQUE(ds_case_)();                                                 \
  static doctest_shim::Registrar DS_UNIQUE(ds_reg_)(name, &DS_UNIQUE(ds_case_),      \
                                                    __FILE__, __LINE__);             \
  static void DS_UNIQUE(ds_case_)()

#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    bool ds_ok_ = static_cast<bool>(__VA_ARGS__);                                    \
    doctest_shim::report(ds_ok_, #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!ds_ok_) throw doctest_shim::RequireFailed{};                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool ds_thrown_ = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      ds_thrown_ = true;                                                             \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest_shim::report(ds_thrown_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg)                                                                    \
  do {                                                                               \
    doctest_shim::report(false, msg, __FILE__, __LINE__);                            \
    throw doctest_shim::RequireFailed{};                                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest_shim::run(argc, argv); }
#endif
