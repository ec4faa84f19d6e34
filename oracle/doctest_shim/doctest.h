// Minimal doctest-compatible test harness (TEST ORACLE INFRASTRUCTURE).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which lives in the reference's git-ignored vendor/ directory
// and is absent (proj/.gitignore:2, proj/tests/main.cpp:1-2).  This header
// provides exactly the macro surface those files use -- TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and variadic FAIL -- so the
// reference tests compile unmodified, both against the reference library
// (oracle/_ref) and against the GPU drop-in shim.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_shim {

  struct Case {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
  };

  inline std::vector<Case> &registry()
  {
    static std::vector<Case> cases;
    return cases;
  }

  struct State {
    const Case *current = nullptr;
    unsigned long long checks = 0;
    unsigned long long failures = 0;
    bool case_failed = false;
  };

  inline State &state()
  {
    static State s;
    return s;
  }

  struct RequireAbort {};

  struct Registrar {
    Registrar(const char *name, const char *file, int line, void (*fn)())
    {
      registry().push_back({name, file, line, fn});
    }
  };

  inline void record(bool ok, const char *expr, const char *file, int line)
  {
    State &s = state();
    s.checks++;
    if (ok) return;
    s.failures++;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line,
                 s.current ? s.current->name : "?", expr);
  }

  template <typename... Args>
  std::string concat(const Args &...args)
  {
    std::ostringstream out;
    (out << ... << args);
    return out.str();
  }

  inline int run_all()
  {
    State &s = state();
    int failed_cases = 0;
    for (const Case &c : registry()) {
      s.current = &c;
      s.case_failed = false;
      try {
        c.fn();
      } catch (const RequireAbort &) {
      } catch (const std::exception &e) {
        record(false, e.what(), c.file, c.line);
      } catch (...) {
        record(false, "unknown exception", c.file, c.line);
      }
      if (s.case_failed) failed_cases++;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
                registry().size(), registry().size() - size_t(failed_cases),
                failed_cases);
    std::printf("[doctest-shim] assertions: %llu | %llu passed | %llu failed\n",
                s.checks, s.checks - s.failures, s.failures);
    return failed_cases == 0 ? 0 : 1;
  }

} // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                        \
  static void fn();                                                        \
  static ::doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(             \
    name, __FILE__, __LINE__, &fn);                                        \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(shim_case_, __COUNTER__), name)

#define CHECK(...)                                                         \
  ::doctest_shim::record(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                       \
  do {                                                                     \
    const bool shim_ok_ = bool(__VA_ARGS__);                               \
    ::doctest_shim::record(shim_ok_, #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!shim_ok_) throw ::doctest_shim::RequireAbort{};                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool shim_ok_ = false;                                                 \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type &) {                                               \
      shim_ok_ = true;                                                     \
    } catch (...) {                                                        \
    }                                                                      \
    ::doctest_shim::record(shim_ok_, "throws " #type ": " #expr, __FILE__, \
                           __LINE__);                                      \
  } while (0)
#define CHECK_NOTHROW(expr)                                                \
  do {                                                                     \
    bool shim_ok_ = true;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (...) {                                                        \
      shim_ok_ = false;                                                    \
    }                                                                      \
    ::doctest_shim::record(shim_ok_, "nothrow: " #expr, __FILE__, __LINE__); \
  } while (0)
#define FAIL(...)                                                          \
  do {                                                                     \
    ::doctest_shim::record(false,                                          \
                           ::doctest_shim::concat(__VA_ARGS__).c_str(),    \
                           __FILE__, __LINE__);                            \
    throw ::doctest_shim::RequireAbort{};                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run_all(); }
#endif
