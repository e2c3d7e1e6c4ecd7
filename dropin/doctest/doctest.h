// doctest.h -- a minimal, self-contained test harness exposing the subset of
// the doctest API the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL).  The real
// doctest is a vendored dependency the reference mount does not carry
// (P:.gitignore:2 ignores /vendor/); this stand-in lets the reference's
// UNMODIFIED test sources run against the B200 drop-in (dropin/Makefile).
#pragma once

#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

namespace mini_doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};  // aborts the current test case

struct State {
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* kind, const char* expr,
                   const std::string& extra = "") {
  state().failures++;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str());
}

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, "unexpected exception");
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[case FAILED] %s\n", tc.name);
    } else {
      std::fprintf(stdout, "[case ok] %s\n", tc.name);
    }
  }
  std::fprintf(stdout, "[doctest] test cases: %zu | %zu passed | %d failed\n", registry().size(),
               registry().size() - (size_t)failed_cases, failed_cases);
  std::fprintf(stdout, "[doctest] assertions: %ld | %ld passed | %ld failed\n", state().checks,
               state().checks - state().failures, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace mini_doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static ::mini_doctest::Registrar MINI_DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) MINI_DOCTEST_CASE_IMPL(MINI_DOCTEST_CAT(mini_doctest_case_, __COUNTER__), name)

#define MINI_DOCTEST_ASSERT(kind, cond, expr_text, on_fail)                                  \
  do {                                                                                        \
    ::mini_doctest::state().checks++;                                                         \
    bool mini_doctest_ok_ = false;                                                            \
    try {                                                                                     \
      mini_doctest_ok_ = static_cast<bool>(cond);                                             \
    } catch (const std::exception& e) {                                                       \
      ::mini_doctest::report(__FILE__, __LINE__, kind, expr_text, std::string("threw: ") + e.what()); \
      on_fail;                                                                                \
      break;                                                                                  \
    }                                                                                         \
    if (!mini_doctest_ok_) {                                                                  \
      ::mini_doctest::report(__FILE__, __LINE__, kind, expr_text);                            \
      on_fail;                                                                                \
    }                                                                                         \
  } while (0)

#define CHECK(...) MINI_DOCTEST_ASSERT("CHECK", (__VA_ARGS__), #__VA_ARGS__, (void)0)
#define CHECK_FALSE(...) MINI_DOCTEST_ASSERT("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, (void)0)
#define REQUIRE(...) \
  MINI_DOCTEST_ASSERT("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, throw ::mini_doctest::RequireFailed{})

#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    ::mini_doctest::state().checks++;                                                       \
    try {                                                                                   \
      static_cast<void>(__VA_ARGS__);                                                       \
    } catch (const std::exception& e) {                                                     \
      ::mini_doctest::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, e.what());  \
    } catch (...) {                                                                         \
      ::mini_doctest::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__);            \
    }                                                                                       \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    ::mini_doctest::state().checks++;                                                       \
    bool mini_doctest_caught_ = false;                                                      \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      mini_doctest_caught_ = true;                                                          \
    } catch (...) {                                                                         \
    }                                                                                       \
    if (!mini_doctest_caught_)                                                              \
      ::mini_doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
  } while (0)

#define FAIL(msg)                                                     \
  do {                                                                \
    ::mini_doctest::report(__FILE__, __LINE__, "FAIL", "", msg);      \
    throw ::mini_doctest::RequireFailed{};                            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::mini_doctest::run_all(); }
#endif
