// doctest.h -- a minimal, independently written stand-in for the doctest
// unit-test framework (the real header is not available in this image), with
// just the features the reference's unit tests use: TEST_CASE, CHECK*,
// REQUIRE, CHECK_THROWS_AS / _WITH_AS, CHECK_NOTHROW, CAPTURE,
// doctest::Approx (same comparison rule: |a-b| < eps*(scale + max(|a|,|b|)),
// default eps = 100*FLT_EPSILON, scale 1) and doctest::Contains.  Used only
// to build the reference's test sources (proj/tests/test_*.cpp) against the
// reference library and against the B200 engine (oracle/Makefile `unit`).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e)
  {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s)
  {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double a, const Approx& b)
  {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& cases()
{
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) { cases().push_back({name, file, line, fn}); }
};
struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  const char* current = "";
};
inline State& state()
{
  static State s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* what, const char* expr, const char* file, int line)
{
  ++state().checks;
  if (ok)
    return;
  ++state().failed_checks;
  state().case_failed = true;
  std::printf("%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"\n", file, line, what, expr, state().current);
}
inline bool matches(const std::string& msg, const char* want) { return msg == want; }
inline bool matches(const std::string& msg, const std::string& want) { return msg == want; }
inline bool matches(const std::string& msg, const Contains& c) { return msg.find(c.text) != std::string::npos; }

inline int run_all()
{
  int failed_cases = 0;
  for (const Case& c : cases())
  {
    state().current = c.name;
    state().case_failed = false;
    try
    {
      c.fn();
    }
    catch (const RequireFailed&)
    {
    }
    catch (const std::exception& e)
    {
      ++state().failed_checks;
      state().case_failed = true;
      std::printf("%s:%d: TEST_CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    }
    catch (...)
    {
      ++state().failed_checks;
      state().case_failed = true;
      std::printf("%s:%d: TEST_CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
    }
    failed_cases += state().case_failed ? 1 : 0;
    std::printf("[doctest-shim] %s: %s\n", state().case_failed ? "FAIL" : "PASS", c.name);
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", cases().size(),
              cases().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                           \
  static void fn();                                                                                \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
  do                                                                                                  \
  {                                                                                                   \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                          \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                \
    if (!doctest_ok_)                                                                                 \
      throw doctest::detail::RequireFailed{};                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
  do                                                                                                  \
  {                                                                                                   \
    bool doctest_ok_ = false;                                                                         \
    try                                                                                               \
    {                                                                                                 \
      static_cast<void>(expr);                                                                        \
    }                                                                                                 \
    catch (const __VA_ARGS__&)                                                                        \
    {                                                                                                 \
      doctest_ok_ = true;                                                                             \
    }                                                                                                 \
    catch (...)                                                                                       \
    {                                                                                                 \
    }                                                                                                 \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                         \
  do                                                                                                  \
  {                                                                                                   \
    bool doctest_ok_ = false;                                                                         \
    try                                                                                               \
    {                                                                                                 \
      static_cast<void>(expr);                                                                        \
    }                                                                                                 \
    catch (const __VA_ARGS__& doctest_e_)                                                             \
    {                                                                                                 \
      doctest_ok_ = doctest::detail::matches(doctest_e_.what(), with);                                \
    }                                                                                                 \
    catch (...)                                                                                       \
    {                                                                                                 \
    }                                                                                                 \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);          \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
  do                                                                                                  \
  {                                                                                                   \
    bool doctest_ok_ = true;                                                                          \
    try                                                                                               \
    {                                                                                                 \
      static_cast<void>(expr);                                                                        \
    }                                                                                                 \
    catch (...)                                                                                       \
    {                                                                                                 \
      doctest_ok_ = false;                                                                            \
    }                                                                                                 \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);                 \
  } while (0)
#define CAPTURE(x) static_cast<void>(x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
