// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's C++ tests (/root/reference/proj/tests/test_*.cpp) use
// doctest, whose header lives in the reference's git-ignored vendor/ and is
// absent here. This header implements the subset those files use -- TEST_CASE,
// SUBCASE, CHECK / REQUIRE (+ _MESSAGE, _THROWS, _THROWS_AS, _THROWS_WITH_AS),
// doctest::Approx (doctest's formula: |a - b| < eps * (scale + max(|a|, |b|)),
// eps = 100 FLT_EPSILON, scale = 1) and doctest::Contains -- so the reference's
// own test files compile unmodified against the B200 drop-in headers
// (tests/cpp/Makefile, target ref_suite). Subcases run in order inside one pass
// of their test case (the reference's subcases are independent).
//
// Command line: -tc=a,b (run test cases whose name contains any of a, b),
// -tce=a,b (exclude), -ltc (list). Exit status 0 iff every check passed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0),
        value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double eps_, scale_, value_;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
};

namespace shim {

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

struct State {
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
  State& st = state();
  ++st.checks;
  if (ok) return;
  ++st.failed_checks;
  st.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : "\n  ", extra.c_str());
}

inline bool message_matches(const std::string& what, const char* expected) {
  return what == expected;
}
inline bool message_matches(const std::string& what, const std::string& expected) {
  return what == expected;
}
inline bool message_matches(const std::string& what, const Contains& c) {
  return what.find(c.text) != std::string::npos;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline std::vector<std::string> split(const char* s) {
  std::vector<std::string> out;
  std::string cur;
  for (; *s; ++s) {
    if (*s == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += *s;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

inline bool name_hits(const std::string& name, const std::vector<std::string>& pats) {
  for (const auto& p : pats) {
    std::string q = p;
    q.erase(std::remove(q.begin(), q.end(), '*'), q.end());
    if (name.find(q) != std::string::npos) return true;
  }
  return false;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> inc, exc;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-tc=", 4)) inc = split(argv[i] + 4);
    else if (!std::strncmp(argv[i], "-tce=", 5)) exc = split(argv[i] + 5);
    else if (!std::strcmp(argv[i], "-ltc")) list = true;
  }
  int ran = 0, failed = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    const std::string name = tc.name;
    if ((!inc.empty() && !name_hits(name, inc)) || (!exc.empty() && name_hits(name, exc))) {
      ++skipped;
      continue;
    }
    if (list) {
      std::printf("%s\n", tc.name);
      continue;
    }
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(false, "TEST_CASE", tc.name, tc.file, tc.line,
             std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(false, "TEST_CASE", tc.name, tc.file, tc.line, "unexpected unknown exception");
    }
    ++ran;
    if (state().case_failed) {
      ++failed;
      std::fprintf(stderr, "[doctest-shim] FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  if (!list)
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n"
                "[doctest-shim] assertions: %d | %d passed | %d failed\n",
                ran, ran - failed, failed, skipped, state().checks,
                state().checks - state().failed_checks, state().failed_checks);
  return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_TEST_CASE(fn, name)                                                  \
  static void fn();                                                                       \
  static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)

#define DOCTEST_SHIM_CHECK(kind, expr, fatal)                                     \
  do {                                                                            \
    bool doctest_shim_ok_ = false;                                                \
    try {                                                                         \
      doctest_shim_ok_ = static_cast<bool>(expr);                                 \
    } catch (const std::exception& e) {                                           \
      ::doctest::shim::report(false, kind, #expr, __FILE__, __LINE__,             \
                              std::string("threw: ") + e.what());                 \
      if (fatal) throw ::doctest::shim::RequireFailed{};                          \
      break;                                                                      \
    }                                                                             \
    ::doctest::shim::report(doctest_shim_ok_, kind, #expr, __FILE__, __LINE__);   \
    if (fatal && !doctest_shim_ok_) throw ::doctest::shim::RequireFailed{};       \
  } while (0)

#define CHECK(...) DOCTEST_SHIM_CHECK("CHECK", (__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_SHIM_CHECK("REQUIRE", (__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_SHIM_CHECK("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_CHECK("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_MESSAGE(cond, msg) DOCTEST_SHIM_CHECK("CHECK_MESSAGE", (cond), false)
#define REQUIRE_MESSAGE(cond, msg)                                                        \
  do {                                                                                    \
    const bool doctest_shim_ok_ = static_cast<bool>(cond);                                \
    ::doctest::shim::report(doctest_shim_ok_, "REQUIRE_MESSAGE", #cond, __FILE__, __LINE__, \
                            doctest_shim_ok_ ? "" : std::string(msg));                    \
    if (!doctest_shim_ok_) throw ::doctest::shim::RequireFailed{};                        \
  } while (0)

#define CHECK_THROWS(...)                                                              \
  do {                                                                                 \
    bool doctest_shim_threw_ = false;                                                  \
    try {                                                                              \
      static_cast<void>(__VA_ARGS__);                                                  \
    } catch (...) {                                                                    \
      doctest_shim_threw_ = true;                                                      \
    }                                                                                  \
    ::doctest::shim::report(doctest_shim_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool doctest_shim_ok_ = false;                                                       \
    std::string doctest_shim_why_ = "did not throw";                                     \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__&) {                                                       \
      doctest_shim_ok_ = true;                                                           \
    } catch (const std::exception& e) {                                                  \
      doctest_shim_why_ = std::string("threw another type: ") + e.what();                \
    } catch (...) {                                                                      \
      doctest_shim_why_ = "threw another type";                                          \
    }                                                                                    \
    ::doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                            __LINE__, doctest_shim_ok_ ? "" : doctest_shim_why_);        \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                            \
  do {                                                                                   \
    bool doctest_shim_ok_ = false;                                                       \
    std::string doctest_shim_why_ = "did not throw";                                     \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__& e) {                                                     \
      doctest_shim_ok_ = ::doctest::shim::message_matches(e.what(), with);               \
      doctest_shim_why_ = std::string("message: ") + e.what();                           \
    } catch (const std::exception& e) {                                                  \
      doctest_shim_why_ = std::string("threw another type: ") + e.what();                \
    } catch (...) {                                                                      \
      doctest_shim_why_ = "threw another type";                                          \
    }                                                                                    \
    ::doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, \
                            doctest_shim_ok_ ? "" : doctest_shim_why_);                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::shim::run_all(argc, argv); }
#endif
