// doctest_lite — TEST INFRASTRUCTURE ONLY.
//
// A minimal stand-in for the doctest API the reference's unit tests use (/root/reference/proj/tests:
// TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, INFO, FAIL,
// doctest::Approx(...).epsilon(...)), so those test files compile and run UNMODIFIED against the
// reference library built here (oracle/Makefile.ref).  The vendored doctest is absent from the
// reference tree (proj/.gitignore), and there is no network.  Semantics follow doctest's documented
// behaviour: each leaf SUBCASE path runs the test case body once from the top; CHECK failures are
// counted and reported, REQUIRE/FAIL abort the test case; Approx compares |a - b| <
// eps * (scale + max(|a|, |b|)) with eps defaulting to 100 * FLT_EPSILON and scale 1.
#ifndef DOCTEST_LITE_H
#define DOCTEST_LITE_H

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool eq(double o) const { return std::fabs(o - v_) < eps_ * (scale_ + std::max(std::fabs(o), std::fabs(v_))); }
  double value() const { return v_; }
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& a, double b) { return a.eq(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.eq(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || b.eq(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || b.eq(a); }
  friend bool operator<=(const Approx& a, double b) { return a.v_ < b || a.eq(b); }
  friend bool operator>=(const Approx& a, double b) { return a.v_ > b || a.eq(b); }
  friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.v_ << ")"; }

 private:
  double v_;
  double eps_ = 100.0 * FLT_EPSILON;
  double scale_ = 1.0;
};

class Contains {
 public:
  explicit Contains(const char* s) : s_(s) {}
  bool check(const std::string& what) const { return what.find(s_) != std::string::npos; }
 private:
  std::string s_;
};

namespace detail {

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
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};

struct RequireFailed {};

// Subcase traversal: one leaf path per run of the body.
struct State {
  std::set<std::vector<std::string>> done;   // finished paths
  std::vector<std::string> path;             // subcases entered in this run
  std::vector<bool> entered_at_level;        // a sibling was already entered at this depth
  bool pending = false;                      // a not-yet-run subcase was skipped in this run
  int failures = 0, checks = 0;
  std::vector<std::string> info;
  const char* test = "";
};
inline State& st() {
  static State s;
  return s;
}

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = st();
    const size_t depth = s.path.size();
    if (s.entered_at_level.size() <= depth) s.entered_at_level.resize(depth + 1, false);
    std::vector<std::string> p = s.path;
    p.push_back(name);
    if (s.done.count(p)) return;
    if (s.entered_at_level[depth]) {
      s.pending = true;
      return;
    }
    s.entered_at_level[depth] = true;
    s.path = p;
    if (s.entered_at_level.size() <= depth + 1) s.entered_at_level.resize(depth + 2, false);
    s.entered_at_level[depth + 1] = false;
    entered_ = true;
    pending_before_ = s.pending;
    s.pending = false;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    if (!s.pending) s.done.insert(s.path);   // no unfinished child: this path is complete
    s.pending = s.pending || pending_before_;
    s.path.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  bool pending_before_ = false;
};

template <class... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (void)std::initializer_list<int>{((os << a), 0)...};
  return os.str();
}

inline void fail(const char* kind, const char* expr, const char* file, int line) {
  State& s = st();
  ++s.failures;
  std::fprintf(stderr, "%s:%d: %s FAILED in \"%s\"", file, line, kind, s.test);
  for (const std::string& p : s.path) std::fprintf(stderr, " / %s", p.c_str());
  std::fprintf(stderr, ": %s\n", expr);
  for (const std::string& i : s.info) std::fprintf(stderr, "    with: %s\n", i.c_str());
}

struct InfoScope {
  explicit InfoScope(std::string m) { st().info.push_back(std::move(m)); }
  ~InfoScope() { st().info.pop_back(); }
};

inline int run_all() {
  int failed_cases = 0, total_checks = 0, total_failures = 0;
  for (const TestCase& tc : registry()) {
    State& s = st();
    s.done.clear();
    s.failures = 0;
    s.test = tc.name;
    for (int run = 0; run < 1000; ++run) {
      s.path.clear();
      s.entered_at_level.assign(1, false);
      s.pending = false;
      s.info.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        fail("unexpected exception", e.what(), tc.file, tc.line);
      }
      if (!s.pending) break;
    }
    total_checks += s.checks;
    total_failures += s.failures;
    if (s.failures) ++failed_cases;
    std::printf("[%s] %s\n", s.failures ? "FAIL" : " ok ", tc.name);
    s.checks = 0;
  }
  std::printf("doctest_lite: %zu test cases, %d failed; %d checks, %d failed\n", registry().size(), failed_cases,
              total_checks, total_failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQ(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                                       \
  static void DOCTEST_UNIQ(doctest_fn_)();                                                                    \
  static ::doctest::detail::Reg DOCTEST_UNIQ(doctest_reg_)(name, __FILE__, __LINE__, &DOCTEST_UNIQ(doctest_fn_)); \
  static void DOCTEST_UNIQ(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_UNIQ(doctest_sc_){name})

#define DOCTEST_CHECK_IMPL(kind, cond, expr, req)                             \
  do {                                                                        \
    ++::doctest::detail::st().checks;                                         \
    bool ok_ = false;                                                         \
    try {                                                                     \
      ok_ = static_cast<bool>(cond);                                          \
    } catch (...) {                                                           \
      ok_ = false;                                                            \
    }                                                                         \
    if (!ok_) {                                                               \
      ::doctest::detail::fail(kind, expr, __FILE__, __LINE__);                \
      if (req) throw ::doctest::detail::RequireFailed{};                      \
    }                                                                         \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                          \
  do {                                                                      \
    ++::doctest::detail::st().checks;                                       \
    bool thrown_ = false;                                                   \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                          \
      thrown_ = true;                                                       \
    } catch (...) {                                                         \
    }                                                                       \
    if (!thrown_) ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                            \
  do {                                                                      \
    ++::doctest::detail::st().checks;                                       \
    bool ok_ = false;                                                       \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const __VA_ARGS__& e_) {                                       \
      ok_ = (matcher).check(e_.what());                                     \
    } catch (...) {                                                         \
    }                                                                       \
    if (!ok_) ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_NOTHROW(expr)                                                 \
  do {                                                                      \
    ++::doctest::detail::st().checks;                                       \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (...) {                                                         \
      ::doctest::detail::fail("CHECK_NOTHROW", #expr, __FILE__, __LINE__);  \
    }                                                                       \
  } while (0)

#define INFO(...) const ::doctest::detail::InfoScope DOCTEST_UNIQ(doctest_info_)(::doctest::detail::cat(__VA_ARGS__))
#define FAIL(msg)                                                           \
  do {                                                                      \
    ::doctest::detail::fail("FAIL", ::doctest::detail::cat(msg).c_str(), __FILE__, __LINE__); \
    throw ::doctest::detail::RequireFailed{};                               \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
