// doctest.h -- a small doctest-compatible test shim (new code, not doctest).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h> from a vendor/ directory that is not shipped
// (proj/.gitignore:2).  This header implements the subset they use, with
// doctest's semantics, so the suites compile and run unchanged against the
// TENSORFEM_B200 build:
//   TEST_CASE, SUBCASE (each run of a test case enters one new leaf
//   subcase; the case re-runs until every subcase has run, once per leaf as
//   doctest does), CHECK,
//   CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE,
//   FAIL, doctest::Approx (epsilon / scale, doctest's comparison rule),
//   DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Failed checks print file:line, the expression and, for binary comparisons,
// both operand values.  The exit status is the number of failed test cases
// (capped at 255), 0 when all pass.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
public:
   explicit Approx(double value)
      : epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0), value_(value)
   {
   }
   Approx &epsilon(double e)
   {
      epsilon_ = e;
      return *this;
   }
   Approx &scale(double s)
   {
      scale_ = s;
      return *this;
   }
   // |lhs - v| < eps (scale + max(|lhs|, |v|))
   friend bool operator==(double lhs, const Approx &rhs)
   {
      return std::fabs(lhs - rhs.value_) <
             rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
   }
   friend bool operator==(const Approx &lhs, double rhs) { return rhs == lhs; }
   friend bool operator!=(double lhs, const Approx &rhs) { return !(lhs == rhs); }
   friend bool operator!=(const Approx &lhs, double rhs) { return !(rhs == lhs); }
   friend bool operator<=(double lhs, const Approx &rhs) { return lhs < rhs.value_ || lhs == rhs; }
   friend bool operator>=(double lhs, const Approx &rhs) { return lhs > rhs.value_ || lhs == rhs; }
   friend std::ostream &operator<<(std::ostream &os, const Approx &a)
   {
      return os << "Approx( " << a.value_ << " )";
   }

private:
   double epsilon_, scale_, value_;
};

namespace detail {

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream &>() << std::declval<const T &>())>>
   : std::true_type {};

template <typename T>
std::string show(const T &v)
{
   if constexpr (std::is_enum_v<T>) {
      return std::to_string(static_cast<long long>(v));
   } else if constexpr (printable<T>::value) {
      std::ostringstream os;
      os.precision(17);
      os << v;
      return os.str();
   } else {
      return "{?}";
   }
}

struct Result {
   bool passed;
   std::string values;
};

template <typename L>
struct Lhs {
   const L &lhs;
   explicit Lhs(const L &l) : lhs(l) {}
   operator Result() const { return {static_cast<bool>(lhs), show(lhs)}; }
#define DOCTEST_SHIM_OP(op)                                                          \
   template <typename R>                                                             \
   Result operator op(const R &rhs) const                                            \
   {                                                                                 \
      return {static_cast<bool>(lhs op rhs), show(lhs) + " " #op " " + show(rhs)};   \
   }
   DOCTEST_SHIM_OP(==)
   DOCTEST_SHIM_OP(!=)
   DOCTEST_SHIM_OP(<)
   DOCTEST_SHIM_OP(<=)
   DOCTEST_SHIM_OP(>)
   DOCTEST_SHIM_OP(>=)
#undef DOCTEST_SHIM_OP
};

struct Decomposer {
   template <typename L>
   Lhs<L> operator<=(const L &l) const
   {
      return Lhs<L>(l);
   }
};

struct RequireFailed {};

struct TestCase {
   const char *name;
   const char *file;
   int line;
   void (*fn)();
};

struct State {
   std::vector<TestCase> cases;
   // subcase traversal of the running test case
   std::set<std::vector<std::string>> done;
   std::vector<std::string> stack;
   std::vector<bool> entered;  // a subcase was entered at this depth in this run
   std::vector<bool> all_done; // per open scope (root first): every child seen is done
   long checks = 0, failed_checks = 0;
   bool case_failed = false;
   const char *current = "";
};

inline State &state()
{
   static State s;
   return s;
}

inline void report(bool ok, const char *file, int line, const char *macro, const char *expr,
                   const std::string &values)
{
   State &s = state();
   s.checks++;
   if (ok) return;
   s.failed_checks++;
   s.case_failed = true;
   std::cerr << file << ":" << line << ": FAILED in TEST_CASE \"" << s.current << "\"";
   for (const std::string &sc : s.stack) std::cerr << " / SUBCASE \"" << sc << "\"";
   std::cerr << "\n  " << macro << "( " << expr << " )";
   if (!values.empty()) std::cerr << "\n  values: " << macro << "( " << values << " )";
   std::cerr << "\n";
}

inline int register_case(const char *name, const char *file, int line, void (*fn)())
{
   state().cases.push_back({name, file, line, fn});
   return 0;
}

class Subcase {
public:
   Subcase(const char *name)
   {
      State &s = state();
      const size_t depth = s.stack.size();
      std::vector<std::string> path = s.stack;
      path.emplace_back(name);
      if (s.done.count(path)) return;   // ran completely in an earlier run
      if (s.entered[depth]) {           // a sibling runs this time: this one later
         s.all_done[depth] = false;
         return;
      }
      s.entered[depth] = true;
      s.stack = path;
      if (s.entered.size() < depth + 2) s.entered.resize(depth + 2, false);
      s.entered[depth + 1] = false;
      s.all_done.push_back(true);
      active_ = true;
   }
   ~Subcase()
   {
      if (!active_) return;
      State &s = state();
      const bool mine = s.all_done.back();
      s.all_done.pop_back();
      if (mine) s.done.insert(s.stack); // no child left: this subcase is complete
      else s.all_done.back() = false;
      s.stack.pop_back();
   }
   explicit operator bool() const { return active_; }

private:
   bool active_ = false;
};

inline int run_all()
{
   State &s = state();
   int failed_cases = 0;
   for (const TestCase &tc : s.cases) {
      s.current = tc.name;
      s.case_failed = false;
      s.done.clear();
      for (;;) {
         s.stack.clear();
         s.entered.assign(1, false);
         s.all_done.assign(1, true);
         try {
            tc.fn();
         } catch (const RequireFailed &) {
            s.case_failed = true;
         } catch (const std::exception &e) {
            std::cerr << tc.file << ":" << tc.line << ": ERROR in TEST_CASE \"" << tc.name
                      << "\": unexpected exception: " << e.what() << "\n";
            s.case_failed = true;
         } catch (...) {
            std::cerr << tc.file << ":" << tc.line << ": ERROR in TEST_CASE \"" << tc.name
                      << "\": unexpected unknown exception\n";
            s.case_failed = true;
         }
         // doctest's traversal: re-run while a subcase seen in this run is
         // still to be entered (one new leaf per run)
         if (s.all_done[0] || s.case_failed) break;
      }
      if (s.case_failed) failed_cases++;
   }
   std::printf("[doctest shim] test cases: %zu | %zu passed | %d failed\n", s.cases.size(),
               s.cases.size() - static_cast<size_t>(failed_cases), failed_cases);
   std::printf("[doctest shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
               s.checks - s.failed_checks, s.failed_checks);
   return failed_cases > 255 ? 255 : failed_cases;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_CASE(fn, name)                                                     \
   static void fn();                                                                    \
   static const int DOCTEST_SHIM_CAT(fn, _reg) =                                        \
      ::doctest::detail::register_case(name, __FILE__, __LINE__, fn);                   \
   static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define SUBCASE(name)                                                                   \
   if (const ::doctest::detail::Subcase DOCTEST_SHIM_CAT(doctest_shim_sub_, __LINE__){name})

#define DOCTEST_SHIM_CHECK(macro, is_require, negate, ...)                              \
   do {                                                                                 \
      ::doctest::detail::Result doctest_shim_r{false, ""};                              \
      try {                                                                             \
         doctest_shim_r = ::doctest::detail::Decomposer() <= __VA_ARGS__;               \
      } catch (const std::exception &doctest_shim_e) {                                  \
         doctest_shim_r = {negate, std::string("threw: ") + doctest_shim_e.what()};     \
      }                                                                                 \
      const bool doctest_shim_ok = negate ? !doctest_shim_r.passed : doctest_shim_r.passed; \
      ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, macro, #__VA_ARGS__, \
                                doctest_shim_r.values);                                 \
      if (!doctest_shim_ok && is_require) throw ::doctest::detail::RequireFailed{};     \
   } while (0)

#define CHECK(...) DOCTEST_SHIM_CHECK("CHECK", false, false, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_SHIM_CHECK("CHECK_FALSE", false, true, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_SHIM_CHECK("REQUIRE", true, false, __VA_ARGS__)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_CHECK("REQUIRE_FALSE", true, true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                      \
   do {                                                                                 \
      bool doctest_shim_ok = false;                                                     \
      std::string doctest_shim_what = "did not throw";                                  \
      try {                                                                             \
         static_cast<void>(expr);                                                       \
      } catch (const __VA_ARGS__ &) {                                                   \
         doctest_shim_ok = true;                                                        \
      } catch (const std::exception &doctest_shim_e) {                                  \
         doctest_shim_what = std::string("threw another type: ") + doctest_shim_e.what(); \
      } catch (...) {                                                                   \
         doctest_shim_what = "threw an unknown type";                                   \
      }                                                                                 \
      ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "CHECK_THROWS_AS", \
                                #expr ", " #__VA_ARGS__,                                \
                                doctest_shim_ok ? std::string() : doctest_shim_what);   \
   } while (0)

#define CHECK_NOTHROW(...)                                                              \
   do {                                                                                 \
      bool doctest_shim_ok = true;                                                      \
      std::string doctest_shim_what;                                                    \
      try {                                                                             \
         static_cast<void>(__VA_ARGS__);                                                \
      } catch (const std::exception &doctest_shim_e) {                                  \
         doctest_shim_ok = false;                                                       \
         doctest_shim_what = std::string("threw: ") + doctest_shim_e.what();            \
      } catch (...) {                                                                   \
         doctest_shim_ok = false;                                                       \
         doctest_shim_what = "threw an unknown type";                                   \
      }                                                                                 \
      ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "CHECK_NOTHROW",   \
                                #__VA_ARGS__, doctest_shim_what);                       \
   } while (0)

#define FAIL(msg)                                                                       \
   do {                                                                                 \
      std::ostringstream doctest_shim_os;                                               \
      doctest_shim_os << msg;                                                           \
      ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL", "",                  \
                                doctest_shim_os.str());                                 \
      throw ::doctest::detail::RequireFailed{};                                         \
   } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
