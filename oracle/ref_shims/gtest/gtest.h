// Minimal GoogleTest-compatible shim — TEST INFRASTRUCTURE ONLY.
//
// GoogleTest is not installed in this image.  This header implements the
// subset the reference's test files use (TEST, EXPECT_/ASSERT_ comparisons,
// EXPECT_THROW / NO_THROW, FAIL, streamed messages, testing::TempDir and a
// listener hook for OnTestEnd) so those files compile UNCHANGED — against the
// reference itself (proving the harness) and against the B200 drop-in.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class TestResult {
 public:
  bool Passed() const { return !failed_; }
  bool failed_ = false;
};

class TestInfo {
 public:
  TestInfo(std::string suite, std::string name) : suite_(std::move(suite)), name_(std::move(name)) {}
  const char* name() const { return name_.c_str(); }
  const char* test_suite_name() const { return suite_.c_str(); }
  const TestResult* result() const { return &result_; }
  std::string suite_, name_;
  TestResult result_;
};

class EmptyTestEventListener {
 public:
  virtual ~EmptyTestEventListener() = default;
  virtual void OnTestStart(const TestInfo&) {}
  virtual void OnTestEnd(const TestInfo&) {}
};

class TestEventListeners {
 public:
  void Append(EmptyTestEventListener* l) { list_.push_back(l); }
  std::vector<EmptyTestEventListener*> list_;
};

namespace internal {

struct Registered {
  std::string suite, name;
  std::function<void()> fn;
};

inline std::vector<Registered>& registry() {
  static std::vector<Registered> r;
  return r;
}

inline TestResult*& current() {
  static TestResult* cur = nullptr;
  return cur;
}

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<void()> fn) {
    registry().push_back({suite, name, std::move(fn)});
  }
};

struct AssertFailure {};

// Collects the streamed message, reports on destruction; fatal variants throw.
class Reporter {
 public:
  Reporter(const char* file, int line, std::string what, bool fatal)
      : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  template <typename T>
  Reporter& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }
  ~Reporter() noexcept(false) {
    std::fprintf(stderr, "%s:%d: Failure\n%s\n%s\n", file_, line_, what_.c_str(), msg_.str().c_str());
    if (current()) current()->failed_ = true;
    if (fatal_ && !std::uncaught_exceptions()) throw AssertFailure{};
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

template <typename T, typename = void>
struct Printable : std::false_type {};
template <typename T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
  if constexpr (Printable<T>::value) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
  } else {
    return "<value>";
  }
}

template <typename A, typename B>
std::pair<std::decay_t<A>, std::decay_t<B>> capture(A&& a, B&& b) {
  return {std::forward<A>(a), std::forward<B>(b)};
}

inline bool double_eq(double a, double b) {
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  // 4 ULPs, like gtest's AlmostEquals
  long long ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if ((ia < 0) != (ib < 0)) return false;
  long long d = ia - ib;
  if (d < 0) d = -d;
  return d <= 4;
}

}  // namespace internal

class UnitTest {
 public:
  static UnitTest* GetInstance() {
    static UnitTest u;
    return &u;
  }
  TestEventListeners& listeners() { return listeners_; }
  TestEventListeners listeners_;
};

inline std::string TempDir() {
  const char* t = std::getenv("TMPDIR");
  std::string d = t ? t : "/tmp";
  if (d.empty() || d.back() != '/') d += '/';
  return d;
}

inline void InitGoogleTest(int*, char**) {}

inline int RunAllTests() {
  int failed = 0, ran = 0;
  for (auto& t : internal::registry()) {
    TestInfo info(t.suite, t.name);
    internal::current() = &info.result_;
    for (auto* l : UnitTest::GetInstance()->listeners_.list_) l->OnTestStart(info);
    try {
      t.fn();
    } catch (const internal::AssertFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "uncaught exception: %s\n", e.what());
      info.result_.failed_ = true;
    }
    ++ran;
    if (info.result_.failed_) ++failed;
    std::printf("[ %s ] %s.%s\n", info.result_.failed_ ? "FAILED" : "    OK", t.suite.c_str(), t.name.c_str());
    for (auto* l : UnitTest::GetInstance()->listeners_.list_) l->OnTestEnd(info);
    internal::current() = nullptr;
  }
  std::printf("[==========] %d tests ran, %d failed\n", ran, failed);
  return failed ? 1 : 0;
}

}  // namespace testing

#define RUN_ALL_TESTS() ::testing::RunAllTests()

#define SCLS_GT_CAT2(a, b) a##b
#define SCLS_GT_CAT(a, b) SCLS_GT_CAT2(a, b)
#define TEST(suite, name)                                                                      \
  static void SCLS_GT_CAT(suite##_##name, _impl)();                                            \
  static ::testing::internal::Registrar SCLS_GT_CAT(suite##_##name, _reg)(#suite, #name,       \
                                                                       &SCLS_GT_CAT(suite##_##name, _impl)); \
  static void SCLS_GT_CAT(suite##_##name, _impl)()

#define SCLS_GT_CMP(a, b, op, fatal)                                                            \
  if (auto _p = ::testing::internal::capture((a), (b)); (_p.first op _p.second)) {             \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__,                                           \
                                  std::string("Expected: ") + #a " " #op " " #b + "\n  actual: " + \
                                      ::testing::internal::show(_p.first) + " vs " +           \
                                      ::testing::internal::show(_p.second),                     \
                                  fatal)

#define EXPECT_EQ(a, b) SCLS_GT_CMP(a, b, ==, false)
#define EXPECT_NE(a, b) SCLS_GT_CMP(a, b, !=, false)
#define EXPECT_LT(a, b) SCLS_GT_CMP(a, b, <, false)
#define EXPECT_LE(a, b) SCLS_GT_CMP(a, b, <=, false)
#define EXPECT_GT(a, b) SCLS_GT_CMP(a, b, >, false)
#define EXPECT_GE(a, b) SCLS_GT_CMP(a, b, >=, false)
#define ASSERT_EQ(a, b) SCLS_GT_CMP(a, b, ==, true)
#define ASSERT_NE(a, b) SCLS_GT_CMP(a, b, !=, true)
#define ASSERT_LT(a, b) SCLS_GT_CMP(a, b, <, true)
#define ASSERT_LE(a, b) SCLS_GT_CMP(a, b, <=, true)
#define ASSERT_GT(a, b) SCLS_GT_CMP(a, b, >, true)
#define ASSERT_GE(a, b) SCLS_GT_CMP(a, b, >=, true)

#define SCLS_GT_BOOL(c, want, fatal)                                                           \
  if (static_cast<bool>(c) == want) {                                                          \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__, std::string("Expected ") + #c " to be " #want, fatal)

#define EXPECT_TRUE(c) SCLS_GT_BOOL(c, true, false)
#define EXPECT_FALSE(c) SCLS_GT_BOOL(c, false, false)
#define ASSERT_TRUE(c) SCLS_GT_BOOL(c, true, true)
#define ASSERT_FALSE(c) SCLS_GT_BOOL(c, false, true)

#define SCLS_GT_NEAR(a, b, tol, fatal)                                                         \
  if (std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol)) { \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__,                                           \
                                  std::string("Expected |") + #a " - " #b "| <= " #tol + " actual " + \
                                      ::testing::internal::show(static_cast<double>(a)) + " vs " +   \
                                      ::testing::internal::show(static_cast<double>(b)),         \
                                  fatal)
#define EXPECT_NEAR(a, b, tol) SCLS_GT_NEAR(a, b, tol, false)
#define ASSERT_NEAR(a, b, tol) SCLS_GT_NEAR(a, b, tol, true)

#define SCLS_GT_DEQ(a, b, fatal)                                                               \
  if (::testing::internal::double_eq(static_cast<double>(a), static_cast<double>(b))) {        \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__,                                           \
                                  std::string("Expected ") + #a " ~= " #b + " actual " +        \
                                      ::testing::internal::show(static_cast<double>(a)) + " vs " + \
                                      ::testing::internal::show(static_cast<double>(b)),         \
                                  fatal)
#define EXPECT_DOUBLE_EQ(a, b) SCLS_GT_DEQ(a, b, false)
#define ASSERT_DOUBLE_EQ(a, b) SCLS_GT_DEQ(a, b, true)

#define SCLS_GT_THROW(stmt, exc, fatal)                                                        \
  if ([&]() -> bool {                                                                           \
        try {                                                                                   \
          stmt;                                                                                 \
        } catch (const exc&) {                                                                  \
          return true;                                                                          \
        } catch (...) {                                                                         \
          return false;                                                                         \
        }                                                                                       \
        return false;                                                                           \
      }()) {                                                                                    \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__, std::string("Expected ") + #stmt " to throw " #exc, fatal)
#define EXPECT_THROW(stmt, exc) SCLS_GT_THROW(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) SCLS_GT_THROW(stmt, exc, true)

#define SCLS_GT_NOTHROW(stmt, fatal)                                                           \
  if ([&]() -> bool {                                                                           \
        try {                                                                                   \
          stmt;                                                                                 \
        } catch (...) {                                                                         \
          return false;                                                                         \
        }                                                                                       \
        return true;                                                                            \
      }()) {                                                                                    \
  } else                                                                                        \
    ::testing::internal::Reporter(__FILE__, __LINE__, std::string("Expected ") + #stmt " not to throw", fatal)
#define EXPECT_NO_THROW(stmt) SCLS_GT_NOTHROW(stmt, false)
#define ASSERT_NO_THROW(stmt) SCLS_GT_NOTHROW(stmt, true)

#define FAIL() ::testing::internal::Reporter(__FILE__, __LINE__, "Failed", true)
