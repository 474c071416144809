// gtest.h -- TEST INFRASTRUCTURE (oracle/_ref build only).
//
// A small stand-in for the GoogleTest API the reference's unit tests
// (/root/reference/proj/tests/*.cpp) use, so they build and run against the
// reference compiled out of tree (oracle/Makefile, target `ref-tests`;
// SURVEY.md 7.1 step 1). GTest is not in this image. Provides TEST / TEST_F,
// ::testing::Test (SetUp / TearDown), the EXPECT_* / ASSERT_* comparisons the
// suite uses (with `<< message` streaming), EXPECT_THROW, and a main() with a
// --gtest_filter=glob option. ASSERT_* return from the enclosing void
// function, as in GoogleTest.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
};

class Message {
 public:
  template <typename T>
  Message& operator<<(const T& v) {
    os_ << v;
    return *this;
  }
  std::string str() const { return os_.str(); }

 private:
  std::ostringstream os_;
};

namespace internal {

struct TestInfo {
  std::string suite, name;
  std::function<Test*()> make;
};
inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}
inline int& current_failures() {
  static int n = 0;
  return n;
}
inline bool register_test(const char* suite, const char* name, std::function<Test*()> make) {
  registry().push_back({suite, name, std::move(make)});
  return true;
}

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <typename T>
std::string show(const T& v) {
  if constexpr (printable<T>::value) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

class AssertHelper {
 public:
  AssertHelper(const char* file, int line, std::string what)
      : file_(file), line_(line), what_(std::move(what)) {}
  void operator=(const Message& m) const {
    ++current_failures();
    std::fprintf(stderr, "%s:%d: Failure\n%s\n%s%s", file_, line_, what_.c_str(), m.str().c_str(),
                 m.str().empty() ? "" : "\n");
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
};

template <typename A, typename B, typename Op>
std::pair<bool, std::string> cmp(const A& a, const B& b, Op op, const char* ea, const char* eb,
                                 const char* opname) {
  if (op(a, b)) return {true, {}};
  return {false, std::string("Expected: (") + ea + ") " + opname + " (" + eb + "), actual: " +
                     show(a) + " vs " + show(b)};
}
inline std::pair<bool, std::string> near(double a, double b, double tol, const char* ea,
                                         const char* eb) {
  const double d = std::abs(a - b);
  if (d <= tol) return {true, {}};
  return {false, std::string("The difference between ") + ea + " and " + eb + " is " + show(d) +
                     ", which exceeds " + show(tol) + " (" + show(a) + " vs " + show(b) + ")"};
}
inline std::pair<bool, std::string> truth(bool v, bool want, const char* e) {
  if (v == want) return {true, {}};
  return {false, std::string("Value of: ") + e + "\n  Actual: " + (v ? "true" : "false") +
                     "\nExpected: " + (want ? "true" : "false")};
}

inline bool glob(const char* p, const char* s) {
  if (!*p) return !*s;
  if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
  return *s && (*p == '?' || *p == *s) && glob(p + 1, s + 1);
}

}  // namespace internal

inline int RunAllTests(int argc, char** argv) {
  std::string filter = "*";
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  int failed = 0, ran = 0;
  std::vector<std::string> failed_names;
  for (auto& t : internal::registry()) {
    const std::string full = t.suite + "." + t.name;
    if (!internal::glob(filter.c_str(), full.c_str())) continue;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    internal::current_failures() = 0;
    Test* obj = t.make();
    try {
      obj->SetUp();
      if (internal::current_failures() == 0) obj->TestBody();
      obj->TearDown();
    } catch (const std::exception& e) {
      ++internal::current_failures();
      std::fprintf(stderr, "uncaught exception: %s\n", e.what());
    } catch (...) {
      ++internal::current_failures();
      std::fprintf(stderr, "uncaught exception\n");
    }
    delete obj;
    ++ran;
    if (internal::current_failures()) {
      ++failed;
      failed_names.push_back(full);
      std::printf("[  FAILED  ] %s\n", full.c_str());
    } else {
      std::printf("[       OK ] %s\n", full.c_str());
    }
    std::fflush(stdout);
  }
  std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", ran, ran - failed);
  for (auto& n : failed_names) std::printf("[  FAILED  ] %s\n", n.c_str());
  return failed ? 1 : 0;
}

}  // namespace testing

#define GTEST_SHIM_CLASS_(suite, name) suite##_##name##_Test

#define GTEST_SHIM_DEFINE_(suite, name, base)                                                 \
  class GTEST_SHIM_CLASS_(suite, name) : public base {                                        \
   public:                                                                                    \
    void TestBody() override;                                                                 \
  };                                                                                          \
  [[maybe_unused]] static const bool suite##_##name##_registered =                            \
      ::testing::internal::register_test(#suite, #name,                                       \
                                         [] { return new GTEST_SHIM_CLASS_(suite, name)(); }); \
  void GTEST_SHIM_CLASS_(suite, name)::TestBody()

#define TEST(suite, name) GTEST_SHIM_DEFINE_(suite, name, ::testing::Test)
#define TEST_F(fixture, name) GTEST_SHIM_DEFINE_(fixture, name, fixture)

#define GTEST_SHIM_CHECK_(result, on_fail)                                                \
  if (const auto gtest_shim_r_ = (result); gtest_shim_r_.first) {                         \
  } else                                                                                  \
    on_fail ::testing::internal::AssertHelper(__FILE__, __LINE__, gtest_shim_r_.second) = \
        ::testing::Message()

#define GTEST_SHIM_CMP_(a, b, op, opname, on_fail)                                           \
  GTEST_SHIM_CHECK_(::testing::internal::cmp(                                                \
                        (a), (b), [](const auto& x_, const auto& y_) { return x_ op y_; }, #a, \
                        #b, opname),                                                         \
                    on_fail)

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", )
#define EXPECT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", )
#define EXPECT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", )
#define EXPECT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", )
#define EXPECT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", )
#define EXPECT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", )
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", return)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", return)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", return)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", return)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", return)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", return)
#define EXPECT_NEAR(a, b, tol) \
  GTEST_SHIM_CHECK_(::testing::internal::near((a), (b), (tol), #a, #b), )
#define ASSERT_NEAR(a, b, tol) \
  GTEST_SHIM_CHECK_(::testing::internal::near((a), (b), (tol), #a, #b), return)
#define EXPECT_TRUE(c) GTEST_SHIM_CHECK_(::testing::internal::truth(bool(c), true, #c), )
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK_(::testing::internal::truth(bool(c), false, #c), )
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK_(::testing::internal::truth(bool(c), true, #c), return)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK_(::testing::internal::truth(bool(c), false, #c), return)

#define GTEST_SHIM_THROW_(stmt, ex, on_fail)                                              \
  GTEST_SHIM_CHECK_(([&]() -> std::pair<bool, std::string> {                              \
                      try {                                                               \
                        stmt;                                                             \
                      } catch (const ex&) {                                               \
                        return {true, {}};                                                \
                      } catch (...) {                                                     \
                        return {false, "Expected: " #stmt " throws " #ex                  \
                                       ", actual: it throws a different type"};           \
                      }                                                                   \
                      return {false, "Expected: " #stmt " throws " #ex                    \
                                     ", actual: it throws nothing"};                      \
                    }()),                                                                 \
                    on_fail)
#define EXPECT_THROW(stmt, ex) GTEST_SHIM_THROW_(stmt, ex, )
#define ASSERT_THROW(stmt, ex) GTEST_SHIM_THROW_(stmt, ex, return)
