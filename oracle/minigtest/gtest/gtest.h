// TEST INFRASTRUCTURE ONLY — a minimal GoogleTest-compatible header.
//
// GoogleTest is absent here.  The reference's unit suites
// (proj/tests/{fft,special,lowrank,oracle,transforms,transform2d}_test.cpp)
// use only TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,NEAR,DOUBLE_EQ,TRUE,FALSE,
// THROW,NO_THROW} and streamed messages, and cli_test.cpp adds TEST_F fixtures
// (SetUp/TearDown) and UnitTest::current_test_info()->name(); this header
// implements exactly that surface so those files compile UNMODIFIED, both
// against the reference headers (oracle validation) and against include/nufft
// (drop-in conformance).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iomanip>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include <sys/wait.h>
#include <unistd.h>

namespace minigtest {

struct TestInfo {
    const char* suite;
    const char* name;
    void (*fn)();
};
inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}
inline bool& current_failed() {
    static bool f = false;
    return f;
}
inline const char*& current_name() {
    static const char* n = "";
    return n;
}
struct Registrar {
    Registrar(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};

template <class T, class = void>
struct printable : std::false_type {};
template <class T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <class T>
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

struct Msg {
    std::ostringstream os;
    Msg() = default;
    Msg(const Msg& o) { os << o.os.str(); }
    template <class T>
    Msg& operator<<(const T& v) {
        if constexpr (printable<T>::value) os << v;
        return *this;
    }
};

struct Reporter {
    const char* file;
    int line;
    std::string what;
    Reporter(const char* f, int l, std::string w) : file(f), line(l), what(std::move(w)) {}
    void operator=(const Msg& m) const {
        current_failed() = true;
        std::cerr << file << ":" << line << ": Failure\n  " << what;
        const std::string extra = m.os.str();
        if (!extra.empty()) std::cerr << "\n  " << extra;
        std::cerr << "\n";
    }
};

inline bool almost_equal(double a, double b) {  // GoogleTest AlmostEquals: within 4 ULPs
    if (std::isnan(a) || std::isnan(b)) return false;
    int64_t ia, ib;
    std::memcpy(&ia, &a, 8);
    std::memcpy(&ib, &b, 8);
    auto biased = [](int64_t v) -> uint64_t {
        const uint64_t u = static_cast<uint64_t>(v);
        const uint64_t sign = uint64_t(1) << 63;
        return (u & sign) ? ~u + 1 : (u | sign);
    };
    const uint64_t x = biased(ia), y = biased(ib);
    return (x >= y ? x - y : y - x) <= 4;
}

inline int run_all() {
    int failed = 0;
    for (const auto& t : registry()) {
        current_failed() = false;
        current_name() = t.name;
        try {
            t.fn();
        } catch (const std::exception& e) {
            current_failed() = true;
            std::cerr << "uncaught exception: " << e.what() << "\n";
        } catch (...) {
            current_failed() = true;
            std::cerr << "uncaught exception\n";
        }
        std::printf("[%s] %s.%s\n", current_failed() ? "  FAILED  " : "       OK ", t.suite, t.name);
        failed += current_failed() ? 1 : 0;
    }
    std::printf("%zu tests, %d failed\n", registry().size(), failed);
    return failed ? 1 : 0;
}

}  // namespace minigtest

#define MGT_CAT2(a, b) a##b
#define MGT_CAT(a, b) MGT_CAT2(a, b)

#define TEST(suite, name)                                                                 \
    static void MGT_CAT(mgt_test_##suite##_, name)();                                     \
    static ::minigtest::Registrar MGT_CAT(mgt_reg_##suite##_, name)(#suite, #name,        \
                                                                    &MGT_CAT(mgt_test_##suite##_, name)); \
    static void MGT_CAT(mgt_test_##suite##_, name)()

#define MGT_EXPECT(cond, text) \
    if (cond)                  \
        ;                      \
    else                       \
        ::minigtest::Reporter(__FILE__, __LINE__, text) = ::minigtest::Msg()
#define MGT_ASSERT(cond, text) \
    if (cond)                  \
        ;                      \
    else                       \
        return ::minigtest::Reporter(__FILE__, __LINE__, text) = ::minigtest::Msg()

#define MGT_BIN(a, op, b) \
    (std::string(#a " " #op " " #b "  [") + ::minigtest::show(a) + " vs " + ::minigtest::show(b) + "]")

#define EXPECT_TRUE(c) MGT_EXPECT((c), "expected true: " #c)
#define EXPECT_FALSE(c) MGT_EXPECT(!(c), "expected false: " #c)
#define ASSERT_TRUE(c) MGT_ASSERT((c), "expected true: " #c)
#define ASSERT_FALSE(c) MGT_ASSERT(!(c), "expected false: " #c)
#define EXPECT_EQ(a, b) MGT_EXPECT((a) == (b), MGT_BIN(a, ==, b))
#define EXPECT_NE(a, b) MGT_EXPECT((a) != (b), MGT_BIN(a, !=, b))
#define EXPECT_LT(a, b) MGT_EXPECT((a) < (b), MGT_BIN(a, <, b))
#define EXPECT_LE(a, b) MGT_EXPECT((a) <= (b), MGT_BIN(a, <=, b))
#define EXPECT_GT(a, b) MGT_EXPECT((a) > (b), MGT_BIN(a, >, b))
#define EXPECT_GE(a, b) MGT_EXPECT((a) >= (b), MGT_BIN(a, >=, b))
#define ASSERT_EQ(a, b) MGT_ASSERT((a) == (b), MGT_BIN(a, ==, b))
#define ASSERT_NE(a, b) MGT_ASSERT((a) != (b), MGT_BIN(a, !=, b))
#define ASSERT_LT(a, b) MGT_ASSERT((a) < (b), MGT_BIN(a, <, b))
#define ASSERT_LE(a, b) MGT_ASSERT((a) <= (b), MGT_BIN(a, <=, b))
#define ASSERT_GT(a, b) MGT_ASSERT((a) > (b), MGT_BIN(a, >, b))
#define ASSERT_GE(a, b) MGT_ASSERT((a) >= (b), MGT_BIN(a, >=, b))
#define EXPECT_NEAR(a, b, tol) MGT_EXPECT(std::abs((a) - (b)) <= (tol), MGT_BIN(a, ~=, b))
#define ASSERT_NEAR(a, b, tol) MGT_ASSERT(std::abs((a) - (b)) <= (tol), MGT_BIN(a, ~=, b))
#define EXPECT_DOUBLE_EQ(a, b) MGT_EXPECT(::minigtest::almost_equal((a), (b)), MGT_BIN(a, ==, b))
#define ASSERT_DOUBLE_EQ(a, b) MGT_ASSERT(::minigtest::almost_equal((a), (b)), MGT_BIN(a, ==, b))
#define FAIL() return ::minigtest::Reporter(__FILE__, __LINE__, "FAIL()") = ::minigtest::Msg()

#define MGT_THROWS(stmt, exc, fatal_ret)                                                 \
    do {                                                                                 \
        bool mgt_ok = false;                                                             \
        try {                                                                            \
            stmt;                                                                        \
        } catch (const exc&) {                                                           \
            mgt_ok = true;                                                               \
        } catch (...) {                                                                  \
        }                                                                                \
        if (!mgt_ok) {                                                                   \
            ::minigtest::Reporter(__FILE__, __LINE__, "expected " #exc " from " #stmt) = \
                ::minigtest::Msg();                                                      \
            fatal_ret;                                                                   \
        }                                                                                \
    } while (0)
#define EXPECT_THROW(stmt, exc) MGT_THROWS(stmt, exc, (void)0)
#define ASSERT_THROW(stmt, exc) MGT_THROWS(stmt, exc, return)
#define EXPECT_NO_THROW(stmt)                                                          \
    do {                                                                               \
        try {                                                                          \
            stmt;                                                                      \
        } catch (...) {                                                                \
            ::minigtest::Reporter(__FILE__, __LINE__, "unexpected exception from " #stmt) = \
                ::minigtest::Msg();                                                    \
        }                                                                              \
    } while (0)
#define ASSERT_NO_THROW(stmt) EXPECT_NO_THROW(stmt)

namespace testing {
class Test {
  public:
    virtual ~Test() = default;
    virtual void SetUp() {}
    virtual void TearDown() {}
};
struct TestInfo {
    const char* name() const { return ::minigtest::current_name(); }
};
class UnitTest {
  public:
    static UnitTest* GetInstance() {
        static UnitTest u;
        return &u;
    }
    const TestInfo* current_test_info() const {
        static TestInfo info;
        return &info;
    }
};
}  // namespace testing

#define TEST_F(fixture, name)                                                                        \
    class MGT_CAT(fixture##_##name, _MgtTest) : public fixture {                                    \
      public:                                                                                        \
        void Body();                                                                                 \
        void Run() {                                                                                 \
            this->SetUp();                                                                           \
            Body();                                                                                  \
            this->TearDown();                                                                        \
        }                                                                                            \
    };                                                                                               \
    static void MGT_CAT(mgt_runf_##fixture##_, name)() {                                             \
        MGT_CAT(fixture##_##name, _MgtTest) t;                                                       \
        t.Run();                                                                                     \
    }                                                                                                \
    static ::minigtest::Registrar MGT_CAT(mgt_regf_##fixture##_, name)(#fixture, #name,             \
                                                                       &MGT_CAT(mgt_runf_##fixture##_, name)); \
    void MGT_CAT(fixture##_##name, _MgtTest)::Body()
