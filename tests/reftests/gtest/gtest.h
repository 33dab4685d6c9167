// A minimal GoogleTest-compatible shim (test infrastructure): enough of the API for the
// reference's own test suites (proj/tests/*.cpp) to compile against the drop-in headers in
// include/reattn and run on the GPU -- TEST, the EXPECT_* / ASSERT_* comparisons with
// streamed messages, EXPECT_THROW / EXPECT_NO_THROW, ::testing::Test::HasFailure /
// HasFatalFailure, ::testing::TempDir and a main() that runs every registered test (an
// optional filter of substrings).  GoogleTest itself is not installed in this image.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace testing {

namespace internal {

struct TestCase {
    const char* suite;
    const char* name;
    std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    bool failure = false;
    bool fatal = false;
    int checks = 0;
};

inline State& state() {
    static State s;
    return s;
}

struct Registrar {
    Registrar(const char* suite, const char* name, std::function<void()> fn) {
        registry().push_back({suite, name, std::move(fn)});
    }
};

// gtest's own pattern: `AssertHelper(...) = Message() << "streamed"` (the assignment runs last)
struct Message {
    std::ostringstream o;
    template <typename T>
    Message& operator<<(const T& v) {
        o << v;
        return *this;
    }
};

class AssertHelper {
public:
    AssertHelper(const char* file, int line, std::string what, bool fatal)
        : file_(file), line_(line), what_(std::move(what)) {
        state().failure = true;
        if (fatal) state().fatal = true;
    }
    void operator=(const Message& m) const {
        const std::string msg = m.o.str();
        std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file_, line_, what_.c_str(), msg.empty() ? "" : "\n  ",
                     msg.c_str());
    }

private:
    const char* file_;
    int line_;
    std::string what_;
};

// swallows streamed messages of a passing check
struct Pass {
    template <typename T>
    Pass& operator<<(const T&) {
        return *this;
    }
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
std::string cmp_text(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
    return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

inline bool float_eq(float a, float b) {
    if (std::isnan(a) || std::isnan(b)) return false;
    if (a == b) return true;
    int32_t ia, ib;
    std::memcpy(&ia, &a, 4);
    std::memcpy(&ib, &b, 4);
    if ((ia < 0) != (ib < 0)) return false;
    return std::abs((long long)ia - (long long)ib) <= 4;  // 4 ULPs, as GoogleTest
}
inline bool double_eq(double a, double b) {
    if (std::isnan(a) || std::isnan(b)) return false;
    if (a == b) return true;
    int64_t ia, ib;
    std::memcpy(&ia, &a, 8);
    std::memcpy(&ib, &b, 8);
    if ((ia < 0) != (ib < 0)) return false;
    const int64_t d = ia > ib ? ia - ib : ib - ia;
    return d <= 4;
}

}  // namespace internal

class Test {
public:
    virtual ~Test() = default;
    static bool HasFailure() { return internal::state().failure; }
    static bool HasFatalFailure() { return internal::state().fatal; }
};

inline std::string TempDir() {
    const char* t = std::getenv("TEST_TMPDIR");
    std::string d = t ? t : "/tmp";
    if (d.empty() || d.back() != '/') d += '/';
    return d;
}

inline int RunAllTests(int argc, char** argv) {
    int failed = 0, run = 0;
    for (auto& t : internal::registry()) {
        const std::string full = std::string(t.suite) + "." + t.name;
        bool selected = argc <= 1;
        for (int i = 1; i < argc; ++i)
            if (full.find(argv[i]) != std::string::npos) selected = true;
        if (!selected) continue;
        internal::state() = internal::State{};
        std::fprintf(stderr, "[ RUN      ] %s\n", full.c_str());
        try {
            t.fn();
        } catch (const std::exception& e) {
            internal::state().failure = true;
            std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        } catch (...) {
            internal::state().failure = true;
            std::fprintf(stderr, "unexpected non-std exception\n");
        }
        ++run;
        if (internal::state().failure) {
            ++failed;
            std::fprintf(stderr, "[  FAILED  ] %s\n", full.c_str());
        } else {
            std::fprintf(stderr, "[       OK ] %s\n", full.c_str());
        }
    }
    std::fprintf(stderr, "[==========] %d tests ran, %d passed, %d failed\n", run, run - failed, failed);
    return failed ? 1 : 0;
}

}  // namespace testing

#define GTS_CAT2(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT2(a, b)

// a TEST body is a member of a ::testing::Test subclass (HasFailure() etc. resolve unqualified)
#define GTS_CLASS(suite, name) GTS_CAT(gts_, GTS_CAT(suite, GTS_CAT(_, name)))
#define TEST(suite, name)                                                                   \
    class GTS_CLASS(suite, name) : public ::testing::Test {                                  \
    public:                                                                                  \
        void TestBody();                                                                     \
    };                                                                                       \
    static ::testing::internal::Registrar GTS_CAT(gts_reg_, GTS_CLASS(suite, name))(         \
        #suite, #name, [] { GTS_CLASS(suite, name) t; t.TestBody(); });                      \
    void GTS_CLASS(suite, name)::TestBody()

#define GTS_NONFATAL(cond, text)                         \
    if (++::testing::internal::state().checks, (cond))     \
        ;                                                  \
    else                                                   \
        ::testing::internal::AssertHelper(__FILE__, __LINE__, text, false) = ::testing::internal::Message()
#define GTS_FATAL(cond, text)                                  \
    if (++::testing::internal::state().checks, (cond))         \
        ;                                                      \
    else                                                       \
        return ::testing::internal::AssertHelper(__FILE__, __LINE__, text, true) = ::testing::internal::Message()

#define GTS_BIN(a, b, op, opname, fatal_or_not)                                                        \
    GTS_##fatal_or_not(([&] { return (a)op(b); })(),                                                  \
                       ::testing::internal::cmp_text(opname, #a, #b, (a), (b)))


#define EXPECT_EQ(a, b) GTS_BIN(a, b, ==, "==", NONFATAL)
#define EXPECT_NE(a, b) GTS_BIN(a, b, !=, "!=", NONFATAL)
#define EXPECT_LT(a, b) GTS_BIN(a, b, <, "<", NONFATAL)
#define EXPECT_LE(a, b) GTS_BIN(a, b, <=, "<=", NONFATAL)
#define EXPECT_GT(a, b) GTS_BIN(a, b, >, ">", NONFATAL)
#define EXPECT_GE(a, b) GTS_BIN(a, b, >=, ">=", NONFATAL)
#define ASSERT_EQ(a, b) GTS_BIN(a, b, ==, "==", FATAL)
#define ASSERT_NE(a, b) GTS_BIN(a, b, !=, "!=", FATAL)
#define ASSERT_LT(a, b) GTS_BIN(a, b, <, "<", FATAL)
#define ASSERT_LE(a, b) GTS_BIN(a, b, <=, "<=", FATAL)
#define ASSERT_GT(a, b) GTS_BIN(a, b, >, ">", FATAL)
#define ASSERT_GE(a, b) GTS_BIN(a, b, >=, ">=", FATAL)
#define EXPECT_TRUE(c) GTS_NONFATAL(static_cast<bool>(c), std::string("Expected true: ") + #c)
#define EXPECT_FALSE(c) GTS_NONFATAL(!static_cast<bool>(c), std::string("Expected false: ") + #c)
#define ASSERT_TRUE(c) GTS_FATAL(static_cast<bool>(c), std::string("Expected true: ") + #c)
#define ASSERT_FALSE(c) GTS_FATAL(!static_cast<bool>(c), std::string("Expected false: ") + #c)
#define EXPECT_NEAR(a, b, tol)                                                                   \
    GTS_NONFATAL(std::fabs((double)(a) - (double)(b)) <= (double)(tol),                          \
                 ::testing::internal::cmp_text("near", #a, #b, (a), (b)) + " tol " + #tol)
#define ASSERT_NEAR(a, b, tol)                                                                   \
    GTS_FATAL(std::fabs((double)(a) - (double)(b)) <= (double)(tol),                             \
              ::testing::internal::cmp_text("near", #a, #b, (a), (b)) + " tol " + #tol)
#define EXPECT_FLOAT_EQ(a, b) \
    GTS_NONFATAL(::testing::internal::float_eq((a), (b)), ::testing::internal::cmp_text("float==", #a, #b, (a), (b)))
#define EXPECT_DOUBLE_EQ(a, b) \
    GTS_NONFATAL(::testing::internal::double_eq((a), (b)), ::testing::internal::cmp_text("double==", #a, #b, (a), (b)))
#define EXPECT_STREQ(a, b) \
    GTS_NONFATAL(std::string(a) == std::string(b), ::testing::internal::cmp_text("streq", #a, #b, std::string(a), std::string(b)))

#define GTS_THROWS(stmt, ex, fatal_or_not)                                                   \
    GTS_##fatal_or_not(([&] {                                                                \
        try {                                                                                \
            stmt;                                                                            \
        } catch (const ex&) {                                                                \
            return true;                                                                     \
        } catch (...) {                                                                      \
            return false;                                                                    \
        }                                                                                    \
        return false;                                                                        \
    })(),                                                                                    \
                       std::string("Expected: ") + #stmt + " throws " + #ex)
#define EXPECT_THROW(stmt, ex) GTS_THROWS(stmt, ex, NONFATAL)
#define ASSERT_THROW(stmt, ex) GTS_THROWS(stmt, ex, FATAL)
#define EXPECT_NO_THROW(stmt)                                                                \
    GTS_NONFATAL(([&] {                                                                      \
        try {                                                                                \
            stmt;                                                                            \
        } catch (...) {                                                                      \
            return false;                                                                    \
        }                                                                                    \
        return true;                                                                         \
    })(),                                                                                    \
                 std::string("Expected no throw: ") + #stmt)

#define SUCCEED() ::testing::internal::Pass()
#define FAIL() GTS_FATAL(false, "Failed")
#define ADD_FAILURE() GTS_NONFATAL(false, "Failed")

#ifndef GTS_NO_MAIN
int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
#endif
