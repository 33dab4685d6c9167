"""The GoogleTest shim (tests/reftests/gtest/gtest.h) that runs the reference's own suites on
the drop-in: a failing check must count as a failure (and a fatal one must stop its test),
passing checks must not, exceptions are caught and messages stream.  CPU only."""
import os
import re
import subprocess
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "reftests")

PROGRAM = textwrap.dedent(r'''
    #include <stdexcept>
    #include <vector>
    #include <gtest/gtest.h>
    static int after_fatal = 0;
    TEST(Shim, Passes) {
        EXPECT_EQ(2 + 2, 4);
        EXPECT_NEAR(1.0, 1.0 + 1e-9, 1e-6);
        EXPECT_FLOAT_EQ(0.1f + 0.2f, 0.3f);
        EXPECT_THROW(throw std::invalid_argument("x"), std::invalid_argument);
        EXPECT_NO_THROW((void)0);
        ASSERT_TRUE(true) << "never printed";
        EXPECT_LE((std::vector<int>{1, 2}.size()), 2u);
    }
    TEST(Shim, NonFatalFailureContinues) {
        EXPECT_EQ(1, 2) << "streamed " << 42;
        EXPECT_TRUE(HasFailure());
        EXPECT_FALSE(HasFatalFailure());
    }
    TEST(Shim, FatalFailureStops) {
        ASSERT_EQ(1, 2);
        ++after_fatal;
    }
    TEST(Shim, WrongExceptionFails) { EXPECT_THROW(throw std::runtime_error("y"), std::invalid_argument); }
    TEST(Shim, UncaughtExceptionFails) { throw std::logic_error("boom"); }
    TEST(Shim, AfterFatalNotReached) { EXPECT_EQ(after_fatal, 0); }
''')


def test_shim_counts_failures(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I", SHIM, str(src), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    out = r.stdout + r.stderr
    assert r.returncode == 1
    m = re.search(r"(\d+) tests ran, (\d+) passed, (\d+) failed", out)
    assert m and m.groups() == ("6", "2", "4"), out
    assert "streamed 42" in out
    for name in ("NonFatalFailureContinues", "FatalFailureStops", "WrongExceptionFails",
                 "UncaughtExceptionFails"):
        assert f"[  FAILED  ] Shim.{name}" in out
    assert "[       OK ] Shim.AfterFatalNotReached" in out
    r2 = subprocess.run([str(exe), "Passes"], capture_output=True, text=True, timeout=60)
    assert r2.returncode == 0 and "1 tests ran, 1 passed, 0 failed" in r2.stderr
