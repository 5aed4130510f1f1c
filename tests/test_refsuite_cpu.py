"""The doctest shim (tests/refsuite/shim/doctest.h) behaves like doctest for
the subset the reference's suites use: every SUBCASE gets its own run of the
test case with the code outside subcases re-executed, REQUIRE aborts the
test case, CHECK_THROWS_AS / CHECK_NOTHROW / Approx, and the exit status and
summary line reflect failures. (The suites themselves run on a GPU:
tests/test_refsuite_gpu.py.)"""
import os
import subprocess
import textwrap

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
SHIM = os.path.join(ROOT, "tests", "refsuite", "shim")

SRC = textwrap.dedent(r"""
    #define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
    #include <doctest.h>
    #include <stdexcept>
    static int outside = 0, a = 0, b = 0;
    TEST_CASE("subcases") {
      ++outside;
      SUBCASE("a") { ++a; CHECK(outside == a + b); }
      SUBCASE("b") { ++b; CHECK(outside == a + b); }
    }
    TEST_CASE("counts") { CHECK(outside == 2); CHECK(a == 1); CHECK(b == 1); }
    TEST_CASE("throws") {
      CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
      CHECK_NOTHROW((void)0);
      CHECK(0.1 + 0.2 == doctest::Approx(0.3));
      CHECK(1.0 == doctest::Approx(1.1).epsilon(0.2));
    }
    TEST_CASE("failing") {
      REQUIRE(1 == 2);
      CHECK(false);  // not reached: REQUIRE aborted the case
    }
""")


def test_doctest_shim(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I", SHIM, "-o", str(exe), str(src)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1  # the "failing" case
    assert "test cases: 4 | 3 passed | 1 failed; assertions: 10 | 9 passed | 1 failed" \
        in r.stdout, r.stdout + r.stderr
    assert "REQUIRE(1 == 2)" in r.stderr
    r = subprocess.run([str(exe), "subcases"], capture_output=True, text=True)
    assert r.returncode == 0 and "test cases: 1 | 1 passed | 0 failed" in r.stdout
