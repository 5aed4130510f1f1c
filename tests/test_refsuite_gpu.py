"""The reference's own doctest suites (proj/tests/test_*.cpp), compiled
unmodified against this repo's labsolve:: drop-in headers and linked to the
B200 library (tests/refsuite/Makefile; doctest shim in tests/refsuite/shim).
Every TEST_CASE of every suite must pass on the device implementation."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BIN = os.path.join(ROOT, "tests", "refsuite", "_bin")
SUITES = ["sequence", "correlation", "tabu", "memetic", "parallel", "skew", "oracle", "fit"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_doctest_suite(suite):
    exe = os.path.join(BIN, f"test_{suite}")
    assert os.path.exists(exe), "built by __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-8000:])
    assert r.returncode == 0, r.stderr[-8000:]
    assert "| 0 failed;" in r.stdout
