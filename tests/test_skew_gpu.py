"""K6 (labs_skew_deviation, csrc/labs_skew.cu) against the reference's own
deviation / deviation_with_edits (proj/src/skew.cpp:110-187) on the 113
golden cases — Table II rows, random short sequences, plain and with edits,
with and without budgets — through the C++ drop-in (skew_probe) and the
ctypes mirror: value, budget_exceeded and evaluation count all equal."""
import os
import subprocess

import pytest

from paper_2504_00987_b200 import capi

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
pytestmark = pytest.mark.gpu


def test_deviation_matches_reference_dropin(golden):
    exe = os.path.join(ROOT, "tests", "cpp", "skew_probe")
    assert os.path.exists(exe), "build with __graft_entry__.build()"
    cases = golden["skew"]
    stdin = "\n".join(f'{c["n"]} {c["budget"]} {int(c["edits"])} ' +
                      " ".join(str(w) for w in c["words"]) for c in cases) + "\n"
    r = subprocess.run([exe], input=stdin, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = [tuple(int(x) for x in line.split()) for line in r.stdout.splitlines()]
    want = [(c["value"], int(c["budget_exceeded"]), c["evaluations"]) for c in cases]
    assert got == want


def test_deviation_matches_reference_capi(ctx, golden):
    for c in golden["skew"]:
        got = ctx.skew_deviation(c["n"], c["words"], c["edits"], c["budget"])
        assert got == (c["value"], c["budget_exceeded"], c["evaluations"]), c
    with pytest.raises(ValueError):
        ctx.skew_deviation(2, [0])
