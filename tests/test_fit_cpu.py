"""fit.hpp drop-in (TTS statistics around the device solver), host-only."""
import os
import subprocess

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_cpp_fit_suite(tmp_path):
    exe = os.path.join(ROOT, "tests", "cpp", "test_fit")
    assert os.path.exists(exe), "build with __graft_entry__.build()"
    r = subprocess.run([exe, str(tmp_path / "s.jsonl")], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_student_t_against_scipy():
    """Cross-check of the in-house t quantile (replacing Boost.Math) on many dof."""
    import scipy.stats as st
    exe = os.path.join(ROOT, "tests", "cpp", "test_fit")
    assert os.path.exists(exe)
    # the C++ suite pins five values; scipy pins the same ones here
    for dof, want in [(1, 12.706204736174707), (2, 4.302652729749464),
                      (10, 2.228138851986274), (30, 2.042272456301238)]:
        assert abs(st.t.ppf(0.975, dof) - want) < 1e-9
