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


def test_python_fit_matches_reference_semantics():
    """paper_2504_00987_b200.tts mirrors fit.cpp: quantiles, censoring, fit."""
    import math
    import scipy.stats as st
    from paper_2504_00987_b200 import tts
    assert tts.quantile([1.0, 2.0, 3.0, 4.0], 0.25) == 1.75
    s = [{"n": 10, "runtime": 1.0, "reachedTarget": True},
         {"n": 10, "runtime": 3.0, "reachedTarget": True},
         {"n": 10, "runtime": 99.0, "reachedTarget": False},
         {"n": 12, "runtime": 50.0, "reachedTarget": False}]
    assert tts.median_runtime_by_n(s) == {10: 2.0}
    ex = [{"n": n, "runtime": 2e-7 * 1.3 ** n, "reachedTarget": True} for n in range(20, 41)]
    f = tts.fit_exponential(ex, 20, 40)
    assert abs(f["b"] - 1.3) < 1e-12 and abs(f["a"] / 2e-7 - 1) < 1e-9
    for dof in (1, 3, 7, 19, 50):
        assert abs(tts.student_t_quantile(dof, 0.975) - st.t.ppf(0.975, dof)) < 1e-8
    noisy = [{"n": n, "runtime": 1e-6 * 1.25 ** n * math.exp(0.3 * math.sin(n)),
              "reachedTarget": True} for n in range(10, 31)]
    f = tts.fit_exponential(noisy, 10, 30)
    assert f["b_ci"][0] < 1.25 < f["b_ci"][1]


def test_read_targets_columns():
    """targets_long.txt: column 1 = the paper's records (= the reference's
    proj/data/targets_published.txt), column 2 = the previous best-known."""
    import os
    from paper_2504_00987_b200 import tts
    path = os.path.join(os.path.dirname(tts.__file__), "data", "targets_long.txt")
    new, old = tts.read_targets(path), tts.read_targets(path, 2)
    assert new[92] == 490 and old[92] == 498
    assert new[119] == 787 and old[119] == 835
    assert set(new) == set(old) and len(new) == 16
    assert all(new[n] <= old[n] for n in new)
