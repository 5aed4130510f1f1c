"""skew.hpp drop-in: the Table II d(S) column of the golden vectors and the
host Rng. The deviation search itself runs on the device (K6) and is checked
against the reference's deviation / deviation_with_edits — values, budgets
and evaluation counts — in tests/test_skew_gpu.py."""
import os
import subprocess

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_table_deviation_column(golden):
    by = {(c["n"], tuple(c["words"])): c["value"] for c in golden["skew"] if not c["edits"]
          and c["budget"] == 0}
    from paper_2504_00987_b200.sequence import decode_hex
    for row in golden["table"]:
        key = (row["n"], tuple(int(x) for x in decode_hex(row["hex"], row["n"])))
        assert by[key] == row["d"]


def test_host_rng_matches_reference(golden):
    """labsolve::Rng (host side of the drop-in) against the reference's draws."""
    exe = os.path.join(ROOT, "tests", "cpp", "rng_probe")
    assert os.path.exists(exe), "build with __graft_entry__.build()"
    lines = []
    for c in golden["rng"]:
        parts = [str(c["seed"]), str(len(c["kinds"]))]
        for k, lo, hi in zip(c["kinds"], c["lo"], c["hi"]):
            parts += [str(k), str(lo), str(hi)]
        lines.append(" ".join(parts))
    r = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True,
                       timeout=60)
    assert r.returncode == 0, r.stderr
    got = [[int(x) for x in line.split()] for line in r.stdout.splitlines()]
    assert got == [c["out"] for c in golden["rng"]]
