"""The C++ labsolve:: drop-in (include/labsolve/*.hpp over the B200 library),
exercised by tests/cpp/test_labsolve.cpp the way the reference's own doctest
suites exercise the reference headers."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BIN = os.path.join(ROOT, "tests", "cpp", "test_labsolve")


@pytest.mark.gpu
def test_cpp_dropin_suite():
    assert os.path.exists(BIN), "build with __graft_entry__.build() (make -C tests/cpp)"
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "table2.txt")],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_suite_two_islands():
    """The same suite with run_replicas spread over two contexts of device 0
    (LABS_DEVICES=0,0 -> labs_run_replicas_multi), plus the multi-GPU
    parity/stop checks that only run when LABS_DEVICES is set."""
    env = dict(os.environ, LABS_DEVICES="0,0")
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "table2.txt")],
                       capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "multi-GPU run_replicas over LABS_DEVICES: ok" in r.stdout
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_plain_c_client():
    exe = os.path.join(ROOT, "tests", "cpp", "test_capi")
    assert os.path.exists(exe), "build with __graft_entry__.build()"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
