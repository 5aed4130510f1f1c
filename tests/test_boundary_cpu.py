"""The product path never reaches the oracle and has no CPU fallback.

oracle/ is test infrastructure (tests/, smoke(), bench.py's cpu_baseline and
--impl reference legs only). These checks keep it that way: no Python module
of the package imports it, no native build links it, the built libraries do
not depend on it, and a missing CUDA library fails loudly.
"""
import ast
import os
import subprocess

import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2504_00987_b200")
LIB_DIR = os.path.join(PKG, "lib")


def _package_files(exts):
    for d, _, files in os.walk(PKG):
        if "__pycache__" in d:
            continue
        for f in files:
            if f.endswith(exts):
                yield os.path.join(d, f)


def test_package_python_never_imports_oracle():
    for path in _package_files((".py",)):
        with open(path) as f:
            tree = ast.parse(f.read(), path)
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            for name in names:
                assert not name.split(".")[0] == "oracle", f"{path} imports {name}"


def test_native_sources_and_build_do_not_reference_oracle():
    paths = list(_package_files((".cu", ".cuh", ".cpp", ".hpp", ".h")))
    paths.append(os.path.join(PKG, "Makefile"))
    inc = os.path.join(ROOT, "include")
    for d, _, files in os.walk(inc):
        paths += [os.path.join(d, f) for f in files]
    for path in paths:
        with open(path, errors="replace") as f:
            text = f.read()
        for bad in ("oracle/", "labs_oracle", "ref_labsolve", "/root/reference/proj/src"):
            assert bad not in text, f"{path} mentions {bad}"


@pytest.mark.parametrize("lib", ["liblabs_b200.so", "liblabsolve_b200.so"])
def test_built_libraries_do_not_depend_on_oracle(lib):
    path = os.path.join(LIB_DIR, lib)
    if not os.path.exists(path):
        pytest.skip(f"{lib} not built")
    out = subprocess.run(["readelf", "-d", path], capture_output=True, text=True).stdout
    needed = [l for l in out.splitlines() if "(NEEDED)" in l]
    for l in needed:
        assert "oracle" not in l and "ref_labsolve" not in l, l


def test_missing_library_fails_loudly(tmp_path):
    from paper_2504_00987_b200 import capi
    saved = capi._lib
    capi._lib = None
    try:
        with pytest.raises(ImportError, match="no CPU fallback"):
            capi.load_library(str(tmp_path / "liblabs_b200.so"))
    finally:
        capi._lib = saved
