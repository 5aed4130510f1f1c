"""CPU tests of the boundary: the CUDA library and the C++ drop-in load and
export every symbol their headers declare; host-side validation paths that
need no device."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2504_00987_b200 import capi

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "labs_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(labs_[a-z_0-9]+)\(",
                                 text, re.M)))


def test_header_and_mirror_agree():
    assert declared_symbols() == sorted(capi.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = capi.load_library()
    for sym in declared_symbols():
        assert hasattr(L, sym), sym
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for sym in declared_symbols():
        assert re.search(rf"\bT {sym}$", out, re.M), sym


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_rng_seed_matches_reference_engine(oracle):
    """labs_rng_seed is Rng(seed)'s engine state (rng.hpp:13)."""
    for seed in (0, 1, 42, 2**64 - 1):
        st = capi.rng_state(seed)
        r = oracle.rng(seed)
        assert list(st.mt) == list(r.mt) and st.idx == r.idx == 312


def test_no_device_means_loud_failure():
    """Without a GPU, creating a context raises — there is no CPU fallback."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises((capi.LabsCudaError, ValueError)):
        capi.Context(0)


def test_struct_layouts_match_header():
    assert C.sizeof(capi.RngState) == 312 * 8 + 8
    assert C.sizeof(capi.TabuStep) == 24
    assert C.sizeof(capi.TabuParams) == 24
    assert C.sizeof(capi.MemeticParams) == 4 + 4 + 8 * 5 + 24 + 8
    assert C.sizeof(capi.RunResult) == 8 * 4 + 8 * 5 + 8 + 8
    assert C.sizeof(capi.MemeticRecord) == 24
