"""The C-ABI library builds, loads and exports every entry point declared in
include/hapod_b200.h (no GPU needed; no compute calls are made)."""

import ctypes
import os
import re

import pytest

from paper_1607_05210_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "hapod_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    decl = declared_functions()
    assert len(decl) >= 20
    assert sorted(N.EXPORTED) == decl


def test_library_exports_every_symbol():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libhapod_b200.so not built (run ./build_native.sh)")
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    loaded = N.load()
    assert loaded.hp_abi_version() == N.ABI_VERSION
    assert loaded.hp_launch_count() >= 0
    # workspace queries are pure host arithmetic
    assert loaded.hp_gemm_workspace_bytes(512, 512, 200000, 1, 0) > 0
    assert loaded.hp_syev_workspace_bytes(1000) >= 2 * 1024 * 1024 * 8


def test_sm100a_cubin_inside():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libhapod_b200.so not built")
    data = open(N.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
