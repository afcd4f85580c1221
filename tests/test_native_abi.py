"""The C-ABI library exists, loads without a GPU and exports every symbol
that include/mbgpu.h declares (no compute calls here)."""

import ctypes
import re

from conftest import ROOT

from paper_2005_05412_b200 import native


def declared_functions():
    text = (ROOT / "include" / "mbgpu.h").read_text()
    return sorted(set(re.findall(r"\b(mbg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_surface():
    names = declared_functions()
    assert set(names) == set(native.SIGNATURES), set(names) ^ set(native.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    lib = native.load(require_device=False)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.mbg_version().startswith(b"mbgpu")


def test_library_is_built_for_sm100a():
    data = native.LIB_PATH.read_bytes()
    assert b"sm_100a" in data


def test_create_rejects_bad_grid_without_touching_the_device():
    lib = native.load(require_device=False)
    g = native.MbgGrid()
    g.num_x, g.num_t, g.dt = 0, 10, 1e-18  # invalid: no cells
    h = ctypes.c_void_p()
    assert lib.mbg_create(ctypes.byref(g), ctypes.byref(h)) != 0
    assert not h.value
