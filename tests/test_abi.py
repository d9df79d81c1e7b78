"""C-ABI checks that run without a GPU: the in-tree sm_100a library builds,
loads, exports every symbol ``include/blreg_b200.h`` declares, and the ctypes
binding covers the whole header."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blreg_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(blr_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1807_05117_b200 import build

    return build.build(verbose=False)


def test_header_declares_entry_points():
    syms = header_symbols()
    assert len(syms) >= 30
    for s in ("blr_ctx_create", "blr_include", "blr_project", "blr_forward_map",
              "blr_state_tangents", "blr_momentum_tangent", "blr_contract", "blr_warp"):
        assert s in syms


def test_library_exports_every_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for s in header_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (blr_\w+)", out))
    assert set(header_symbols()) <= exported


def test_ctypes_binding_covers_header(libpath):
    from paper_1807_05117_b200 import _lib

    assert set(header_symbols()) == set(_lib.SIGNATURES)
    lib = _lib.load(libpath)
    assert lib.blr_version() == 1
    assert _lib.launch_count() >= 0


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_are_reported_without_gpu(libpath):
    from paper_1807_05117_b200 import _lib

    lib = _lib.load(libpath)
    rc = lib.blr_include(None, 0, None, 1, None, None)
    assert rc == 1
    assert "bad arguments" in _lib.last_error()
