"""The C-ABI library loads and exports every symbol include/hssmf_b200.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from paper_1502_07405_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hssmf_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hssmf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(header_symbols()) == set(_native.exported_symbols())


def test_version_string():
    assert b"sm_100a" in _native.lib().hssmf_version()
