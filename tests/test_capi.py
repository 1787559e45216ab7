"""The C-ABI library loads without a GPU and exports every symbol the header
declares; the Python binding declares the same set (CPU only)."""

import ctypes
import os
import re

from paper_1909_08723_b200 import _lib
from paper_1909_08723_b200.csrc.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            text = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"\b(fb_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_header_symbols():
    path = build()
    lib = ctypes.CDLL(path)
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.fb_abi_version() == 1


def test_binding_covers_header():
    try:
        import paper_1909_08723_b200.models  # noqa: F401  (registers model entry points)
    except ImportError:
        pass
    assert _declared() <= set(_lib._SIGS)


def test_error_text_round_trip():
    lib = ctypes.CDLL(build())
    lib.fb_gather_rows.restype = ctypes.c_int
    rc = lib.fb_gather_rows(ctypes.c_int32(1), None, None, None, ctypes.c_int64(0), None)
    assert rc == 1
    lib.fb_last_error.restype = ctypes.c_char_p
    assert b"row size" in lib.fb_last_error()


def test_attention_tiling_setter_validates():
    lib = ctypes.CDLL(build())
    f = lib.fb_set_attention_tiling
    f.restype = ctypes.c_int
    i = ctypes.c_int32
    assert f(i(3), i(0), i(0)) == 1           # frame warps must be 2/4/8
    assert f(i(0), i(5), i(0)) == 1           # rows must be even
    assert f(i(0), i(0), i(-1)) == 1
    assert f(i(4), i(4), i(160)) == 0
    assert f(i(0), i(0), i(0)) == 0           # back to the defaults
