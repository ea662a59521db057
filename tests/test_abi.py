"""The C-ABI library loads and exports every symbol include/qpalette.h declares; host-side
validation paths that need no GPU return the documented status codes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2509_20214_b200 import _lib as L

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "qpalette.h")


def _lib_or_skip():
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("libqpalette.so not built (run __graft_entry__.build())")
    return L.lib()


def test_header_declarations_match_binding():
    decl = set(re.findall(r"\b(qp_[a-z0-9_]+)\s*\(", open(HEADER).read()))
    assert decl == set(L.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib_or_skip()
    for name in L.EXPORTS:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.qp_version()


def test_validation_without_gpu():
    lib = _lib_or_skip()
    h = C.c_void_p()
    t = np.zeros(100, dtype=np.float16)
    # wrong tlut length -> QP_ERR_LENGTH, checked before any device work
    assert lib.qp_codebook_load(3, 8, 16, t.ctypes.data, t.nbytes, C.byref(h)) == 6
    # TCQ 2.25 bits is not in Table 1 (only half-TCQ) -> QP_ERR_UNSUPPORTED_WIDTH
    assert lib.qp_codebook_load(3, 9, 16, t.ctypes.data, t.nbytes, C.byref(h)) == 2
    # bad window length
    assert lib.qp_codebook_load(3, 8, 10, t.ctypes.data, 2048, C.byref(h)) == 5
    # rotation width not a multiple of 256 -> QP_ERR_DIM
    assert lib.qp_rht_create(7, 100, 0, C.byref(h)) == 4
    assert b"256" in lib.qp_last_error()


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(L, "_lib", None)
    monkeypatch.setattr(L, "LIB_PATH", "/nonexistent/libqpalette.so")
    with pytest.raises(ImportError):
        L.lib()
