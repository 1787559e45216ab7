"""Test-only device helpers (not part of the product): the fp32 SIMT GEMM in
``tests/csrc/simt_gemm.cu``, built into ``tests/libfb_testkit.so`` by
``paper_1909_08723_b200.csrc.build``, used as an independent cross-check of
the tcgen05 GEMM's epilogues."""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libfb_testkit.so")
_h = None


def _lib():
    global _h
    if _h is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run python -m paper_1909_08723_b200.csrc.build")
        from paper_1909_08723_b200 import _lib as L
        _h = C.CDLL(LIB)
        _h.fbt_gemm_simt.restype = C.c_int
        _h.fbt_gemm_simt.argtypes = [C.POINTER(L.FbGemm), C.c_void_p]
        _h.fbt_last_error.restype = C.c_char_p
    return _h


def _ld(t) -> int:
    return 0 if t is None else t.stride(0)


def gemm(a, w, *, m: Optional[int] = None, m_dev=None, k: Optional[int] = None, bias=None,
         out=None, rows=None, mode: int = 0, hidden: int = 0, parent=None, c_in=None,
         c_out=None, h_out=None, h_res=None, addend=None, lda: Optional[int] = None) -> None:
    """C = A . W^T (fp32 A and W) with the fb_gemm_t epilogues, SIMT fp32."""
    from paper_1909_08723_b200 import _lib as L
    P = L.ptr
    g = L.FbGemm()
    g.m_max = a.shape[0] if m is None else m
    g.m_dev = P(m_dev)
    g.n = w.shape[0]
    g.k = w.shape[1] if k is None else k
    g.a, g.lda = P(a), (a.stride(0) if lda is None else lda)
    g.w, g.ldw = P(w), w.stride(0)
    g.bias = P(bias)
    g.c, g.ldc = P(out), _ld(out)
    g.mode, g.hidden = mode, hidden
    g.rows, g.parent = P(rows), P(parent)
    g.c_in, g.ld_cin = P(c_in), _ld(c_in)
    g.c_out, g.ld_cout = P(c_out), _ld(c_out)
    g.h_out, g.ld_h = P(h_out), _ld(h_out)
    g.h_res, g.ld_res = P(h_res), _ld(h_res)
    g.addend, g.ld_add = P(addend), _ld(addend)
    h = _lib()
    rc = h.fbt_gemm_simt(C.byref(g), L.stream_ptr())
    if rc != 0:
        msg = h.fbt_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)
