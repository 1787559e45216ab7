"""Thin typed wrappers over the C-ABI launchers (device tensors in, no sync).

Every function here launches exactly one library entry point on the current
torch stream; shapes are validated by the C side (ValueError/ConfigError).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib

P = _lib.ptr


# ---- tensor-core operand format of the loaded library (fb_operand_format) ----
_FMT = None


def operand_format():
    """(planes, torch dtype, activation scale): default build = two fp16 planes
    of x * 2^8; FB_OPERAND_FP16X2=0 build = three bf16 planes."""
    global _FMT
    if _FMT is None:
        p, f, s = C.c_int32(), C.c_int32(), C.c_float()
        _lib.call("fb_operand_format", C.byref(p), C.byref(f), C.byref(s))
        _FMT = (p.value, torch.float16 if f.value else torch.bfloat16, float(s.value))
    return _FMT


def operand_planes(rows: int, k: int, device) -> torch.Tensor:
    """A-operand buffer [planes, rows, k] in the library's operand format."""
    planes, dt, _ = operand_format()
    return torch.empty((planes, rows, k), dtype=dt, device=device)


def operand_weight(w: torch.Tensor) -> torch.Tensor:
    """A weight matrix (bf16-exact values) in the operand format.  fp16 builds
    scale it by a power of two that puts its largest entry near the top of the
    fp16 range (exact for bf16 values); the GEMM epilogue divides it out again
    (``fb_acc_scale`` on the returned tensor)."""
    _, dt, act = operand_format()
    w = w.to(torch.float32)
    if dt == torch.bfloat16:
        out = w.to(torch.bfloat16)
        out.fb_acc_scale = 1.0 / act
        return out
    mx = float(w.abs().max().item()) if w.numel() else 0.0
    e = 0 if mx == 0.0 else int(np.floor(np.log2(32768.0 / mx)))
    out = (w * (2.0 ** e)).to(torch.float16)
    out.fb_acc_scale = 1.0 / (act * 2.0 ** e)
    return out


def _ld(t: Optional[torch.Tensor]) -> int:
    return 0 if t is None else t.stride(0)


def pack(out: torch.Tensor, segs: Sequence[Tuple], *, m: int, m_dev=None, rows=None,
         parent=None, tokens=None, ranks=None, tok_default: int = 0,
         k_pad: Optional[int] = None, split: bool = False) -> None:
    """out[i] = concat(segments) zero-padded; segs = (src|None, width, mode, ld?);
    mode 5 leaves the segment's columns untouched (written by another kernel).
    split=True: out is bf16 [3, plane_rows, k_pad] (hi/mid/lo planes)."""
    p = _lib.FbPack()
    for j, s in enumerate(segs):
        src, width, mode = s[0], s[1], s[2]
        ld = s[3] if len(s) > 3 else (src.stride(0) if src is not None else 0)
        p.seg[j] = _lib.FbSeg(P(src), ld, width, mode)
    p.nseg = len(segs)
    p.k_pad = out.shape[-1] if k_pad is None else k_pad
    p.tok_default = tok_default
    p.out_mode = 1 if split else 0
    p.plane_rows = out.shape[1] if split else 0
    ld = out.stride(1) if split else out.stride(0)
    _lib.call("fb_pack_rows", C.byref(p), m, P(m_dev), P(rows), P(parent), P(tokens), P(ranks),
              P(out), ld, _lib.stream_ptr())


# Instrumentation (bench.py): when set to a list, every tensor-core GEMM launch
# appends (start_event, end_event, rows (int or device tensor), n, k_alg).
GEMM_LOG = None


def log_gemm_begin():
    if GEMM_LOG is None:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def log_gemm_end(e0, m, m_dev, n: int, k_alg: int) -> None:
    if e0 is None:
        return
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    GEMM_LOG.append((e0, e1, m_dev.clone() if m_dev is not None else m, n, k_alg))


class SplitK:
    """Stream-K workspace of fb_gemm_tc (fp32 partial tiles + zeroed arrival
    counters).  One per stream: GEMMs that may run concurrently need their own."""

    SMS = 148

    def __init__(self, device, bn: int = 128):
        self.ws = torch.empty(2 * self.SMS * 128 * bn, dtype=torch.float32, device=device)
        self.cnt = torch.zeros(self.SMS, dtype=torch.int32, device=device)


def gemm_tc(ap: torch.Tensor, w: torch.Tensor, *, m: Optional[int] = None, m_dev=None,
            k: Optional[int] = None, bias=None, out=None, rows=None, mode: int = 0,
            hidden: int = 0, parent=None, c_in=None, c_out=None, h_out=None, h_res=None,
            addend=None, h_split=None, row_stats=None, stats_vw: int = 0,
            k_alg: Optional[int] = None, kcb: int = 0, splitk=None,
            hs_by_row: bool = False, out_exp2: bool = False,
            out_logsoftmax: bool = False) -> None:
    """Tensor-core GEMM: ap = operand planes [P, rows, k_pad] (operand_planes),
    w = operand_weight(...) [n, k_pad].  h_split: optional operand planes
    receiving h (next A operand).  kcb: K blocks per TMEM accumulation chunk
    (0 default; 1 for score logits)."""
    _, dt, act = operand_format()
    if ap.dtype != dt or w.dtype != dt:
        raise ValueError(f"GEMM operands must be {dt} (operand_planes / operand_weight)")
    g = _lib.FbGemm()
    g.acc_scale = getattr(w, "fb_acc_scale", 1.0 / act)
    g.m_max = ap.shape[1] if m is None else m
    g.m_dev = P(m_dev)
    g.n = w.shape[0]
    g.k = w.shape[1] if k is None else k
    g.a, g.lda = P(ap), ap.stride(1)
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
    if h_split is not None:
        g.h_split, g.hs_plane_rows, g.ld_hs = P(h_split), h_split.shape[1], h_split.stride(1)
        g.hs_row_mode = 1 if hs_by_row else 0
    if row_stats is not None:
        g.row_stats, g.stats_vw = P(row_stats), stats_vw
    g.kcb = kcb
    g.out_exp2 = 1 if out_exp2 else 0
    g.out_logsoftmax = 1 if out_logsoftmax else 0
    if splitk is not None:
        g.splitk_ws, g.splitk_cnt = P(splitk.ws), P(splitk.cnt)
    e0 = log_gemm_begin()
    _lib.call("fb_gemm_tc", C.byref(g), ap.shape[0], ap.shape[1], _lib.stream_ptr())
    log_gemm_end(e0, g.m_max, m_dev, g.n, k_alg if k_alg is not None else g.k)


def log_softmax_rows(x: torch.Tensor, out: torch.Tensor, n: int, *, m: int, m_dev=None,
                     rows=None) -> None:
    _lib.call("fb_log_softmax_rows", m, P(m_dev), P(rows), P(x), x.stride(0), n, P(out),
              out.stride(0), _lib.stream_ptr())


def copy_rows(src: torch.Tensor, dst: torch.Tensor, *, m: int, m_dev=None, src_idx=None,
              dst_idx=None, row_bytes: Optional[int] = None) -> None:
    rb = row_bytes if row_bytes is not None else src.stride(0) * src.element_size()
    _lib.call("fb_copy_rows", m, P(m_dev), P(src_idx), P(dst_idx), P(src), P(dst), rb,
              _lib.stream_ptr())


def logits_to_g(logits: torch.Tensor, vw: int, v_out: int, *, m: int, m_dev=None,
                src_rows=None, slots=None, g_pool=None, eos_out=None) -> None:
    _lib.call("fb_logits_to_g", m, P(m_dev), P(logits), logits.stride(0), P(src_rows), vw, v_out,
              P(slots), P(g_pool), _ld(g_pool), P(eos_out), _lib.stream_ptr())


def stats_to_g(logits: torch.Tensor, stats: torch.Tensor, vw: int, v_out: int, *, m: int,
               m_dev=None, src_rows=None, slots=None, g_pool=None, eos_out=None,
               seg_ws=None, stat_out=None, stat_in=None, fus=None, fus_eos: int = 0) -> None:
    """stat_out: per-row {M_w, lse} pairs to reuse; stat_in: reuse them (by
    source row) instead of the statistics pass; fus: also add each row's
    log P(</s>) into its fusion row's <eos> column (fb_eos_fixup, fused)."""
    _lib.call("fb_stats_to_g", m, P(m_dev), P(logits), logits.stride(0), P(stats), v_out,
              P(src_rows), vw, P(slots), P(g_pool), _ld(g_pool), P(eos_out), P(seg_ws),
              P(stat_out), P(stat_in), P(fus), 0 if fus is None else fus.stride(0), fus_eos,
              _lib.stream_ptr())
