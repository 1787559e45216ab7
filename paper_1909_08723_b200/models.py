"""Random-init neural scorers on the device, behind the reference contracts.

* ``AttnLstmScorer`` -- ``AcousticScorer`` (reference ``decoder.py:109-128``):
  BiLSTM encoder + attention-LSTM decoder (equations in
  DESIGN.md §3).  ``is_device_scorer`` routes ``decode_batch`` to the fused
  engine; ``init/step/reorder`` also work one utterance at a time for the
  plugin driver and the kernel parity tests.
* ``LstmWordLM`` -- ``WordLM`` (reference ``word_lm.py:160-186``): tied-
  embedding LSTM LM.  ``is_device_lm`` makes a
  ``LookaheadFusion`` over it device-native.
* ``LstmSubwordLM`` -- ``CharLM`` (reference ``char_lm.py:23-33``): token-level
  LSTM LM for ``SubwordFusion`` (config 4); device-native in the fused engine,
  where its rows never materialise (the selection kernel reads its fp32 logits
  and an fp64 log-normaliser per row).

Weights are stored for the kernels: LSTM gate rows interleaved (row 4u+q =
gate q of unit u), input and recurrent matrices concatenated along K so one
GEMM produces all gates, K zero-padded to the GEMM granule.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import itertools
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .fusion import _device
from .synth import AsrDims, LmDims, SubwordLmDims

KGRAN = 64           # K granule of the tensor-core GEMM (one 128 B swizzle atom of bf16)
# Score-producing projections (AM / LM logits) drain the TMEM accumulator every
# 64-K chunk: the tensor core's accumulation truncates, which otherwise biases
# logits toward zero and shows up in long flat decodes.
KCB_LOGITS = 1
import os as _os
# bf16 planes of the word-LM activations (dev knob; 2 planes measured +2 % c2
# throughput at unchanged parity -- 3 keeps every GEMM fp32-accurate)
LM_PLANES = int(_os.environ.get("FB_LM_PLANES", "3"))     # capped at the format's planes
# stream-K for the word-LM LSTM GEMMs (few event rows -> fewer tiles than SMs)
LM_SPLITK = _os.environ.get("FB_LM_SPLITK", "0") == "1"
# fused engine: per-GEMM A operands, h planes from the epilogues, prev-step
# segments packed on a side stream (dev knob to compare against the plain path)
AM_PIPELINE = _os.environ.get("FB_AM_PIPELINE", "1") == "1"
# TMEM accumulation chunk (K blocks of 64) per GEMM family: the tensor core's
# in-TMEM fp32 adds truncate, so long chunks bias every pre-activation toward
# zero; a looping 470-step c5 decode drifted -6.5e-4 from the fp64 model with
# the library default (4 blocks) in every GEMM and -4e-9/step with 1 block
# (scripts/parity_drift.py); the decoder LSTM GEMMs carry it (1 block there:
# -6e-8/step at +3 % decode time; the encoder and LM GEMMs do not matter).
# 0 = library default.
KCB_AM = int(_os.environ.get("FB_KCB_AM", "1"))       # attention-decoder LSTM + query
KCB_ENC = int(_os.environ.get("FB_KCB_ENC", "0"))     # encoder input + key projections
KCB_LM = int(_os.environ.get("FB_KCB_LM", "0"))       # word / token LM GEMMs
# fused GEMM epilogues: E_q = exp(2 q) for the attention, log-softmax of the
# acoustic output (dev knob for A/B timing)
FUSE_EPI = _os.environ.get("FB_FUSE_EPI", "1") == "1"
# fused engine: the attention context kernel writes the acoustic output GEMM's
# A (context planes at each row's compact position) instead of a pack launch
AM_CTX_PLANES = _os.environ.get("FB_AM_CTX_PLANES", "1") == "1"


def _pad(k: int, g: int = KGRAN) -> int:
    return (k + g - 1) // g * g


def interleave_gates(w: np.ndarray, hidden: int) -> np.ndarray:
    """Rows (q*H + u) -> (4u + q) for q in (i, f, g, o)."""
    tail = w.shape[1:]
    return np.ascontiguousarray(
        w.reshape(4, hidden, *tail).swapaxes(0, 1).reshape(4 * hidden, *tail))


def _dev(a, device, cols: Optional[int] = None) -> torch.Tensor:
    a = np.ascontiguousarray(a, np.float32)
    if cols is not None and a.ndim == 2 and a.shape[1] != cols:
        z = np.zeros((a.shape[0], cols), np.float32)
        z[:, :a.shape[1]] = a
        a = z
    return torch.as_tensor(a, device=device)


def _devw(a, device, cols: Optional[int] = None) -> torch.Tensor:
    """GEMM weight operand in the library's operand format (exact: the
    synthesizer rounds weights to bf16), K zero-padded to the granule."""
    return K.operand_weight(_dev(a, device, cols))


def split_scratch(rows: int, k: int, device) -> torch.Tensor:
    """A-operand buffer [planes, rows, k] for the split fp32 activations."""
    return K.operand_planes(rows, k, device)


@dataclass
class LstmLayer:
    w: torch.Tensor        # [4H, k_pad] gate-interleaved, [W_ih | W_hh] along K
    b: torch.Tensor        # [4H]
    k_in: int
    hidden: int

    @property
    def k_pad(self) -> int:
        return self.w.shape[1]


class AsrWeights:
    """Device copies of the encoder/decoder weights in kernel layout."""

    def __init__(self, W: Dict[str, np.ndarray], d: AsrDims, device):
        self.d = d
        He, H, C_, A = d.enc_hidden, d.dec_hidden, d.ctx, d.att
        # per layer: both directions' input projections as ONE GEMM operand
        # [W_ih_fwd; W_ih_bwd] (gate-interleaved) + biases, and W_hh per direction
        self.enc = []
        for l in range(d.enc_layers):
            fin = d.feat_dim * d.subsample if l == 0 else 2 * He
            w_ih = np.concatenate([interleave_gates(W[f"enc.{l}.{r}.w_ih"], He) for r in range(2)])
            b = np.concatenate([interleave_gates(W[f"enc.{l}.{r}.b"], He) for r in range(2)])
            w_hh = [_devw(interleave_gates(W[f"enc.{l}.{r}.w_hh"], He), device, _pad(He))
                    for r in range(2)]
            self.enc.append((_devw(w_ih, device, _pad(fin)), _dev(b, device), w_hh))
        self.emb = _dev(W["dec.emb"], device)
        self.dec: List[LstmLayer] = []
        for l in range(d.dec_layers):
            fin = (d.emb + C_) if l == 0 else (H + C_)
            w = np.concatenate([W[f"dec.{l}.w_ih"], W[f"dec.{l}.w_hh"]], axis=1)
            self.dec.append(LstmLayer(_devw(interleave_gates(w, H), device, _pad(fin + H)),
                                      _dev(interleave_gates(W[f"dec.{l}.b"], H), device),
                                      fin + H, H))
        self.w_k = _devw(W["dec.att.w_k"], device, _pad(C_))
        self.b_k = _dev(W["dec.att.b_k"], device)
        self.w_q = _devw(W["dec.att.w_q"], device, _pad(H))
        self.v = _dev(W["dec.att.v"], device)
        self.w_out = _devw(W["dec.out.w"], device, _pad(H + C_))
        self.b_out = _dev(W["dec.out.b"], device)
        self.k_max = max([l.k_pad for l in self.dec] + [self.w_q.shape[1], self.w_out.shape[1],
                                                        self.w_k.shape[1]])


class AmState:
    """Decoder state per slot: h/c per layer, attention context."""

    def __init__(self, L: int, N: int, H: int, C_: int, device):
        self.h = torch.zeros((L, N, H), dtype=torch.float32, device=device)
        self.c = torch.zeros((L, N, H), dtype=torch.float32, device=device)
        self.ctx = torch.zeros((N, C_), dtype=torch.float32, device=device)


class Encoder:
    """Frame stacking + stacked BiLSTM on the device.  The backward direction
    runs forward over per-utterance reversed frames, so variable lengths need
    no masking (frames past an utterance's end are never attended)."""

    def __init__(self, w: AsrWeights, device):
        self.w = w
        self.device = device
        self.streams = None
        self._pinned = None

    def stage(self, feats: Sequence[np.ndarray], pin: bool = False, to_device: bool = False,
              chunks: int = 4):
        """Host-side frame stacking into one [B*TM, Din_pad] array (+ lengths).
        to_device: also upload it, chunk by chunk (utterance blocks), each chunk's
        host->device copy running while the host threads stack the next one; the
        device tensor is returned (the pinned buffer must not be restaged before
        the stream has consumed it)."""
        d = self.w.d
        B = len(feats)
        T = [int(x.shape[0]) // d.subsample for x in feats]
        if min(T) < 1:
            raise ValueError("utterance shorter than the subsampling factor")
        TM = max(T)
        Din = d.feat_dim * d.subsample
        shape = (B, TM, _pad(Din))
        if pin:
            # reuse one pinned staging buffer (cudaHostAlloc per call costs more
            # than the copy); the caller must consume it before the next stage()
            n = B * TM * _pad(Din)
            if self._pinned is None or self._pinned.numel() < n:
                # zeroed once: later batches leave finite stale values in padding,
                # which only meets zero weight columns / unattended frames
                self._pinned = torch.zeros(n, dtype=torch.float32, pin_memory=True)
            x = self._pinned[:n].view(shape)
        else:
            x = torch.zeros(shape, dtype=torch.float32)
        xn = x.numpy()
        xd = (torch.empty(shape, dtype=torch.float32, device=self.device) if to_device
              else None)
        nchunk = max(1, min(chunks if to_device else 1, B))
        bounds = [B * i // nchunk for i in range(nchunk + 1)]
        keep = []
        for c in range(nchunk):
            u0, u1 = bounds[c], bounds[c + 1]
            if _pad(Din) == Din:
                # contiguous per-utterance copies on the C++ thread pool
                srcs = []
                for f in feats[u0:u1]:
                    a = np.ascontiguousarray(f, np.float32)
                    keep.append(a)
                    srcs.append(a.ctypes.data)
                row = Din * 4
                dsts = [xn.ctypes.data + u * TM * row for u in range(u0, u1)]
                nbytes = np.asarray([T[u] * row for u in range(u0, u1)], np.int64)
                n = len(srcs)
                _lib.call("fb_host_copy_batch", n, (C.c_void_p * n)(*srcs),
                          (C.c_void_p * n)(*dsts), nbytes.ctypes.data, 16)
            else:
                for u in range(u0, u1):
                    f = feats[u]
                    xn[u, :T[u], :Din] = np.asarray(f, np.float32)[:T[u] * d.subsample].reshape(
                        T[u], Din)
            if xd is not None:
                xd[u0:u1].copy_(x[u0:u1], non_blocking=True)
        if xd is not None:
            return xd.reshape(B * TM, -1), T
        return x.reshape(B * TM, -1), T

    def __call__(self, feats, lengths: Optional[Sequence[int]] = None, out=None):
        """feats: list of [T, feat_dim] arrays, or a staged device tensor
        [B*TM, Din_pad] with ``lengths`` (encoder frames per utterance)."""
        d = self.w.d
        dev = self.device
        if lengths is None:
            X, T = self.stage(feats)
            X = X.to(dev, non_blocking=False)
        else:
            X, T = feats, list(lengths)
        B = len(T)
        TM = X.shape[0] // B
        t_dev = torch.as_tensor(np.asarray(T, np.int32)).to(dev, non_blocking=True)
        He = d.enc_hidden
        kr = _pad(He)
        kout = _pad(2 * He)
        big = split_scratch(B * TM, max(X.shape[1], kout), dev)
        if self.streams is None:
            self.streams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
        planes, pdt, _ = K.operand_format()
        for l, (w_ih, b, w_hh) in enumerate(self.w.enc):
            kin = X.shape[1]
            # both directions' input projections in one GEMM: xp [B*TM, 8He];
            # the backward recurrence reads its half in reversed time per
            # utterance (t_rev), so no reversed copy of the input is made
            K.pack(big, [(X, kin, 0)], m=B * TM, k_pad=kin, split=True)
            xp = torch.empty((B * TM, 8 * He), dtype=torch.float32, device=dev)
            K.gemm_tc(big[:, :, :kin], w_ih, m=B * TM, k=kin, bias=b, out=xp, kcb=KCB_ENC,
                      k_alg=d.feat_dim * d.subsample if l == 0 else 2 * He)
            # both directions write the next layer's input [h_fwd | h_bwd] in
            # forward time order, in place (no concatenation / un-reversal pass)
            Xn = (torch.zeros if kout != 2 * He else torch.empty)(
                (B * TM, kout), dtype=torch.float32, device=dev)
            main = torch.cuda.current_stream(dev)
            for r in range(2):
                st = self.streams[r]
                st.wait_stream(main)
                rec = torch.zeros((2, planes, B, kr), dtype=pdt, device=dev)
                sync = torch.zeros(32 * ((B + 127) // 128), dtype=torch.int32, device=dev)
                for tns in (rec, sync, xp, Xn, t_dev):
                    tns.record_stream(st)
                with torch.cuda.stream(st):
                    # one persistent cooperative launch per direction
                    e0 = K.log_gemm_begin()
                    _lib.call("fb_lstm_recurrence", TM, B, He, _lib.ptr(w_hh[r]), kr,
                              _lib.ptr(xp) + 4 * (4 * He) * r, TM * 8 * He, 8 * He,
                              _lib.ptr(Xn) + 4 * He * r, TM * kout, kout,
                              _lib.ptr(rec), _lib.ptr(sync), w_hh[r].fb_acc_scale,
                              _lib.ptr(t_dev) if r == 1 else None, int(st.cuda_stream))
                    K.log_gemm_end(e0, TM * B, None, 4 * He, He)
            for st in self.streams:
                main.wait_stream(st)
            X = Xn
        C_ = 2 * He
        exact = True
        if out is not None:
            # session buffers may be larger than the batch (B and frame
            # capacity of a corpus-wide session): fill the leading block
            enc_o, keys_o = out
            exact = tuple(enc_o.shape[:2]) == (B, TM) and keys_o.shape[2] == TM
            if exact:
                enc_o.view(B * TM, C_).copy_(X[:, :C_])
            else:
                enc_o[:B, :TM].copy_(X[:, :C_].view(B, TM, C_))
            enc = enc_o
            keys = keys_o if exact else torch.empty((B, d.att, TM), dtype=torch.float32,
                                                    device=dev)
        else:
            enc = X[:, :C_].contiguous()
            keys = torch.empty((B, d.att, TM), dtype=torch.float32, device=dev)
        kk = self.w.w_k.shape[1]
        K.pack(big, [(X, kk, 0)], m=B * TM, k_pad=kk, split=True)
        kraw = torch.empty((B * TM, d.att), dtype=torch.float32, device=dev)
        K.gemm_tc(big[:, :, :kk], self.w.w_k, m=B * TM, k=kk, bias=self.w.b_k, out=kraw, kcb=KCB_ENC,
                  k_alg=C_)
        # the attention kernels consume E_K^T = exp(2 K) per utterance as [A, T]
        # (tanh via one reciprocal; frames contiguous for the energy kernel)
        _lib.call("fb_keys_exp2t", B, TM, d.att, _lib.ptr(kraw), _lib.ptr(keys),
                  _lib.stream_ptr())
        if not exact:
            keys_o[:B, :, :TM].copy_(keys)
            return enc_o, keys_o, T
        return enc.view(B, TM, C_), keys.view(B, d.att, TM), T


class DecoderStep:
    """One attention-LSTM decoder step over a compact row list (slot layout)."""

    def __init__(self, w: AsrWeights, eos_id: int, device):
        self.w = w
        self.eos = eos_id
        self.device = device

    def __call__(self, *, N: int, rows, m: int, m_dev, parent, last_tok, prev: AmState,
                 cur: AmState, scratch: torch.Tensor, q: torch.Tensor, logits: torch.Tensor,
                 am_logp: torch.Tensor, cfg_ref, num_utts: int, active, n_live, t_enc,
                 keys, enc, acc_in, acc_out, cov, energy, sync, attn_out=None,
                 timer=None, abufs=None, pack_stream=None, row_pos=None) -> None:
        w, d = self.w, self.w.d
        tm = timer if timer is not None else _null_timer
        H, C_, E = d.dec_hidden, d.ctx, d.emb
        L = d.dec_layers
        kw = dict(m=m, m_dev=m_dev, rows=rows, parent=parent)
        if abufs is not None:
            self._pipelined(abufs, pack_stream, tm, kw, N=N, m=m, m_dev=m_dev, rows=rows,
                            parent=parent, last_tok=last_tok, prev=prev, cur=cur, q=q,
                            logits=logits, am_logp=am_logp, cfg_ref=cfg_ref,
                            num_utts=num_utts, active=active, n_live=n_live, t_enc=t_enc,
                            keys=keys, enc=enc, acc_in=acc_in, acc_out=acc_out, cov=cov,
                            energy=energy, sync=sync, attn_out=attn_out, row_pos=row_pos)
            return
        span = tm("am_lstm")
        span.__enter__()
        for l, lay in enumerate(w.dec):
            if l == 0:
                segs = [(w.emb, E, 3), (prev.ctx, C_, 2), (prev.h[0], H, 2)]
            else:
                segs = [(cur.h[l - 1], H, 1), (prev.ctx, C_, 2), (prev.h[l], H, 2)]
            K.pack(scratch, segs, tokens=last_tok, tok_default=self.eos, k_pad=lay.k_pad,
                   split=True, **kw)
            K.gemm_tc(scratch, lay.w, k=lay.k_pad, bias=lay.b, mode=1, hidden=H, kcb=KCB_AM,
                      c_in=prev.c[l], c_out=cur.c[l], h_out=cur.h[l],
                      h_res=cur.h[l - 1] if l > 0 else None, k_alg=lay.k_in, **kw)
        span.__exit__(None, None, None)
        top = cur.h[L - 1]
        kq = w.w_q.shape[1]
        K.pack(scratch, [(top, H, 1)], k_pad=kq, split=True, **kw)
        K.gemm_tc(scratch, w.w_q, k=kq, out=q, m=m, m_dev=m_dev, rows=rows, k_alg=H, kcb=KCB_AM)
        with tm("am_attention"):
            _lib.call("fb_attention_step", cfg_ref, num_utts, _lib.ptr(active),
                      _lib.ptr(n_live), _lib.ptr(t_enc), _lib.ptr(keys), _lib.ptr(enc), d.att, C_,
                      _lib.ptr(w.v), _lib.ptr(q), q.stride(0), _lib.ptr(parent),
                      _lib.ptr(acc_in), _lib.ptr(acc_out), _lib.ptr(cov), _lib.ptr(cur.ctx),
                      cur.ctx.stride(0), _lib.ptr(attn_out),
                      0 if attn_out is None else attn_out.stride(0), _lib.ptr(energy),
                      _lib.ptr(sync), 0, None, 0, 0, None, _lib.stream_ptr())
        ko = w.w_out.shape[1]
        with tm("am_output"):
            K.pack(scratch, [(top, H, 1), (cur.ctx, C_, 1)], k_pad=ko, split=True, **kw)
            K.gemm_tc(scratch, w.w_out, k=ko, bias=w.b_out, out=logits, m=m, m_dev=m_dev,
                      rows=rows, k_alg=H + C_, kcb=KCB_LOGITS)
            K.log_softmax_rows(logits, am_logp, d.vocab, m=m, m_dev=m_dev, rows=rows)

    def abuf_shapes(self):
        """k_pad of the per-layer A operands + the output projection's."""
        return [lay.k_pad for lay in self.w.dec] + [self.w.w_out.shape[1]]

    def _pipelined(self, A, pack_stream, tm, kw, *, N, m, m_dev, rows, parent, last_tok, prev,
                   cur, q, logits, am_logp, cfg_ref, num_utts, active, n_live, t_enc, keys,
                   enc, acc_in, acc_out, cov, energy, sync, attn_out, row_pos=None):
        """Same step with one A operand per GEMM: each LSTM epilogue writes its h
        as bf16 planes straight into the next GEMM's A (h_split, GEMM row
        order), and the previous-step segments of layers 1.. (ctx, h gathered by
        parent) are packed on `pack_stream` while layer 0 runs -- two packs on
        the critical path instead of L + 2.  With `row_pos` (each slot's
        position in `rows`, written by the search's row compaction) the
        attention context kernel stores the context planes of the output A
        itself and the second pack goes too."""
        w, d = self.w, self.w.d
        H, C_, E = d.dec_hidden, d.ctx, d.emb
        L = d.dec_layers
        main = torch.cuda.current_stream()
        if L > 1:
            if pack_stream is not None:
                pack_stream.wait_stream(main)
                ctx = torch.cuda.stream(pack_stream)
            else:
                ctx = contextlib.nullcontext()
            with ctx:
                for l in range(1, L):
                    K.pack(A[l], [(None, H, 5), (prev.ctx, C_, 2), (prev.h[l], H, 2)],
                           k_pad=w.dec[l].k_pad, split=True, **kw)
        kq = w.w_q.shape[1]
        ko = w.w_out.shape[1]
        q_from_out = kq == H            # q's A = the first H columns of the output A
        with tm("am_lstm"):
            for l, lay in enumerate(w.dec):
                if l == 0:
                    K.pack(A[0], [(w.emb, E, 3), (prev.ctx, C_, 2), (prev.h[0], H, 2)],
                           tokens=last_tok, tok_default=self.eos, k_pad=lay.k_pad, split=True,
                           **kw)
                elif l == 1 and pack_stream is not None:
                    main.wait_stream(pack_stream)
                nxt = A[l + 1] if l + 1 < L else A[L]
                K.gemm_tc(A[l], lay.w, k=lay.k_pad, bias=lay.b, mode=1, hidden=H, kcb=KCB_AM,
                          c_in=prev.c[l], c_out=cur.c[l], h_out=cur.h[l],
                          h_res=cur.h[l - 1] if l > 0 else None, k_alg=lay.k_in,
                          h_split=nxt, hs_by_row=True, **kw)
        top = cur.h[L - 1]
        # the epilogue stores E_q = exp(2 q) (fb_attention_step q_is_exp)
        if q_from_out:
            K.gemm_tc(A[L], w.w_q, k=kq, out=q, m=m, m_dev=m_dev, rows=rows, k_alg=H, kcb=KCB_AM,
                      out_exp2=FUSE_EPI)
        else:
            K.pack(A[0], [(top, H, 1)], k_pad=kq, split=True, **kw)
            K.gemm_tc(A[0], w.w_q, k=kq, out=q, m=m, m_dev=m_dev, rows=rows, k_alg=H, kcb=KCB_AM,
                      out_exp2=FUSE_EPI)
        with tm("am_attention"):
            _lib.call("fb_attention_step", cfg_ref, num_utts, _lib.ptr(active),
                      _lib.ptr(n_live), _lib.ptr(t_enc), _lib.ptr(keys), _lib.ptr(enc), d.att, C_,
                      _lib.ptr(w.v), _lib.ptr(q), q.stride(0), _lib.ptr(parent),
                      _lib.ptr(acc_in), _lib.ptr(acc_out), _lib.ptr(cov), _lib.ptr(cur.ctx),
                      cur.ctx.stride(0), _lib.ptr(attn_out),
                      0 if attn_out is None else attn_out.stride(0), _lib.ptr(energy),
                      _lib.ptr(sync), 1 if FUSE_EPI else 0,
                      None if row_pos is None else A[L].data_ptr() + H * A[L].element_size(),
                      A[L].stride(0), A[L].stride(1), _lib.ptr(row_pos), _lib.stream_ptr())
        with tm("am_output"):
            if row_pos is None:
                K.pack(A[L], [(None, H, 5), (cur.ctx, C_, 1)], k_pad=ko, split=True, **kw)
            if d.vocab <= 64 and FUSE_EPI:
                # the epilogue holds whole rows: log-softmax fused, logits never stored
                K.gemm_tc(A[L], w.w_out, k=ko, bias=w.b_out, out=am_logp, m=m, m_dev=m_dev,
                          rows=rows, k_alg=H + C_, kcb=KCB_LOGITS, out_logsoftmax=True)
            else:
                K.gemm_tc(A[L], w.w_out, k=ko, bias=w.b_out, out=logits, m=m, m_dev=m_dev,
                          rows=rows, k_alg=H + C_, kcb=KCB_LOGITS)
                K.log_softmax_rows(logits, am_logp, d.vocab, m=m, m_dev=m_dev, rows=rows)


class _NullSpan:
    def __call__(self, name):
        return self

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_null_timer = _NullSpan()


@dataclass
class _UttState:
    enc: torch.Tensor      # [1, T, C]
    keys: torch.Tensor     # [1, A, T]  E_K^T = exp(2 K)
    T: int
    am: AmState            # n rows


class AttnLstmScorer:
    """AcousticScorer over the device attention-LSTM model."""

    is_device_scorer = True

    def __init__(self, W: Dict[str, np.ndarray], dims: AsrDims, eos_id: int, device=None):
        self.device = _device(device)
        self.dims = dims
        self.eos_id = eos_id
        self.weights = AsrWeights(W, dims, self.device)
        self.encoder = Encoder(self.weights, self.device)
        self.step_fn = DecoderStep(self.weights, eos_id, self.device)

    # ---- reference AcousticScorer protocol (one utterance) ------------------
    def init(self, features) -> _UttState:
        enc, keys, T = self.encoder([np.asarray(features.data, np.float32)])
        d = self.dims
        return _UttState(enc, keys, T[0], AmState(d.dec_layers, 1, d.dec_hidden, d.ctx,
                                                  self.device))

    def enc_length(self, state: _UttState) -> int:
        return state.T

    def step(self, state: _UttState, last_tokens: Sequence[int]):
        d, dev = self.dims, self.device
        n = len(last_tokens)
        cur = AmState(d.dec_layers, n, d.dec_hidden, d.ctx, dev)
        rows = torch.arange(n, dtype=torch.int32, device=dev)
        tok = torch.as_tensor(np.asarray(last_tokens, np.int32), device=dev)
        cfg = _lib.FbSearchCfg(beam=n, vocab=d.vocab, t_max=state.T)
        one = torch.ones(1, dtype=torch.int32, device=dev)
        nl = torch.full((1,), n, dtype=torch.int32, device=dev)
        te = torch.full((1,), state.T, dtype=torch.int32, device=dev)
        acc0 = torch.zeros((n, state.T), dtype=torch.float64, device=dev)
        acc1 = torch.empty_like(acc0)
        attn = torch.empty((n, state.T), dtype=torch.float32, device=dev)
        scratch = split_scratch(n, self.weights.k_max, dev)
        energy = torch.empty((2, n, state.T), dtype=torch.float32, device=dev)
        q = torch.empty((n, d.att), dtype=torch.float32, device=dev)
        logits = torch.empty((n, d.vocab), dtype=torch.float32, device=dev)
        logp = torch.empty((n, d.vocab), dtype=torch.float32, device=dev)
        self.step_fn(N=n, rows=rows, m=n, m_dev=None, parent=rows, last_tok=tok, prev=state.am,
                     cur=cur, scratch=scratch, q=q, logits=logits, am_logp=logp,
                     cfg_ref=C.byref(cfg), num_utts=1, active=one, n_live=nl, t_enc=te,
                     keys=state.keys, enc=state.enc, acc_in=acc0, acc_out=acc1, cov=None,
                     energy=energy, sync=torch.zeros((n + 1) // 2 + 1, dtype=torch.int32,
                                                     device=dev), attn_out=attn)
        return (logp.cpu().numpy(), attn.cpu().numpy(),
                _UttState(state.enc, state.keys, state.T, cur))

    def reorder(self, state: _UttState, parent_indices: Sequence[int]) -> _UttState:
        idx = torch.as_tensor(np.asarray(parent_indices, np.int64), device=self.device)
        am = AmState(self.dims.dec_layers, len(idx), self.dims.dec_hidden, self.dims.ctx,
                     self.device)
        am.h = state.am.h[:, idx].contiguous()
        am.c = state.am.c[:, idx].contiguous()
        am.ctx = state.am.ctx[idx].contiguous()
        return _UttState(state.enc, state.keys, state.T, am)


# ---- word LM -----------------------------------------------------------------
class LmWeights:
    def __init__(self, W: Dict[str, np.ndarray], d: LmDims, device):
        self.d = d
        H = d.hidden
        self.v_out = d.words + 3
        self.k_out = _pad(H)
        self.emb = _dev(W["lm.emb"], device, self.k_out)      # [V+3, k_out] fp32 input rows
        self.emb_w = K.operand_weight(self.emb)                # tied output weight operand
        self.b_out = _dev(W["lm.b_out"], device)
        self.layers: List[LstmLayer] = []
        for l in range(d.layers):
            w = np.concatenate([W[f"lm.{l}.w_ih"], W[f"lm.{l}.w_hh"]], axis=1)
            self.layers.append(LstmLayer(_devw(interleave_gates(w, H), device, _pad(2 * H)),
                                         _dev(interleave_gates(W[f"lm.{l}.b"], H), device),
                                         2 * H, H))
        self.k_max = max([l.k_pad for l in self.layers] + [self.k_out])
        self.eos_tok, self.unk_tok, self.bos_tok = d.words, d.words + 1, d.words + 2
        self.in_width = H
        self.out_w = self.emb_w
        self.stats_vw = d.words
        # the 65k-way output feeds look-ahead masses (sums over word ranges), not
        # argmax-per-step scores: coarse chunking is accurate enough there (c2
        # parity) and KCB_LOGITS would cost ~6% of the c2 decode.  5 blocks:
        # K = 1216 in four chunks = the four TMEM slots, so the MMA runs a whole
        # tile ahead of the statistics epilogue (95 -> 91.5 us at 240 rows)
        self.kcb_out = int(_os.environ.get("FB_KCB_LMOUT", "5"))


def lm_step(w: LmWeights, *, m: int, m_dev, state_src, src_idx, state_dst, ranks,
            tok_default: int, scratch: torch.Tensor, logits: Optional[torch.Tensor],
            timer=None, stats: Optional[torch.Tensor] = None, splitk=None, abufs=None,
            pack_stream=None) -> None:
    """Batched LSTM-LM step.  Row i: input token ranks[i] (or tok_default),
    recurrent state from state_src[src_idx[i]] (None -> zero state), new state
    into state_dst[i]; state tensors are [rows, L, 2, H] (h then c per layer).
    Optionally logits[i] = E . h_top + b.
    abufs: one A operand per GEMM (k_pad of each layer, then k_out with zeroed
    padding): every layer's epilogue writes its h planes into the next A, the
    recurrent-h segments of layers 1.. are packed on pack_stream (or inline)."""
    H = w.d.hidden
    L = len(w.layers)
    if abufs is not None and state_src is not None:
        main = torch.cuda.current_stream()
        if L > 1:
            if pack_stream is not None:
                pack_stream.wait_stream(main)
                ctx = torch.cuda.stream(pack_stream)
            else:
                ctx = contextlib.nullcontext()
            with ctx:
                for l in range(1, L):
                    K.pack(abufs[l], [(None, H, 5), (state_src[:, l, 0], H, 1, state_src.stride(0))],
                           m=m, m_dev=m_dev, rows=src_idx, k_pad=w.layers[l].k_pad, split=True)
        for l, lay in enumerate(w.layers):
            if l == 0:
                K.pack(abufs[0], [(w.emb, w.in_width, 4, w.emb.stride(0)),
                                  (state_src[:, 0, 0], H, 1, state_src.stride(0))],
                       m=m, m_dev=m_dev, rows=src_idx, ranks=ranks, tok_default=tok_default,
                       k_pad=lay.k_pad, split=True)
            elif l == 1 and pack_stream is not None:
                main.wait_stream(pack_stream)
            nxt = abufs[l + 1] if l + 1 < L else (abufs[L] if logits is not None else None)
            K.gemm_tc(abufs[l][:LM_PLANES], lay.w, m=m, m_dev=m_dev, k=lay.k_pad, bias=lay.b, kcb=KCB_LM,
                      mode=1, hidden=H, parent=src_idx, c_in=state_src[:, l, 1],
                      c_out=state_dst[:, l, 1], h_out=state_dst[:, l, 0], k_alg=lay.k_in,
                      splitk=splitk, h_split=nxt, hs_by_row=True)
        if logits is not None:
            kw = dict(m=m, m_dev=m_dev, k=w.k_out, bias=w.b_out, out=logits, row_stats=stats,
                      stats_vw=w.stats_vw, k_alg=H, kcb=w.kcb_out)
            with (timer("lm_out_gemm") if timer is not None else contextlib.nullcontext()):
                K.gemm_tc(abufs[L][:LM_PLANES], w.out_w, **kw)
        return
    for l, lay in enumerate(w.layers):
        if l == 0:
            x = (w.emb, w.in_width, 4, w.emb.stride(0))
        else:
            x = (state_dst[:, l - 1, 0], H, 0, state_dst.stride(0))
        if state_src is None:
            hseg = (None, H, 1, 0)
            c_in = None
        else:
            hseg = (state_src[:, l, 0], H, 1, state_src.stride(0))
            c_in = state_src[:, l, 1]
        K.pack(scratch, [x, hseg], m=m, m_dev=m_dev, rows=src_idx, ranks=ranks,
               tok_default=tok_default, k_pad=lay.k_pad, split=True)
        K.gemm_tc(scratch[:LM_PLANES], lay.w, m=m, m_dev=m_dev, k=lay.k_pad, bias=lay.b, kcb=KCB_LM,
                  mode=1,
                  hidden=H, parent=src_idx, c_in=c_in, c_out=state_dst[:, l, 1],
                  h_out=state_dst[:, l, 0], k_alg=lay.k_in, splitk=splitk)
    if logits is not None:
        K.pack(scratch, [(state_dst[:, L - 1, 0], H, 0, state_dst.stride(0))], m=m, m_dev=m_dev,
               k_pad=w.k_out, split=True)
        kw = dict(m=m, m_dev=m_dev, k=w.k_out, bias=w.b_out, out=logits, row_stats=stats,
                  stats_vw=w.stats_vw, k_alg=H, kcb=w.kcb_out)
        if timer is not None:
            with timer("lm_out_gemm"):
                K.gemm_tc(scratch[:LM_PLANES], w.out_w, **kw)
        else:
            K.gemm_tc(scratch[:LM_PLANES], w.out_w, **kw)


class _DevHist:
    __slots__ = ("uid", "state", "logits", "_eos")
    _ids = itertools.count()

    def __init__(self, state, logits):
        self.uid = next(_DevHist._ids)
        self.state = state            # [1, L, 2, H]
        self.logits = logits          # [1, V+3]
        self._eos = None


class LstmWordLM:
    """WordLM over the device LSTM LM (outputs: ranks, </s>, <unk>, <s>)."""

    is_device_lm = True

    def __init__(self, W: Dict[str, np.ndarray], dims: LmDims, device=None):
        self.device = _device(device)
        self.dims = dims
        self.vocab_size = dims.words
        self.weights = LmWeights(W, dims, self.device)
        self._kids: Dict[tuple, _DevHist] = {}
        self._root = self._run(None, self.weights.bos_tok)

    def _run(self, parent: Optional[_DevHist], token: int) -> _DevHist:
        w, d, dev = self.weights, self.dims, self.device
        st = torch.empty((1, d.layers, 2, d.hidden), dtype=torch.float32, device=dev)
        lg = torch.empty((1, w.v_out), dtype=torch.float32, device=dev)
        scratch = split_scratch(1, w.k_max, dev)
        lm_step(w, m=1, m_dev=None, state_src=None if parent is None else parent.state,
                src_idx=None, state_dst=st, ranks=None, tok_default=token, scratch=scratch,
                logits=lg)
        return _DevHist(st, lg)

    def start_history(self) -> _DevHist:
        return self._root

    def extend_history(self, hist: _DevHist, rank: int) -> _DevHist:
        if rank != -1 and not 0 <= rank < self.vocab_size:
            raise ValueError(f"word rank {rank} out of range")
        key = (hist.uid, rank)
        kid = self._kids.get(key)
        if kid is None:
            kid = self._run(hist, self.weights.unk_tok if rank == -1 else rank)
            self._kids[key] = kid
        return kid

    def full_distribution(self, hist: _DevHist) -> np.ndarray:
        g = torch.empty((1, self.vocab_size), dtype=torch.float64, device=self.device)
        K.logits_to_g(hist.logits, self.vocab_size, self.weights.v_out, m=1, g_pool=g)
        return np.diff(g[0].cpu().numpy(), prepend=0.0)

    def eos_log_prob(self, hist: _DevHist) -> float:
        if hist._eos is None:
            out = torch.empty(1, dtype=torch.float64, device=self.device)
            K.logits_to_g(hist.logits, self.vocab_size, self.weights.v_out, m=1, eos_out=out)
            hist._eos = float(out.item())
        return hist._eos

    def write_g_rows(self, hists: List[_DevHist], pool: torch.Tensor, slots: torch.Tensor) -> None:
        lg = torch.cat([h.logits for h in hists], dim=0)
        K.logits_to_g(lg, self.vocab_size, self.weights.v_out, m=len(hists), slots=slots,
                      g_pool=pool)


# ---- token-level (subword) LM: CharLM protocol ------------------------------------
SCORE_FLOOR = -30.0            # reference char_lm.py:20


class SubLmWeights:
    """Device weights of the token LSTM LM (same kernel layout as LmWeights)."""

    def __init__(self, W: Dict[str, np.ndarray], d: SubwordLmDims, device):
        self.d = d
        H, E = d.hidden, d.emb
        self.in_width = E
        self.emb = _dev(W["slm.emb"], device, _pad(E))          # [V, E_pad] fp32 input rows
        self.layers: List[LstmLayer] = []
        for l in range(d.layers):
            fin = E if l == 0 else H
            w = np.concatenate([W[f"slm.{l}.w_ih"], W[f"slm.{l}.w_hh"]], axis=1)
            self.layers.append(LstmLayer(_devw(interleave_gates(w, H), device, _pad(fin + H)),
                                         _dev(interleave_gates(W[f"slm.{l}.b"], H), device),
                                         fin + H, H))
        self.k_out = _pad(H)
        self.out_w = _devw(W["slm.out.w"], device, self.k_out)
        self.b_out = _dev(W["slm.out.b"], device)
        self.stats_vw = 0
        self.kcb_out = KCB_LOGITS
        self.k_max = max([l.k_pad for l in self.layers] + [self.k_out])


class _TokState:
    """One hypothesis' LM state after consuming <eos> + its token history."""
    __slots__ = ("state", "logits")

    def __init__(self, state, logits):
        self.state = state            # [1, L, 2, H]
        self.logits = logits          # [1, V] fp32


class LstmSubwordLM:
    """CharLM over the device token LSTM LM.  ``log_probs`` row = fp64
    log-softmax of the fp32 logits over the non-pad tokens, floored at
    SCORE_FLOOR, ``<pad>`` = SCORE_FLOOR (the row contract of char_lm.py:1-7)."""

    is_device_lm = True

    def __init__(self, W: Dict[str, np.ndarray], dims: SubwordLmDims, pad_id: int, eos_id: int,
                 device=None):
        self.device = _device(device)
        self.dims = dims
        self.pad_id, self.eos_id = pad_id, eos_id
        self.score_floor = SCORE_FLOOR
        self.weights = SubLmWeights(W, dims, self.device)
        self._start = self._run(None, [eos_id])[0]

    def _run(self, src: Optional[torch.Tensor], tokens: Sequence[int]) -> List[_TokState]:
        w, d, dev = self.weights, self.dims, self.device
        n = len(tokens)
        st = torch.empty((n, d.layers, 2, d.hidden), dtype=torch.float32, device=dev)
        lg = torch.empty((n, d.vocab), dtype=torch.float32, device=dev)
        scratch = split_scratch(n, w.k_max, dev)
        ranks = torch.as_tensor(np.asarray(tokens, np.int32), device=dev)
        lm_step(w, m=n, m_dev=None, state_src=src, src_idx=None, state_dst=st, ranks=ranks,
                tok_default=self.eos_id, scratch=scratch, logits=lg)
        return [_TokState(st[i:i + 1], lg[i:i + 1]) for i in range(n)]

    # ---- reference CharLM protocol --------------------------------------------
    def start(self) -> _TokState:
        return self._start

    def advance(self, state: _TokState, token_id: int) -> _TokState:
        return self.advance_many([state], [token_id])[0]

    def advance_many(self, states: Sequence[_TokState], tokens: Sequence[int]
                     ) -> List[_TokState]:
        if not states:
            return []
        return self._run(torch.cat([s.state for s in states]), tokens)

    def log_probs(self, state: _TokState) -> np.ndarray:
        return self.log_probs_device([state])[0].cpu().numpy()

    def log_probs_device(self, states: Sequence[_TokState]) -> torch.Tensor:
        lg = torch.cat([s.logits for s in states])
        n, V = lg.shape
        norm = torch.empty(n, dtype=torch.float64, device=self.device)
        _lib.call("fb_row_logsumexp", n, None, None, _lib.ptr(lg), lg.stride(0), V, self.pad_id,
                  _lib.ptr(norm), _lib.stream_ptr())
        rows = (lg.double() - norm[:, None]).clamp_(min=SCORE_FLOOR)
        rows[:, self.pad_id] = SCORE_FLOOR
        return rows


class SubLmState:
    """Token-LM state per slot: h/c per layer (one ping-pong half)."""

    def __init__(self, L: int, N: int, H: int, device):
        self.h = torch.zeros((L, N, H), dtype=torch.float32, device=device)
        self.c = torch.zeros((L, N, H), dtype=torch.float32, device=device)


def subword_step(w: SubLmWeights, *, m: int, m_dev, rows, parent, last_tok, eos_id: int,
                 pad_id: int, prev: SubLmState, cur: SubLmState, scratch: torch.Tensor,
                 logits: torch.Tensor, norm: torch.Tensor) -> None:
    """Token-LM step over the compact row list (slot layout), the same
    parent-indirect recurrence as the decoder: slot r consumes last_tok[r]
    (<eos> at the first step) on top of its parent's state; logits[r] and the
    fp64 log-normaliser over non-pad tokens norm[r]."""
    H = w.d.hidden
    L = len(w.layers)
    kw = dict(m=m, m_dev=m_dev, rows=rows, parent=parent)
    for l, lay in enumerate(w.layers):
        if l == 0:
            segs = [(w.emb, w.in_width, 3), (prev.h[0], H, 2)]
        else:
            segs = [(cur.h[l - 1], H, 1), (prev.h[l], H, 2)]
        K.pack(scratch, segs, tokens=last_tok, tok_default=eos_id, k_pad=lay.k_pad, split=True,
               **kw)
        K.gemm_tc(scratch, lay.w, k=lay.k_pad, bias=lay.b, mode=1, hidden=H, kcb=KCB_LM,
                  c_in=prev.c[l],
                  c_out=cur.c[l], h_out=cur.h[l], k_alg=lay.k_in, **kw)
    K.pack(scratch, [(cur.h[L - 1], H, 1)], k_pad=w.k_out, split=True, **kw)
    K.gemm_tc(scratch, w.out_w, k=w.k_out, bias=w.b_out, out=logits, m=m, m_dev=m_dev,
              rows=rows, k_alg=H, kcb=w.kcb_out)
    _lib.call("fb_row_logsumexp", m, P_(m_dev), P_(rows), P_(logits), logits.stride(0),
              w.d.vocab, pad_id, P_(norm), _lib.stream_ptr())


P_ = _lib.ptr
