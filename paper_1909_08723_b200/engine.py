"""Fused device decode: the whole lock-step loop of ``decode_batch``
(reference ``decoder.py:363-462`` + ``fusion.py:118-233``) on the GPU.

Per step, for the compact list of live rows of active utterances:

 1. attention-LSTM decoder step  (pack -> GEMM+LSTM-cell x L -> query GEMM ->
    attention + fp64 accumulator + coverage -> output GEMM -> log-softmax);
 2. speculative word-LM events for rows at final trie states (the ``<eos>``
    column, fusion.py:181-183): LSTM-LM step + logits + log P(</s>);
 3. look-ahead scores over the CSR trie and fp64 g rows (Eq. 4);
 4. selection kernel (combine, EOS gate, stable top-beam, coverage, finished
    set, early stop, results) -> parent/token per new row, next row list;
 5. trie advance + word-boundary plan; ``<unk>`` LM events; new history slots
    get the LM state and g row of their event.

State never leaves the device; rows index per-slot buffers through ``parent``
(no physical reorder).  The host only polls the live-row count.
"""

from __future__ import annotations

import collections
import contextlib
import ctypes as C
import os
import math
import threading
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .decoder import DecodeConfig, DecodeResult, SearchBuffers, search_cfg
from .errors import ConfigError
from .models import (AM_CTX_PLANES, AM_PIPELINE, LM_SPLITK, AmState, SubLmState, lm_step,
                     split_scratch, subword_step)

P = _lib.ptr


# dev knob: word-boundary g rows reuse the speculative events' statistics
# instead of a second statistics pass (measured 2 ms slower over the c2 decode:
# the extra pass on the side stream shifts the g-row kernels to a better overlap)
_STAT_REUSE = os.environ.get("FB_STAT_REUSE", "0") == "1"


# lock-step tail: below this many live rows the step graphs captured with fine
# attention tiles replace the default ones (frame warps, rows, quads per CTA)
_TAIL_ROWS = int(os.environ.get("FB_TAIL_ROWS", "1500"))
_TAIL_TILING = tuple(int(x) for x in os.environ.get("FB_TAIL_TILING", "4,4,160").split(","))
# lock-step tail: the word-LM LSTM GEMMs of few event rows run stream-K (more
# CTAs over the long K = 2432 loop) in the tail graph set (dev knob)
_TAIL_SPLITK = os.environ.get("FB_TAIL_SPLITK", "0") == "1"
# speculative </s> events unpruned on the side stream beside the acoustic step
# (instead of pruned by the acoustic scores after it)
_SPEC_EARLY = os.environ.get("FB_SPEC_EARLY", "0") == "1"


class _LmPool:
    """History slots (LM state + g row + eos) and per-step LM events."""

    def __init__(self, lw, N: int, device):
        d = lw.d
        self.lw = lw
        self.N = N
        self.P = 2 * N + 2
        L, H = d.layers, d.hidden
        f32, i32 = torch.float32, torch.int32
        z = lambda *s, dt=i32: torch.zeros(s, dtype=dt, device=device)  # noqa: E731
        self.state = torch.zeros((self.P, L, 2, H), dtype=f32, device=device)
        self.g = torch.empty((self.P, d.words), dtype=torch.float64, device=device)
        self.eos = torch.zeros(self.P, dtype=torch.float64, device=device)
        E = 2 * N
        self.ev_state = torch.zeros((E, L, 2, H), dtype=f32, device=device)
        # row stride padded to 16 bytes: the output GEMM stores tiles with TMA
        # rows padded to 32 bytes: 256-bit loads in the g-row passes
        self.ev_logits = torch.empty((E, (lw.v_out + 7) // 8 * 8), dtype=f32,
                                     device=device)[:, :lw.v_out]
        self.ntiles = (lw.v_out + 63) // 64
        self.ev_stats = torch.empty((E, self.ntiles, 4), dtype=f32, device=device)
        self.seg_ws = torch.empty((N, (d.words + 4095) // 4096 + 2), dtype=torch.float64,
                                  device=device)     # segment sums + per-row {M_w, lse}
        self.ev_row, self.ev_rank, self.ev_slot, self.row_ev = z(N), z(N), z(N), z(N)
        self.ev_count = z(1)
        self.trie = [z(N), z(N)]
        self.hist = [z(N), z(N)]
        self.brank = z(N)
        self.bnd_slot, self.bnd_src, self.unk_slot, self.unk_tok = z(N), z(N), z(N), z(N)
        self.late_row, self.late_dst = z(N), z(N)
        self.bnd_count, self.unk_count = z(1), z(1)
        self.mark = z(2 * self.P)
        self.ext_eos = torch.zeros(N, dtype=torch.float64, device=device)
        self.zero_eos = torch.zeros(N, dtype=torch.float64, device=device)
        self.scratch = split_scratch(N, lw.k_max, device)
        # stream-K workspace of the LM LSTM GEMMs (spec and late events never
        # overlap: the side stream joins before the speculative events)
        self.splitk = K.SplitK(device) if LM_SPLITK else None
        self.splitk_tail = (self.splitk or K.SplitK(device)) if _TAIL_SPLITK else None
        # {M_w, lse} per speculative event: reused by the word-boundary g rows
        self.ev_stat = torch.zeros((N, 2), dtype=torch.float64, device=device)
        # per-GEMM A operands (the output one's K padding stays zero)
        self.abufs = ([split_scratch(N, lay.k_pad, device) for lay in lw.layers] +
                      [K.operand_planes(N, lw.k_out, device).zero_()]
                      if AM_PIPELINE else None)

    def start(self) -> None:
        """Slot 0 = LM state after <s> from the zero state (word_lm start_history)."""
        lw = self.lw
        lm_step(lw, m=1, m_dev=None, state_src=None, src_idx=None, state_dst=self.ev_state,
                ranks=None, tok_default=lw.bos_tok, scratch=self.scratch, logits=self.ev_logits)
        self.state[0].copy_(self.ev_state[0])
        K.logits_to_g(self.ev_logits, lw.d.words, lw.v_out, m=1, g_pool=self.g, eos_out=self.eos)


class StageTimer:
    """CUDA-event spans per named stage on the current stream (instrumented
    runs only; the timed bench pass runs without it)."""

    def __init__(self):
        self.spans = {}

    def __call__(self, name: str):
        return _Span(self, name)

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for k, lst in self.spans.items():
            out[k] = (sum(a.elapsed_time(b) for a, b in lst), len(lst))
        return out


class _Span:
    def __init__(self, t: StageTimer, name: str):
        self.t, self.name = t, name

    def __enter__(self):
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)
        self.a.record()
        return self

    def __exit__(self, *exc):
        self.b.record()
        self.t.spans.setdefault(self.name, []).append((self.a, self.b))


class _NoTimer:
    def __call__(self, name):
        return self

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_HINT = threading.local()


@contextlib.contextmanager
def corpus_hint(batch_size: int, t_max: int):
    """decode_corpus: every batch of this corpus fits one session of
    ``batch_size`` utterances and ``t_max`` encoder frames, so the device
    buffers and captured step graphs are built once per corpus, not per batch
    (the last, smaller batch runs with its surplus utterances inactive)."""
    prev = getattr(_HINT, "caps", None)
    _HINT.caps = (int(batch_size), int(t_max))
    try:
        yield
    finally:
        _HINT.caps = prev


def _engine_key(fusion, config: DecodeConfig, token_dict):
    """What a cached engine depends on: the fusion's resources (trie and LM
    objects, penalties), never the fusion instance -- the reference pipeline
    builds a fresh fusion per batch (pipeline.py:148-149) over shared ones."""
    if fusion is None:
        fk = None
    elif hasattr(fusion, "char_lm"):
        fk = ("subword", id(fusion.char_lm))
    else:
        fk = ("lookahead", id(fusion.trie), id(fusion.word_lm), fusion.oov_penalty,
              fusion.score_floor)
    return (fk, tuple(sorted(vars(config).items())), tuple(token_dict.tokens))


_MAX_ENGINES = 2


def decode_fused(features, scorer, fusion, config: DecodeConfig, token_dict
                 ) -> List[DecodeResult]:
    """decode_batch entry: host features -> staged device batch -> engine.
    Engines are cached on the scorer by content (_engine_key) and keep their
    device sessions, so repeated calls -- including decode_corpus with a
    fusion factory -- reuse buffers and CUDA graphs.  One decode at a time per
    scorer: decode_corpus(workers > 1) threads serialise here (the GPU already
    batches; the staging buffer, streams and sessions are shared)."""
    lock = scorer.__dict__.setdefault("_engine_lock", threading.Lock())
    with lock:
        # staging and upload pipelined in utterance chunks (copy of chunk i while
        # the host threads stack chunk i+1)
        X, T = scorer.encoder.stage([np.asarray(f.data, np.float32) for f in features],
                                    pin=True, to_device=True)
        done = torch.cuda.Event()
        done.record()
        key = _engine_key(fusion, config, token_dict)
        cache = scorer.__dict__.setdefault("_fused_cache", collections.OrderedDict())
        dec = cache.get(key)
        if dec is None:
            while len(cache) >= _MAX_ENGINES:
                cache.popitem(last=False)
            dec = cache[key] = FusedDecoder(scorer, fusion, config, token_dict)
        cache.move_to_end(key)
        out = dec.run(X, T, [f.utt_id for f in features], fusion=fusion,
                      caps=getattr(_HINT, "caps", None))
        done.synchronize()          # the pinned staging buffer may be reused afterwards
        return out


class _Session:
    """All device buffers of one batch shape (B, T_max, max_tokens) plus the two
    captured step graphs; reused by every decode of that shape."""

    def __init__(self, dec: "FusedDecoder", B: int, TM: int, MT: int):
        scorer, fusion, config, token_dict = dec.scorer, dec.fusion, dec.config, dec.token_dict
        dev = scorer.device
        w = scorer.weights
        d = w.d
        self.B, self.TM, self.MT = B, TM, MT
        Kb = config.beam_size
        self.K = Kb
        N = self.N = B * Kb
        V = self.V = len(token_dict)
        self.buf = SearchBuffers(B, Kb, MT, TM, dev, vocab=len(token_dict),
                                 select_flags=dec.select_flags)
        self.has_fusion = fusion is not None
        early = (not self.has_fusion) or bool(fusion.nonpositive_scores)
        self.cfg = search_cfg(config, token_dict, self.has_fusion, early, True, MT, TM)
        self.cfg_ref = C.byref(self.cfg)
        self.rows = [torch.zeros(N, dtype=torch.int32, device=dev) for _ in range(2)]
        self.count = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(2)]
        self.views = [_view_with_rows(self.buf, p, self.rows[1 - p], self.count[1 - p])
                      for p in range(2)]
        L, H, C_ = d.dec_layers, d.dec_hidden, d.ctx
        self.X2 = [AmState(L, N, H, C_, dev), AmState(L, N, H, C_, dev)]
        self.scratch = split_scratch(N, w.k_max, dev)
        # one A operand per decoder GEMM (epilogues write the next one's h planes)
        # (zeroed: the output A's context columns come from the attention
        # kernel by row position, its padding columns are never written)
        self.am_abufs = ([split_scratch(N, k, dev).zero_() for k in scorer.step_fn.abuf_shapes()]
                         if AM_PIPELINE else None)
        self.pack_stream = torch.cuda.Stream(device=dev) if AM_PIPELINE else None
        self.q = torch.empty((N, d.att), dtype=torch.float32, device=dev)
        self.logits = torch.empty((N, V), dtype=torch.float32, device=dev)
        self.am_logp = torch.zeros((N, V), dtype=torch.float32, device=dev)
        self.energy = torch.empty((2, N, TM), dtype=torch.float32, device=dev)   # [part][row][t]
        self.att_sync = torch.zeros(B * ((Kb + 1) // 2), dtype=torch.int32, device=dev)
        self.enc = torch.empty((B, TM, C_), dtype=torch.float32, device=dev)
        self.keys = torch.empty((B, d.att, TM), dtype=torch.float32, device=dev)   # E_K^T
        self.slots0 = torch.arange(B, dtype=torch.int32, device=dev) * Kb
        self.fus_buf = None
        self.lm = None
        self.sub = None
        if self.has_fusion and hasattr(fusion, "char_lm"):
            # SubwordFusion over the device token LM: the selection reads the
            # fp32 logits and an fp64 normaliser per slot (rows never built)
            sw = fusion.char_lm.weights
            sd = sw.d
            self.sub = sw
            self.sub_X2 = [SubLmState(sd.layers, N, sd.hidden, dev),
                           SubLmState(sd.layers, N, sd.hidden, dev)]
            self.sub_scratch = split_scratch(N, sw.k_max, dev)
            self.fus_buf = torch.zeros((N, V), dtype=torch.float32, device=dev)
            self.sub_norm = torch.zeros(N, dtype=torch.float64, device=dev)
            self.buf.set_fusion_logits(self.sub_norm, fusion.char_lm.score_floor)
            self.views = [_view_with_rows(self.buf, p, self.rows[1 - p], self.count[1 - p])
                          for p in range(2)]
        elif self.has_fusion:
            self.lm = _LmPool(fusion.word_lm.weights, N, dev)
            self.fus_buf = torch.zeros((N + 1, V), dtype=torch.float64, device=dev)
        self.graphs = None
        self.graphs_tail = None
        self.per_step_launches = 0.0
        self.side_stream = torch.cuda.Stream(device=dev)
        # look-ahead floored-score count of the running decode (credited to the
        # caller's fusion.diagnostics afterwards; the graphs capture this buffer)
        self.floored = torch.zeros(1, dtype=torch.int64, device=dev)

    def reset(self, T: Sequence[int], max_len: Sequence[int]) -> None:
        """Per-decode initial state (decoder.py:350-361): one live row per
        utterance, zero decoder state, root trie state, <s> word history.
        A batch smaller than the session leaves its surplus utterances
        inactive from the start (like utterances that already finished)."""
        buf = self.buf
        stream = _lib.stream_ptr()
        Bn = len(T)
        ml = torch.ones(self.B, dtype=torch.int32)
        te = torch.ones(self.B, dtype=torch.int32)
        ml[:Bn] = torch.as_tensor(list(max_len), dtype=torch.int32)
        te[:Bn] = torch.as_tensor(list(T), dtype=torch.int32)
        buf.max_len.copy_(ml, non_blocking=True)
        buf.t_enc.copy_(te, non_blocking=True)
        _lib.call("fb_search_init", self.cfg_ref, C.byref(buf.view(0)), self.B, stream)
        if Bn < self.B:
            buf.active[Bn:].zero_()
            buf.n_live[Bn:].zero_()
        buf.acc[0].zero_()
        prev = self.X2[1]
        prev.h.zero_()
        prev.c.zero_()
        prev.ctx.zero_()
        self.rows[0][:Bn] = self.slots0[:Bn]
        self.count[0].fill_(Bn)
        self.floored.zero_()
        if self.sub is not None:
            self.sub_X2[1].h.zero_()
            self.sub_X2[1].c.zero_()
        if self.lm is not None:
            lm = self.lm
            lm.trie[0].zero_()
            lm.hist[0].zero_()
            lm.start()

    def fits(self, B: int, TM: int, MT: int) -> bool:
        return self.B >= B and self.TM >= TM and self.MT >= MT


class FusedDecoder:
    def __init__(self, scorer, fusion, config: DecodeConfig, token_dict):
        d = scorer.weights.d
        if len(token_dict) != d.vocab:
            raise ConfigError(f"acoustic model scores {d.vocab} tokens but the dictionary"
                              f" has {len(token_dict)}")
        self.scorer, self.fusion, self.config, self.token_dict = scorer, fusion, config, token_dict
        self.spec_counts: Optional[torch.Tensor] = None
        self.steps_run = 0
        self.kernel_launches = 0
        self.prune_spec = True      # exact pruning of speculative <eos> LM events
        self.select_flags = 0       # tests: bit 0 two-stage, bit 1 radix top-K (any size)
        self.use_graphs = True      # one CUDA graph per step parity, replayed
        # host polls the live-row count every k steps (dev override FB_POLL)
        self.poll_every = int(os.environ.get("FB_POLL", "8"))
        self._sessions: List[_Session] = []       # most recently used last

    def _session(self, B: int, TM: int, MT: int, caps=None) -> _Session:
        """A session that holds the batch: with a corpus hint (caps = batch
        size, encoder frames of the corpus) any session within the caps, else
        one no more than about twice the batch; otherwise a new one sized to
        the caps (or the batch), evicting the least recently used beyond two."""
        if caps is not None:
            lim_b, lim_t = max(caps[0], B), max(caps[1], TM)
        else:
            lim_b, lim_t = 2 * B + 64, 2 * TM + 64
        for s in reversed(self._sessions):
            if s.fits(B, TM, MT) and s.B <= lim_b and s.TM <= lim_t:
                self._sessions.remove(s)
                self._sessions.append(s)
                return s
        Bc, TMc = (lim_b, lim_t) if caps is not None else (B, TM)
        MTc = max(MT, max(1, int(math.floor(self.config.max_len_ratio * TMc))) + 1)
        while len(self._sessions) >= 2:
            self._sessions.pop(0)       # release before allocating the new one
        s = _Session(self, Bc, TMc, MTc)
        self._sessions.append(s)
        return s

    def _step(self, S: _Session, c: int, tm, counts) -> None:
        """One lock-step decode step on parity c, in order (eager / instrumented)."""
        self._am(S, c, tm)
        self._body(S, c, tm, counts)
        self._tail(S, c, tm, counts)

    def _step_overlapped(self, S: _Session, c: int, prev_tail: bool) -> None:
        """Graph-captured step: step t's word-boundary tail (trie advance, late
        LM events, g rows -- only read by step t+1's look-ahead) runs on a side
        stream concurrently with step t+1's acoustic step, then joins."""
        if prev_tail and S.lm is not None:
            main = torch.cuda.current_stream()
            side = S.side_stream
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self._tail(S, 1 - c, _NoTimer(), None)
                self._lookahead(S, c, _NoTimer())     # needs the tail, not the AM step
                if _SPEC_EARLY:
                    # every speculative </s> event of the step (no pruning by the
                    # acoustic scores) beside the acoustic step instead of after it
                    self._spec(S, c, _NoTimer(), None, prune=False, pack_stream=None)
            self._am(S, c, _NoTimer())
            main.wait_stream(side)
            self._body(S, c, _NoTimer(), None, lookahead=False, spec=not _SPEC_EARLY)
        else:
            self._am(S, c, _NoTimer())
            self._body(S, c, _NoTimer(), None)

    def _am(self, S: _Session, c: int, tm) -> None:
        """Acoustic step (+ token LM for SubwordFusion) of parity c."""
        scorer, fusion = self.scorer, self.fusion
        buf, N, B = S.buf, S.N, S.B
        rc, nc = S.rows[c], S.count[c]
        with tm("am_step"):
            scorer.step_fn(N=N, rows=rc, m=N, m_dev=nc, parent=buf.parent,
                           last_tok=buf.last_tok, prev=S.X2[1 - c], cur=S.X2[c],
                           scratch=S.scratch, q=S.q, logits=S.logits, am_logp=S.am_logp,
                           cfg_ref=S.cfg_ref, num_utts=B, active=buf.active,
                           n_live=buf.n_live, t_enc=buf.t_enc, keys=S.keys, enc=S.enc,
                           acc_in=buf.acc[c], acc_out=buf.acc[1 - c], cov=buf.cov,
                           energy=S.energy, sync=S.att_sync,
                           timer=None if isinstance(tm, _NoTimer) else tm,
                           abufs=S.am_abufs, pack_stream=S.pack_stream,
                           row_pos=buf.row_pos if AM_CTX_PLANES else None)
        fus_buf = S.fus_buf
        if S.sub is not None:
            with tm("lm_subword"):
                subword_step(S.sub, m=N, m_dev=nc, rows=rc, parent=buf.parent,
                             last_tok=buf.last_tok, eos_id=fusion.char_lm.eos_id,
                             pad_id=fusion.char_lm.pad_id, prev=S.sub_X2[1 - c],
                             cur=S.sub_X2[c], scratch=S.sub_scratch, logits=fus_buf,
                             norm=S.sub_norm)

    def _lookahead(self, S: _Session, c: int, tm) -> None:
        """Eq. 4 rows of parity c (needs the previous step's tail only)."""
        if S.lm is None:
            return
        fusion, lm = self.fusion, S.lm
        rc, nc = S.rows[c], S.count[c]
        with tm("lookahead"):
            # word_end in the eos column of final rows; log P(</s>) added later
            _lib.call("fb_lookahead_scores", fusion.dtrie.ref, S.N, P(nc), P(rc), P(lm.trie[c]),
                      P(lm.hist[c]), P(lm.g), lm.lw.d.words, P(lm.eos), P(lm.zero_eos),
                      fusion.space_id, fusion.eos_id, fusion.oov_penalty, fusion.score_floor,
                      P(S.fus_buf), S.V, P(S.floored), _lib.stream_ptr())

    def _body(self, S: _Session, c: int, tm, counts, lookahead: bool = True,
              spec: bool = True) -> None:
        """Look-ahead, speculative <eos> LM events and selection of parity c."""
        fusion = self.fusion
        buf, N, V, B = S.buf, S.N, S.V, S.B
        stream = _lib.stream_ptr()              # the capture stream inside a graph
        fus_buf = S.fus_buf
        if S.lm is not None:
            lm = S.lm
            if lookahead:
                self._lookahead(S, c, tm)
            if spec:
                self._spec(S, c, tm, counts, prune=self.prune_spec, pack_stream=S.pack_stream)
        with tm("select"):
            _lib.call("fb_search_step", S.cfg_ref, C.byref(S.views[c]), B, P(S.am_logp), V,
                      P(fus_buf), V, stream)

    def _spec(self, S: _Session, c: int, tm, counts, prune: bool, pack_stream) -> None:
        """Speculative <eos> LM events of parity c's final-state rows and their
        log P(</s>) (fusion.py:181-183); pruned exactly against the acoustic
        scores when `prune` (then after the acoustic step)."""
        fusion = self.fusion
        N, V, B = S.N, S.V, S.B
        rc, nc = S.rows[c], S.count[c]
        stream = _lib.stream_ptr()
        fus_buf = S.fus_buf
        if True:
            lm, dtrie = S.lm, fusion.dtrie
            lw = lm.lw
            Vw = lw.d.words
            with tm("lm_spec"):
                if prune:
                    _lib.call("fb_spec_select", S.cfg_ref, C.byref(S.views[c]), B, dtrie.ref,
                              P(lm.trie[c]), P(lm.hist[c]), P(S.am_logp), V, P(fus_buf), V,
                              P(lm.ev_row), P(lm.ev_rank), P(lm.ev_slot), P(lm.ev_count),
                              P(lm.row_ev), None, stream)
                else:
                    _lib.call("fb_spec_events", dtrie.ref, N, P(nc), P(rc), P(lm.trie[c]),
                              P(lm.hist[c]), P(lm.ev_row), P(lm.ev_rank), P(lm.ev_slot),
                              P(lm.ev_count), P(lm.row_ev), stream)
                lm_step(lw, m=N, m_dev=lm.ev_count, state_src=lm.state, src_idx=lm.ev_slot,
                        state_dst=lm.ev_state, ranks=lm.ev_rank, tok_default=0,
                        scratch=lm.scratch, logits=lm.ev_logits, timer=tm, stats=lm.ev_stats,
                        splitk=lm.splitk, abufs=lm.abufs, pack_stream=pack_stream)
            with tm("lm_eos"):
                # log P(</s>) per event, also added into the fusion rows' <eos>
                # column in the same launch (fb_eos_fixup fused)
                K.stats_to_g(lm.ev_logits, lm.ev_stats, Vw, lw.v_out, m=N, m_dev=lm.ev_count,
                             slots=lm.ev_row, eos_out=lm.ext_eos,
                             stat_out=lm.ev_stat if _STAT_REUSE else None,
                             fus=fus_buf, fus_eos=fusion.eos_id)
            if counts is not None:
                counts.append(lm.ev_count.clone())

    def _tail(self, S: _Session, c: int, tm, counts) -> None:
        """Word-boundary bookkeeping after the selection of parity c."""
        fusion = self.fusion
        buf, N = S.buf, S.N
        rc, nc = S.rows[c], S.count[c]
        stream = _lib.stream_ptr()
        if S.lm is not None:
            lm, dtrie = S.lm, fusion.dtrie
            lw = lm.lw
            Vw = lw.d.words
            rn, cn = S.rows[1 - c], S.count[1 - c]
            with tm("advance"):
                _lib.call("fb_trie_advance", dtrie.ref, N, P(cn), P(rn), P(buf.parent),
                          P(lm.trie[c]), P(lm.hist[c]), P(buf.last_tok), fusion.space_id,
                          fusion.eos_id, fusion.pad_id, P(lm.trie[1 - c]), P(lm.hist[1 - c]),
                          P(lm.brank), stream)
                _lib.call("fb_boundary_plan", N, P(cn), P(rn), P(buf.parent), P(lm.brank),
                          P(lm.row_ev), P(rc), P(nc), P(lm.hist[c]), P(lm.hist[1 - c]),
                          lm.P, P(lm.mark), P(lm.bnd_slot), P(lm.bnd_src), P(lm.bnd_count),
                          P(lm.unk_slot), P(lm.unk_tok), P(lm.late_row), P(lm.late_dst),
                          P(lm.unk_count), N, stream)
            with tm("lm_late"):
                # boundary rows without a speculative event: (h, rank) or (h, <unk>)
                lm_step(lw, m=N, m_dev=lm.unk_count, state_src=lm.state, src_idx=lm.unk_slot,
                        state_dst=lm.ev_state[N:], ranks=lm.unk_tok, tok_default=lw.unk_tok,
                        scratch=lm.scratch, logits=lm.ev_logits[N:], timer=tm,
                        stats=lm.ev_stats[N:], splitk=lm.splitk, abufs=lm.abufs)
            with tm("g_build"):
                K.copy_rows(lm.ev_state, lm.state, m=N, m_dev=lm.bnd_count, src_idx=lm.bnd_src,
                            dst_idx=lm.bnd_slot)
                K.stats_to_g(lm.ev_logits, lm.ev_stats, Vw, lw.v_out, m=N, m_dev=lm.bnd_count,
                             src_rows=lm.bnd_src, slots=lm.bnd_slot, g_pool=lm.g,
                             eos_out=lm.eos, seg_ws=lm.seg_ws,
                             stat_in=lm.ev_stat if _STAT_REUSE else None)
                K.copy_rows(lm.ev_state[N:], lm.state, m=N, m_dev=lm.unk_count,
                            dst_idx=lm.late_dst)
                K.stats_to_g(lm.ev_logits[N:], lm.ev_stats[N:], Vw, lw.v_out, m=N,
                             m_dev=lm.unk_count, slots=lm.late_dst, g_pool=lm.g,
                             eos_out=lm.eos, seg_ws=lm.seg_ws)
            if counts is not None:
                counts.append(lm.bnd_count.clone())
                counts.append(lm.unk_count.clone())

    def run(self, X: torch.Tensor, T: Sequence[int], utt_ids: Sequence[str], timer=None,
            record_counts: bool = False, fusion=None, caps=None) -> List[DecodeResult]:
        """Decode one staged batch.  fusion: the caller's fusion instance (its
        diagnostics are credited); caps: corpus hint (see corpus_hint)."""
        config = self.config
        tm = timer if timer is not None else _NoTimer()
        lib = _lib.lib()
        l0 = lib.fb_launch_count()
        B = len(T)
        if B == 0:
            return []
        Tenc = list(T)
        TM = max(Tenc)
        max_len = [max(1, int(math.floor(config.max_len_ratio * t))) for t in Tenc]
        MT = max(max_len) + 1
        S = self._session(B, TM, MT, caps)
        with tm("encoder"):
            _, _, Tenc = self.scorer.encoder(X, Tenc, out=(S.enc, S.keys))
        S.reset(Tenc, max_len)
        counts = [] if record_counts else None
        parity = 0
        steps = 0
        replayed = 0
        if self.use_graphs and timer is None and counts is None:
            if S.graphs is None:
                # first step (no previous tail) + one graph per parity whose
                # previous step's tail overlaps this step's acoustic step
                g = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
                c0 = lib.fb_launch_count()
                with torch.cuda.graph(g[2]):
                    self._step_overlapped(S, 0, prev_tail=False)
                c1 = lib.fb_launch_count()
                for p_ in (0, 1):
                    with torch.cuda.graph(g[p_]):
                        self._step_overlapped(S, p_, prev_tail=True)
                S.per_step_launches = (lib.fb_launch_count() - c1) / 2.0
                l0 += lib.fb_launch_count() - c0          # captures launch nothing
                S.graphs = g
                if _TAIL_ROWS > 0:
                    c2 = lib.fb_launch_count()
                    _lib.call("fb_set_attention_tiling", *_TAIL_TILING)
                    sk_main = S.lm.splitk if S.lm is not None else None
                    if S.lm is not None and S.lm.splitk_tail is not None:
                        S.lm.splitk = S.lm.splitk_tail
                    try:
                        gt = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
                        for p_ in (0, 1):
                            with torch.cuda.graph(gt[p_]):
                                self._step_overlapped(S, p_, prev_tail=True)
                    finally:
                        _lib.call("fb_set_attention_tiling", 0, 0, 0)
                        if S.lm is not None:
                            S.lm.splitk = sk_main
                    l0 += lib.fb_launch_count() - c2
                    S.graphs_tail = gt
            first = True
            live = S.N
            while True:
                tail = _TAIL_ROWS > 0 and live < _TAIL_ROWS
                for _ in range(self.poll_every):
                    if first:
                        S.graphs[2].replay()
                    elif tail:
                        S.graphs_tail[parity].replay()
                    else:
                        S.graphs[parity].replay()
                    first = False
                    parity ^= 1
                    steps += 1
                    replayed += 1
                live = int(S.count[parity].item())
                if live == 0:
                    break
        else:
            while True:
                self._step(S, parity, tm, counts)
                parity ^= 1
                steps += 1
                if int(S.count[parity].item()) == 0:
                    break
        self.steps_run = steps
        # kernels this run put on the GPU (graph replays included)
        self.kernel_launches = int(lib.fb_launch_count() - l0 + S.per_step_launches * replayed)
        if counts is not None:
            self.spec_counts = torch.cat(counts).view(steps, 3).cpu() if counts else None
        target = fusion if fusion is not None else self.fusion
        if S.lm is not None and target is not None and hasattr(target, "_floored"):
            target._floored += S.floored
        return S.buf.results(list(utt_ids), Tenc)


def _view_with_rows(buf: SearchBuffers, p: int, next_rows, next_count):
    out = _lib.FbSearchState.from_buffer_copy(buf.view(p))
    out.next_rows = P(next_rows)
    out.next_count = P(next_count)
    return out
