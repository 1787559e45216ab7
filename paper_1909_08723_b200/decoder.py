"""Batched beam search with fusion, coverage and the EOS gate -- on the GPU.

Keeps the reference API (``decoder.py:64-128, 312-319, 339-504``):
``DecodeConfig``, ``DecodeResult``, ``AcousticScorer``, ``decode_batch`` and
``decode_corpus`` with the same arguments, validation errors and result order.

Two drivers sit behind ``decode_batch``:

* the fused engine (``engine.py``) when the scorer is a device scorer
  (``models.AttnLstmScorer``) and the fusion is ``None`` or a device-native
  ``LookaheadFusion`` (LSTM word LM on the GPU): the whole lock-step loop runs on
  the device, one CUDA-graph replay per step;
* the plugin driver below for any other ``AcousticScorer`` / word LM (e.g. the
  reference's trace tables or n-gram LMs): host scorers hand over their rows
  each step, but score combination, the EOS gate, top-beam selection,
  coverage, the finished set, early stop and the result pick all run in the
  ``fb_search_step`` kernel, and fusion runs in the look-ahead kernels.
"""

from __future__ import annotations

import os

import ctypes as C
import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, FormatError
from .kaldi_io import FeatureMatrix
from .fusion import _device


@dataclass
class DecodeConfig:
    beam_size: int = 50
    lm_weight: float = 0.9
    coverage_mode: str = "off"            # off | original | improved
    coverage_weight: float = 0.01
    tau1: float = 0.5
    tau2: float = 1.0
    cov_margin: float = 0.7
    eos_gamma: Optional[float] = None     # None = gate off
    max_len_ratio: float = 1.0

    def validate(self) -> None:
        if self.beam_size < 1:
            raise ConfigError(f"beam size must be positive, got {self.beam_size}")
        if self.lm_weight < 0:
            raise ConfigError(f"LM weight must be >= 0, got {self.lm_weight}")
        if self.coverage_mode not in ("off", "original", "improved"):
            raise ConfigError(f"unknown coverage mode {self.coverage_mode!r}")
        if self.coverage_weight < 0:
            raise ConfigError("coverage weight must be >= 0")
        if self.coverage_mode == "original" and self.tau1 <= 0:
            raise ConfigError("original coverage requires tau1 > 0")
        if self.coverage_mode == "improved":
            if not self.tau2 > self.tau1 > 0:
                raise ConfigError(f"improved coverage requires tau2 > tau1 > 0,"
                                  f" got tau1={self.tau1} tau2={self.tau2}")
            if self.cov_margin <= 0:
                raise ConfigError("improved coverage requires cov_margin > 0")
        if self.eos_gamma is not None and self.eos_gamma < 0:
            raise ConfigError("eos gamma must be >= 0 (or off)")
        if self.max_len_ratio <= 0:
            raise ConfigError("max length ratio must be positive")

    def coverage(self, attn_accum) -> float:
        if self.coverage_mode == "original":
            return coverage_original(attn_accum, self.tau1)
        if self.coverage_mode == "improved":
            return coverage_improved(attn_accum, self.tau1, self.tau2, self.cov_margin)
        return 0.0

    @property
    def cov_code(self) -> int:
        return {"off": 0, "original": 1, "improved": 2}[self.coverage_mode]


@dataclass
class DecodeResult:
    utt_id: str
    tokens: List[int]           # best hypothesis, trailing <eos> stripped
    score: float
    attn_accum: np.ndarray
    finished: bool
    steps: int


class AcousticScorer:
    """Contract of the acoustic side (reference decoder.py:109-128)."""

    def init(self, features: FeatureMatrix):
        raise NotImplementedError

    def enc_length(self, state) -> int:
        raise NotImplementedError

    def step(self, state, last_tokens: Sequence[int]):
        raise NotImplementedError

    def reorder(self, state, parent_indices: Sequence[int]):
        raise NotImplementedError


# ---- coverage / gate as single-row device evaluations ------------------------
def _one_row_coverage(acc, mode: int, tau1: float, tau2: float, margin: float) -> float:
    dev = _device()
    a = torch.as_tensor(np.asarray(acc, np.float64).reshape(1, -1), device=dev)
    T = a.shape[1]
    cfg = _lib.FbSearchCfg(beam=1, vocab=1, cov_mode=mode, t_max=max(T, 1), tau1=tau1,
                           tau2=tau2, cov_margin=margin)
    z = torch.zeros_like(a)
    out = torch.empty_like(a)
    cov = torch.zeros(1, dtype=torch.float64, device=dev)
    te = torch.full((1,), T, dtype=torch.int32, device=dev)
    _lib.call("fb_attend_coverage", C.byref(cfg), 1, None, None, None, _lib.ptr(te),
              _lib.ptr(z), _lib.ptr(a), 0, max(T, 1), _lib.ptr(out), _lib.ptr(cov),
              _lib.stream_ptr())
    return float(cov.item())


def coverage_original(attn_accum, tau1: float) -> float:
    """Eq. 5: frames whose accumulated attention exceeds tau1 (decoder.py:36-38)."""
    return _one_row_coverage(attn_accum, 1, tau1, 0.0, 0.0)


def coverage_improved(attn_accum, tau1: float, tau2: float, cov_margin: float) -> float:
    """Eq. 6: count above tau1 minus (c + acc - tau2) above tau2 (decoder.py:41-48)."""
    return _one_row_coverage(attn_accum, 2, tau1, tau2, cov_margin)


def eos_allowed(log_probs_row, gamma: Optional[float], eos_id: int) -> bool:
    """Eq. 7: log P(eos) > gamma * max_t log P(t); None disables the gate."""
    if gamma is None:
        return True
    row = torch.as_tensor(np.asarray(log_probs_row), device=_device())
    return bool((row[eos_id] > gamma * row.max()).item())


# ---- device search state -----------------------------------------------------
class SearchBuffers:
    """Per-batch search state in HBM (slot layout: utterance u owns rows
    u*beam .. u*beam+beam-1).  ``in``/``out`` pairs ping-pong by step parity."""

    def __init__(self, B: int, K: int, max_tokens: int, t_max: int, device, vocab: int = 0,
                 select_flags: int = 0):
        z = lambda *s, dt=torch.int32: torch.zeros(s, dtype=dt, device=device)  # noqa: E731
        f64 = torch.float64
        N = B * K
        self.B, self.K, self.MT, self.TM = B, K, max_tokens, t_max
        self.active, self.n_live, self.steps = z(B), z(B), z(B)
        self.max_len, self.t_enc = z(B), z(B)
        self.base = [z(N, dt=f64), z(N, dt=f64)]
        self.total = [z(N, dt=f64), z(N, dt=f64)]
        self.tok = [z(N, max_tokens), z(N, max_tokens)]
        self.acc = [z(N, t_max, dt=f64), z(N, t_max, dt=f64)]
        self.cov = z(N, dt=f64)
        self.parent, self.last_tok = z(N), z(N)
        self.fin_valid, self.fin_len = z(B, 2 * K), z(B, 2 * K)
        self.fin_total = z(B, 2 * K, dt=f64)
        self.fin_tokens = z(B, 2 * K, max_tokens)
        self.fin_acc = z(B, 2 * K, t_max, dt=f64)
        self.res_len, self.res_finished, self.res_steps = z(B), z(B), z(B)
        self.res_score = z(B, dt=f64)
        self.res_tokens = z(B, max_tokens)
        self.res_acc = z(B, t_max, dt=f64)
        self.next_rows, self.next_count = z(N), z(1)
        self.row_pos = z(N)            # slot -> position in next_rows
        # the last selection CTA builds the next row list (FB_SELECT_COMPACT=0:
        # separate compaction launch, dev A/B)
        self.select_arrive = z(1) if os.environ.get("FB_SELECT_COMPACT", "1") == "1" else None
        # exact two-stage selection for beam x vocab beyond one CTA's shared memory
        # (select_flags: test knobs, bit 0 force two-stage, bit 1 force radix top-K)
        self.two_stage = bool(select_flags & 1) or \
            13 * K * vocab + 16 * K + 24 * K + 4 * (4 * K + 64) + 16 > 220 * 1024
        self.cand_score = z(N, K, dt=f64) if self.two_stage else None
        self.cand_flat = z(N, K) if self.two_stage else None
        self.select_flags = int(select_flags)
        self.fus_norm = None           # set by the fused engine for token-LM logits
        self.fus_floor = 0.0
        self._views = [self._view(0), self._view(1)]

    def _view(self, p: int):
        q = 1 - p
        P = _lib.ptr
        return _lib.FbSearchState(
            P(self.active), P(self.n_live), P(self.steps), P(self.max_len), P(self.t_enc),
            P(self.base[p]), P(self.base[q]), P(self.total[p]), P(self.total[q]),
            P(self.tok[p]), P(self.tok[q]), P(self.parent), P(self.last_tok),
            P(self.acc[q]), P(self.cov),
            P(self.fin_valid), P(self.fin_total), P(self.fin_len), P(self.fin_tokens),
            P(self.fin_acc), P(self.res_len), P(self.res_score), P(self.res_finished),
            P(self.res_steps), P(self.res_tokens), P(self.res_acc),
            P(self.next_rows), P(self.next_count), P(self.cand_score), P(self.cand_flat),
            self.select_flags, 0, P(self.fus_norm), float(self.fus_floor), P(self.row_pos),
            P(self.select_arrive))

    def set_fusion_logits(self, norm: torch.Tensor, floor: float) -> None:
        """Fusion rows given as fp32 logits + this fp64 per-slot normaliser."""
        self.fus_norm, self.fus_floor = norm, floor
        self._views = [self._view(0), self._view(1)]

    def view(self, parity: int):
        return self._views[parity]

    def results(self, utt_ids: Sequence[str], t_enc: Sequence[int]) -> List[DecodeResult]:
        L = self.res_len.cpu().numpy()
        score = self.res_score.cpu().numpy()
        fin = self.res_finished.cpu().numpy()
        steps = self.res_steps.cpu().numpy()
        toks = self.res_tokens.cpu().numpy()
        acc = self.res_acc.cpu().numpy()
        out = []
        for u, uid in enumerate(utt_ids):
            if L[u] < 0:
                raise ConfigError(f"utterance {uid!r}: no hypotheses survived decoding")
            out.append(DecodeResult(uid, toks[u, :L[u]].tolist(), float(score[u]),
                                    acc[u, :t_enc[u]].copy(), bool(fin[u]), int(steps[u])))
        return out


def search_cfg(config: DecodeConfig, token_dict, has_fusion: bool, early_stop: bool,
               am_f32: bool, max_tokens: int, t_max: int) -> _lib.FbSearchCfg:
    g = config.eos_gamma
    return _lib.FbSearchCfg(
        beam=config.beam_size, vocab=len(token_dict), pad_id=token_dict.pad_id,
        eos_id=token_dict.eos_id, cov_mode=config.cov_code, gate_on=int(g is not None),
        early_stop=int(early_stop), has_fusion=int(has_fusion), am_f32=int(am_f32),
        max_tokens=max_tokens, t_max=t_max, pad0=0, lm_weight=float(config.lm_weight),
        cov_weight=float(config.coverage_weight), tau1=float(config.tau1),
        tau2=float(config.tau2), cov_margin=float(config.cov_margin),
        gamma=float(g) if g is not None else 0.0)


# ---- decode ------------------------------------------------------------------
def decode_batch(features: Sequence[FeatureMatrix], scorer: AcousticScorer, fusion,
                 config: DecodeConfig, token_dict) -> List[DecodeResult]:
    """Decodes a batch of utterances in lock step; results follow input order."""
    config.validate()
    for f in features:
        if np.asarray(f.data).size == 0:
            raise ConfigError(f"utterance {f.utt_id!r}: empty feature matrix")
    if getattr(scorer, "is_device_scorer", False) and (
            fusion is None or getattr(fusion, "device_native", False)):
        from .engine import decode_fused
        return decode_fused(features, scorer, fusion, config, token_dict)
    return _decode_plugins(features, scorer, fusion, config, token_dict)


_SELECT_FLAGS = 0       # tests: bit 0 two-stage selection, bit 1 radix top-K, at any size


def _decode_plugins(features, scorer, fusion, config: DecodeConfig, token_dict):
    dev = fusion.device if fusion is not None else _device()
    V = len(token_dict)
    K = config.beam_size
    states, t_enc, max_len = [], [], []
    for f in features:
        st = scorer.init(f)
        T = int(scorer.enc_length(st))
        states.append(st)
        t_enc.append(T)
        max_len.append(max(1, int(math.floor(config.max_len_ratio * T))))
    B = len(features)
    if B == 0:
        return []
    MT = max(max_len) + 1
    TM = max(t_enc)
    buf = SearchBuffers(B, K, MT, TM, dev, vocab=V, select_flags=_SELECT_FLAGS)
    buf.max_len.copy_(torch.as_tensor(max_len, dtype=torch.int32))
    buf.t_enc.copy_(torch.as_tensor(t_enc, dtype=torch.int32))
    early = fusion is None or bool(fusion.nonpositive_scores)
    fstate = fusion.start(B) if fusion is not None else None
    stream = _lib.stream_ptr()

    active = [True] * B
    n_live = [1] * B
    last = [[-1] for _ in range(B)]
    cfg = None
    am_buf = attn_buf = None
    fus_buf = torch.zeros((B * K, V), dtype=torch.float64, device=dev) if fusion else None
    parity = 0
    while any(active):
        act = [u for u in range(B) if active[u]]
        offs, pos = {}, 0
        slots = []
        for u in act:
            offs[u] = pos
            pos += n_live[u]
            slots.extend(range(u * K, u * K + n_live[u]))
        slots_t = torch.as_tensor(np.asarray(slots, np.int64), device=dev)
        if fusion is not None:
            dev_rows = getattr(fusion, "char_scores_device", None)
            rows = (dev_rows(fstate) if dev_rows is not None else
                    torch.as_tensor(np.asarray(fusion.char_scores(fstate), np.float64),
                                    device=dev))
            if tuple(rows.shape) != (pos, V):
                raise ConfigError(f"fusion scorer returned shape {tuple(rows.shape)},"
                                  f" expected ({pos}, {V})")
            fus_buf[slots_t] = rows
        ams, attns = [], []
        for u in act:
            am, attn, states[u] = scorer.step(states[u], last[u])
            am = np.asarray(am)
            if am.shape != (n_live[u], V):
                raise ConfigError(f"acoustic scorer returned shape {am.shape},"
                                  f" expected ({n_live[u]}, {V})")
            ams.append(am)
            attns.append(np.asarray(attn, np.float64))
        if cfg is None:
            f32 = ams[0].dtype == np.float32
            cfg = search_cfg(config, token_dict, fusion is not None, early, f32, MT, TM)
            cfg_ref = C.byref(cfg)
            am_buf = torch.zeros((B * K, V), dtype=torch.float32 if f32 else torch.float64,
                                 device=dev)
            attn_buf = torch.zeros((B * K, TM), dtype=torch.float64, device=dev)
            _lib.call("fb_search_init", cfg_ref, C.byref(buf.view(0)), B, stream)
        am_cat = np.concatenate(ams).astype(np.float32 if cfg.am_f32 else np.float64)
        am_buf[slots_t] = torch.as_tensor(am_cat, device=dev)
        for u, a in zip(act, attns):
            if a.shape != (n_live[u], t_enc[u]):
                raise ConfigError(f"acoustic scorer returned attention of shape {a.shape}")
            attn_buf[u * K:u * K + n_live[u], :t_enc[u]] = torch.as_tensor(a, device=dev)
        rows_i32 = slots_t.to(torch.int32)
        _lib.call("fb_attend_coverage", cfg_ref, len(slots), None, _lib.ptr(rows_i32),
                  _lib.ptr(buf.parent), _lib.ptr(buf.t_enc), _lib.ptr(buf.acc[parity]),
                  _lib.ptr(attn_buf), 0, TM, _lib.ptr(buf.acc[1 - parity]), _lib.ptr(buf.cov),
                  stream)
        _lib.call("fb_search_step", cfg_ref, C.byref(buf.view(parity)), B, _lib.ptr(am_buf),
                  V, _lib.ptr(fus_buf), V, stream)
        act_now = buf.active.cpu().numpy()
        nl = buf.n_live.cpu().numpy()
        par = buf.parent.cpu().numpy()
        chosen = buf.last_tok.cpu().numpy()
        flat_par, flat_tok = [], []
        for u in act:
            active[u] = bool(act_now[u])
            n_live[u] = int(nl[u])
            if not active[u]:
                continue
            loc = (par[u * K:u * K + n_live[u]] - u * K).tolist()
            last[u] = chosen[u * K:u * K + n_live[u]].tolist()
            states[u] = scorer.reorder(states[u], loc)
            if fusion is not None:
                flat_par.extend(offs[u] + p for p in loc)
                flat_tok.extend(last[u])
        if fusion is not None:
            fstate = fusion.reorder(fstate, flat_par)
            if flat_tok:
                fstate = fusion.advance(fstate, np.asarray(flat_tok, dtype=np.int64))
        parity ^= 1
    return buf.results([f.utt_id for f in features], t_enc)


def decode_corpus(features: Sequence[FeatureMatrix], scorer: AcousticScorer, fusion_factory,
                  config: DecodeConfig, token_dict, batch_size: int = 8,
                  workers: int = 1) -> List[DecodeResult]:
    """Chunks utterances into batches; output order always matches input order."""
    if batch_size < 1:
        raise ConfigError(f"batch size must be positive, got {batch_size}")
    if workers < 1:
        raise ConfigError(f"worker count must be positive, got {workers}")
    chunks = [features[i:i + batch_size] for i in range(0, len(features), batch_size)]
    hint = None
    if getattr(scorer, "is_device_scorer", False) and len(features):
        # one device session (buffers + step graphs) for every batch of the corpus
        from .engine import corpus_hint
        t_max = max(np.asarray(f.data).shape[0] for f in features) // scorer.dims.subsample
        hint = (min(batch_size, len(features)), max(1, t_max))

    def run(chunk):
        fus = fusion_factory() if fusion_factory is not None else None
        if hint is None:
            return decode_batch(chunk, scorer, fus, config, token_dict)
        with corpus_hint(*hint):
            return decode_batch(chunk, scorer, fus, config, token_dict)

    if workers == 1 or len(chunks) <= 1:
        parts = [run(c) for c in chunks]
    else:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            parts = list(ex.map(run, chunks))
    return [r for p in parts for r in p]
