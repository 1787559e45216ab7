"""Fusion scorers behind the reference plugin surface (``fusion.py:45-233``).

``LookaheadFusion`` keeps the reference constructor, the ``start /
char_scores / advance / reorder`` protocol and functional value semantics, but
its state lives on the GPU: per-row trie states and g-pool slot ids (int32),
and a pool of fp64 cumulative word-mass rows ``g`` shared by every row with the
same word history.  Eq. 4 is evaluated by ``fb_lookahead_scores`` (one warp per
row over the CSR trie), the trie transition by ``fb_trie_advance`` and new ``g``
rows by ``fb_cumsum_rows`` / ``fb_logits_to_g``.  Nothing falls back to numpy.

``SubwordFusion`` (``fusion.py:236-266``) is plain token-level LM fusion over
the ``CharLM`` protocol (``char_lm.py:23-33``): host providers' rows are stacked
and uploaded; the device token LSTM LM (``models.LstmSubwordLM``) makes it
device-native, and the fused engine then never materialises the rows.

Word LMs: any object with the reference ``WordLM`` protocol
(``word_lm.py:160-186``) works -- host distributions are uploaded once per
distinct history.  The device LSTM LM (``models.LstmWordLM``) writes its rows
on the device instead and is what the fused decode engine drives.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import ctypes as C
import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .lexicon_trie import PrefixTreeAutomaton

OOV_STATE = -2                 # a row whose current word left the lexicon
DEFAULT_OOV_PENALTY = -10.0
SCORE_FLOOR = -30.0
UNK_RANK = -1


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1909_08723_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def cumsum_distribution(dist) -> np.ndarray:
    """Running prefix sums of a word distribution (reference fusion.py:40-42),
    computed by the device scan kernel."""
    dev = _device()
    d = torch.as_tensor(np.asarray(dist, np.float64), device=dev).reshape(1, -1)
    g = torch.empty_like(d)
    slot = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("fb_cumsum_rows", 1, _lib.ptr(d), d.shape[1], d.shape[1], _lib.ptr(slot),
              _lib.ptr(g), d.shape[1], _lib.stream_ptr())
    return g[0].cpu().numpy()


class FusionScorer:
    """Common surface of the batched fusion scorers (reference fusion.py:45-62)."""

    nonpositive_scores = True

    def start(self, n: int):
        raise NotImplementedError

    def char_scores(self, state) -> np.ndarray:
        raise NotImplementedError

    def advance(self, state, tokens: Sequence[int]):
        raise NotImplementedError

    def reorder(self, state, parent_indices: Sequence[int]):
        raise NotImplementedError


class DeviceTrie:
    """CSR trie resident in HBM plus the ``fb_trie_t`` view the kernels take.
    ``DeviceTrie.of(trie, device)`` uploads once per (automaton, device): a
    fusion per batch (pipeline.py:148-149) shares the resident copy."""

    @staticmethod
    def of(trie: PrefixTreeAutomaton, device) -> "DeviceTrie":
        cache = trie.__dict__.setdefault("_device_tries", {})
        key = str(device)
        dt = cache.get(key)
        if dt is None:
            dt = cache[key] = DeviceTrie(trie, device)
        return dt

    def __init__(self, trie: PrefixTreeAutomaton, device):
        row_ptr, lab, kid, info = trie.csr()
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=device)  # noqa: E731
        self.row_ptr, self.label, self.child, self.info = t(row_ptr), t(lab), t(kid), t(info)
        self.view = _lib.FbTrie(_lib.ptr(self.row_ptr), _lib.ptr(self.label),
                                _lib.ptr(self.child), _lib.ptr(self.info), trie.num_states,
                                trie.num_words, trie.alphabet_size)
        self.ref = C.byref(self.view)
        self.num_words = trie.num_words
        self.is_final = trie.is_final
        self.word_index = trie.word_index


class GPool:
    """Growable pool of fp64 cumulative-mass rows on the device (allocated on
    first use: the fused engine keeps its own history pool)."""

    def __init__(self, vw: int, device, cap: int = 16):
        self.vw = vw
        self.device = device
        self.cap0 = cap
        self.rows = torch.empty((0, vw), dtype=torch.float64, device=device)
        self.used = 0

    def alloc(self, k: int) -> np.ndarray:
        need = self.used + k
        if need > self.rows.shape[0]:
            cap = max(need, 2 * self.rows.shape[0], self.cap0)
            grown = torch.empty((cap, self.vw), dtype=torch.float64, device=self.device)
            grown[:self.used] = self.rows[:self.used]
            self.rows = grown
        ids = np.arange(self.used, need, dtype=np.int32)
        self.used = need
        return ids


class LookaheadBatch:
    """Per-hypothesis state: trie position, word history, cumulative mass row."""

    def __init__(self, fusion: "LookaheadFusion", states: torch.Tensor, slots: torch.Tensor,
                 histories: list):
        self._fusion = fusion
        self.states_dev = states        # [n] int32 (>= 0 or OOV_STATE)
        self.slots_dev = slots          # [n] int32 g-pool row per hypothesis
        self.histories = histories

    def __len__(self) -> int:
        return len(self.histories)

    @property
    def trie_states(self) -> np.ndarray:
        return self.states_dev.cpu().numpy().astype(np.int64)

    @property
    def g(self) -> np.ndarray:
        pool = self._fusion._pool.rows
        return pool[self.slots_dev.long()].cpu().numpy()


_CONVERTED: Dict[int, tuple] = {}


def _converted(trie) -> PrefixTreeAutomaton:
    """A reference automaton object converted once (kept alive with its source,
    so a fusion per batch over the same automaton shares one device copy)."""
    hit = _CONVERTED.get(id(trie))
    if hit is None or hit[0] is not trie:
        hit = _CONVERTED[id(trie)] = (trie, PrefixTreeAutomaton.from_reference(trie))
    return hit[1]


def _hkey(h):
    try:
        hash(h)
        return ("h", h)
    except TypeError:
        return ("id", id(h))


class LookaheadFusion(FusionScorer):
    """Word-LM look-ahead over the prefix-tree automaton (Eq. 4), on the GPU."""

    def __init__(self, trie, word_lm, token_dict, oov_penalty: float = DEFAULT_OOV_PENALTY,
                 score_floor: float = SCORE_FLOOR, device=None):
        if word_lm.vocab_size != trie.num_words:
            raise ConfigError(f"word LM vocabulary ({word_lm.vocab_size}) does not match"
                              f" the automaton ({trie.num_words} words)")
        if trie.alphabet_size != len(token_dict):
            raise ConfigError(f"automaton alphabet ({trie.alphabet_size}) does not match"
                              f" the token dictionary ({len(token_dict)})")
        if not isinstance(trie, PrefixTreeAutomaton):
            trie = _converted(trie)
        self.trie = trie
        self.word_lm = word_lm
        self.oov_penalty = float(oov_penalty)
        self.score_floor = float(score_floor)
        self.space_id, self.eos_id, self.pad_id = (token_dict.space_id, token_dict.eos_id,
                                                   token_dict.pad_id)
        self.dict_size = len(token_dict)
        self.device = _device(device)
        self.dtrie = DeviceTrie.of(trie, self.device)
        self._pool = GPool(trie.num_words, self.device)
        self._slot_of: Dict[tuple, int] = {}
        self._eos_of: Dict[tuple, float] = {}
        self._floored = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._final = trie.is_final
        self._rank = trie.word_index

    @property
    def diagnostics(self) -> dict:
        return {"floored_scores": int(self._floored.item())}

    @property
    def device_native(self) -> bool:
        return bool(getattr(self.word_lm, "is_device_lm", False))

    # ---- history -> g-pool slot ------------------------------------------------
    def _slots_for(self, hists: list) -> List[int]:
        out: List[Optional[int]] = []
        todo: Dict[tuple, object] = {}
        for h in hists:
            k = _hkey(h)
            s = self._slot_of.get(k)
            if s is None and k not in todo:
                todo[k] = h
            out.append(s)
        if todo:
            keys = list(todo)
            ids = self._pool.alloc(len(keys))
            writer = getattr(self.word_lm, "write_g_rows", None)
            slots_t = torch.as_tensor(ids, device=self.device)
            if writer is not None:
                writer([todo[k] for k in keys], self._pool.rows, slots_t)
            else:
                dists = np.stack([np.asarray(self.word_lm.full_distribution(todo[k]), np.float64)
                                  for k in keys])
                dd = torch.as_tensor(dists, device=self.device)
                _lib.call("fb_cumsum_rows", len(keys), _lib.ptr(dd), dd.shape[1], dd.shape[1],
                          _lib.ptr(slots_t), _lib.ptr(self._pool.rows), self._pool.vw,
                          _lib.stream_ptr())
            for k, s in zip(keys, ids):
                self._slot_of[k] = int(s)
        return [self._slot_of[_hkey(h)] for h in hists]

    def _eos(self, h) -> float:
        k = _hkey(h)
        v = self._eos_of.get(k)
        if v is None:
            v = float(self.word_lm.eos_log_prob(h))
            self._eos_of[k] = v
        return v

    # ---- protocol ------------------------------------------------------------
    def start(self, n: int) -> LookaheadBatch:
        h0 = self.word_lm.start_history()
        s0 = self._slots_for([h0])[0]
        return LookaheadBatch(self, torch.zeros(n, dtype=torch.int32, device=self.device),
                              torch.full((n,), s0, dtype=torch.int32, device=self.device),
                              [h0] * n)

    def char_scores_device(self, state: LookaheadBatch, out: Optional[torch.Tensor] = None
                           ) -> torch.Tensor:
        n = len(state)
        if out is None:
            out = torch.empty((n, self.dict_size), dtype=torch.float64, device=self.device)
        if n == 0:
            return out
        # LM end-of-sentence terms (fusion.py:175-184): root -> eos(h),
        # final state -> eos(extend(h, rank)); evaluated by the word LM.
        states = state.states_dev.cpu().numpy()
        ext = np.zeros(n, np.float64)
        for b in np.nonzero(states >= 0)[0]:
            st = int(states[b])
            if st == 0:
                ext[b] = self._eos(state.histories[b])
            elif self._final[st]:
                ext[b] = self._eos(self.word_lm.extend_history(state.histories[b],
                                                               int(self._rank[st])))
        ext_t = torch.as_tensor(ext, device=self.device)
        _lib.call("fb_lookahead_scores", self.dtrie.ref, n, None, None,
                  _lib.ptr(state.states_dev), _lib.ptr(state.slots_dev),
                  _lib.ptr(self._pool.rows), self._pool.vw, None, _lib.ptr(ext_t),
                  self.space_id, self.eos_id, self.oov_penalty, self.score_floor,
                  _lib.ptr(out), out.stride(0), _lib.ptr(self._floored), _lib.stream_ptr())
        return out

    def char_scores(self, state: LookaheadBatch) -> np.ndarray:
        return self.char_scores_device(state).cpu().numpy()

    def advance(self, state: LookaheadBatch, tokens: Sequence[int]) -> LookaheadBatch:
        tok = np.asarray(tokens, dtype=np.int64)
        n = len(state)
        if tok.shape != (n,):
            raise ValueError("one chosen token per hypothesis row required")
        if n == 0:
            return LookaheadBatch(self, state.states_dev.clone(), state.slots_dev.clone(), [])
        tok_d = torch.as_tensor(tok.astype(np.int32), device=self.device)
        s_out = torch.empty_like(state.states_dev)
        h_out = torch.empty_like(state.slots_dev)
        brank = torch.empty_like(state.states_dev)
        _lib.call("fb_trie_advance", self.dtrie.ref, n, None, None, None,
                  _lib.ptr(state.states_dev), _lib.ptr(state.slots_dev), _lib.ptr(tok_d),
                  self.space_id, self.eos_id, self.pad_id, _lib.ptr(s_out), _lib.ptr(h_out),
                  _lib.ptr(brank), _lib.stream_ptr())
        hist = list(state.histories)
        br = brank.cpu().numpy()
        rows = np.nonzero(br != -2)[0]
        if rows.size:
            for b in rows:
                hist[b] = self.word_lm.extend_history(hist[b], int(br[b]))
            slots = self._slots_for([hist[b] for b in rows])
            h_out[torch.as_tensor(rows, device=self.device)] = torch.as_tensor(
                np.asarray(slots, np.int32), device=self.device)
        return LookaheadBatch(self, s_out, h_out, hist)

    def reorder(self, state: LookaheadBatch, parent_indices: Sequence[int]) -> LookaheadBatch:
        idx_np = np.asarray(parent_indices, dtype=np.int64)
        idx = torch.as_tensor(idx_np, device=self.device)
        return LookaheadBatch(self, state.states_dev[idx], state.slots_dev[idx],
                              [state.histories[i] for i in idx_np])


# ---- plain token-level LM fusion (fusion.py:236-266) -------------------------------
class SubwordBatch:
    """Per-row provider states (reference ``SubwordBatch`` fusion.py:236-241)."""

    def __init__(self, char_states: list):
        self.char_states = char_states

    def __len__(self) -> int:
        return len(self.char_states)


class SubwordFusion(FusionScorer):
    """The character/subword provider's rows, unchanged (fusion.py:244-266).
    ``nonpositive_scores`` stays True (rows are log-probabilities)."""

    def __init__(self, char_lm, device=None):
        self.char_lm = char_lm
        self.diagnostics: dict = {}
        self.device = _device(device)

    @property
    def device_native(self) -> bool:
        return bool(getattr(self.char_lm, "is_device_lm", False))

    def start(self, n: int) -> SubwordBatch:
        s0 = self.char_lm.start()
        return SubwordBatch([s0] * n)

    def char_scores_device(self, state: SubwordBatch) -> torch.Tensor:
        dev_rows = getattr(self.char_lm, "log_probs_device", None)
        if dev_rows is not None:
            return dev_rows(state.char_states)
        rows = np.stack([np.asarray(self.char_lm.log_probs(s), np.float64)
                         for s in state.char_states])
        return torch.as_tensor(rows, device=self.device)

    def char_scores(self, state: SubwordBatch) -> np.ndarray:
        if getattr(self.char_lm, "log_probs_device", None) is not None:
            return self.char_scores_device(state).cpu().numpy()
        return np.stack([self.char_lm.log_probs(s) for s in state.char_states])

    def advance(self, state: SubwordBatch, tokens: Sequence[int]) -> SubwordBatch:
        toks = [int(t) for t in np.asarray(tokens).reshape(-1)]
        if len(toks) != len(state):
            raise ValueError("one chosen token per hypothesis row required")
        many = getattr(self.char_lm, "advance_many", None)
        if many is not None:
            return SubwordBatch(many(state.char_states, toks))
        return SubwordBatch([self.char_lm.advance(s, t) for s, t in zip(state.char_states, toks)])

    def reorder(self, state: SubwordBatch, parent_indices: Sequence[int]) -> SubwordBatch:
        return SubwordBatch([state.char_states[i] for i in parent_indices])


# ---- multilevel fusion (fusion.py:268-380) ----------------------------------------
class MultilevelBatch:
    """Per-row state: provider states (host list), trie state / g... slot / char
    accumulator on the device, word histories (host)."""

    def __init__(self, fusion, char_states, states_dev, slots_dev, accum_dev, histories):
        self._fusion = fusion
        self.char_states = char_states
        self.states_dev = states_dev          # int32 [n]: >= 0 or OOV_STATE
        self.slots_dev = slots_dev            # int32 [n]: distribution-pool slot of histories[i]
        self.accum_dev = accum_dev            # fp64 [n]: char log-prob mass of the open word
        self.histories = histories

    def __len__(self) -> int:
        return len(self.char_states)

    @property
    def trie_states(self) -> np.ndarray:
        return self.states_dev.cpu().numpy().astype(np.int64)

    @property
    def char_accum(self) -> np.ndarray:
        return self.accum_dev.cpu().numpy()


class MultilevelFusion(FusionScorer):
    """Character-LM rows with word-LM rescoring at word boundaries (reference
    fusion.py:280-380): the <space>/<eos> columns get log P_W(w|h) minus the char
    mass paid for the word's spelling (known word), ``oov_factor`` (unknown or
    partial word) or nothing (empty word).  Scores can be positive, so
    ``nonpositive_scores`` is False (the decoder then never stops early).

    Device side: the row adjustment (``fb_multilevel_rows``) and the per-row
    state update (``fb_multilevel_advance``: accumulator, CSR trie walk,
    boundary ranks, empty-word count); each distinct word history's
    distribution row is uploaded once into a device pool."""

    nonpositive_scores = False

    def __init__(self, char_lm, word_lm, trie, token_dict,
                 oov_factor: float = DEFAULT_OOV_PENALTY, device=None):
        if word_lm.vocab_size != trie.num_words:
            raise ConfigError(f"word LM vocabulary ({word_lm.vocab_size}) does not match"
                              f" the automaton ({trie.num_words} words)")
        if not isinstance(trie, PrefixTreeAutomaton):
            trie = _converted(trie)
        self.char_lm, self.word_lm, self.trie = char_lm, word_lm, trie
        self.oov_factor = float(oov_factor)
        self.space_id, self.eos_id, self.pad_id = (token_dict.space_id, token_dict.eos_id,
                                                   token_dict.pad_id)
        self.dict_size = len(token_dict)
        self.device = _device(device)
        self.dtrie = DeviceTrie.of(trie, self.device)
        self._pool = GPool(trie.num_words, self.device)     # rows = distributions (not cumsum)
        self._slot_of: Dict[tuple, int] = {}
        self._empty = torch.zeros(1, dtype=torch.int64, device=self.device)

    @property
    def diagnostics(self) -> dict:
        return {"empty_words": int(self._empty.item())}

    def _slots_for(self, hists: list) -> List[int]:
        todo = {}
        for h in hists:
            k = _hkey(h)
            if k not in self._slot_of and k not in todo:
                todo[k] = h
        if todo:
            keys = list(todo)
            ids = self._pool.alloc(len(keys))
            dists = np.stack([np.asarray(self.word_lm.full_distribution(todo[k]), np.float64)
                              for k in keys])
            self._pool.rows[torch.as_tensor(ids, device=self.device).long()] = torch.as_tensor(
                dists, device=self.device)
            for k, s_ in zip(keys, ids):
                self._slot_of[k] = int(s_)
        return [self._slot_of[_hkey(h)] for h in hists]

    def _char_rows(self, char_states) -> torch.Tensor:
        dev_rows = getattr(self.char_lm, "log_probs_device", None)
        if dev_rows is not None:
            return dev_rows(char_states).to(torch.float64).clone()
        rows = np.stack([np.asarray(self.char_lm.log_probs(s), np.float64) for s in char_states])
        return torch.as_tensor(rows, device=self.device)

    def start(self, n: int) -> MultilevelBatch:
        h0 = self.word_lm.start_history()
        s0 = self._slots_for([h0])[0]
        z32 = lambda v: torch.full((n,), v, dtype=torch.int32, device=self.device)  # noqa: E731
        return MultilevelBatch(self, [self.char_lm.start()] * n, z32(0), z32(s0),
                               torch.zeros(n, dtype=torch.float64, device=self.device), [h0] * n)

    def char_scores_device(self, state: MultilevelBatch) -> torch.Tensor:
        n = len(state)
        rows = self._char_rows(state.char_states) if n else \
            torch.empty((0, self.dict_size), dtype=torch.float64, device=self.device)
        if n:
            _lib.call("fb_multilevel_rows", self.dtrie.ref, n, _lib.ptr(state.states_dev),
                      _lib.ptr(state.slots_dev), _lib.ptr(self._pool.rows), self._pool.vw,
                      _lib.ptr(state.accum_dev), self.space_id, self.eos_id, self.oov_factor,
                      SCORE_FLOOR, _lib.ptr(rows), rows.stride(0), _lib.stream_ptr())
        return rows

    def char_scores(self, state: MultilevelBatch) -> np.ndarray:
        return self.char_scores_device(state).cpu().numpy()

    def advance(self, state: MultilevelBatch, tokens: Sequence[int]) -> MultilevelBatch:
        tok = np.asarray(tokens, dtype=np.int64).reshape(-1)
        n = len(state)
        if tok.shape != (n,):
            raise ValueError("one chosen token per hypothesis row required")
        if n == 0:
            return MultilevelBatch(self, [], state.states_dev.clone(), state.slots_dev.clone(),
                                   state.accum_dev.clone(), [])
        char_rows = self._char_rows(state.char_states)      # unadjusted rows of the old states
        tok_d = torch.as_tensor(tok.astype(np.int32), device=self.device)
        s_out = torch.empty_like(state.states_dev)
        a_out = torch.empty_like(state.accum_dev)
        brank = torch.empty_like(state.states_dev)
        _lib.call("fb_multilevel_advance", self.dtrie.ref, n, _lib.ptr(state.states_dev),
                  _lib.ptr(state.accum_dev), _lib.ptr(tok_d), _lib.ptr(char_rows),
                  char_rows.stride(0), self.space_id, self.eos_id, self.pad_id, _lib.ptr(s_out),
                  _lib.ptr(a_out), _lib.ptr(brank), _lib.ptr(self._empty), _lib.stream_ptr())
        many = getattr(self.char_lm, "advance_many", None)
        toks = [int(t) for t in tok]
        char_states = (many(state.char_states, toks) if many is not None else
                       [self.char_lm.advance(s_, t) for s_, t in zip(state.char_states, toks)])
        hist = list(state.histories)
        slots = state.slots_dev.clone()
        br = brank.cpu().numpy()
        rows_b = np.nonzero(br != -2)[0]
        if rows_b.size:
            for b in rows_b:
                hist[b] = self.word_lm.extend_history(hist[b], int(br[b]))
            new = self._slots_for([hist[b] for b in rows_b])
            slots[torch.as_tensor(rows_b, device=self.device)] = torch.as_tensor(
                np.asarray(new, np.int32), device=self.device)
        return MultilevelBatch(self, char_states, s_out, slots, a_out, hist)

    def reorder(self, state: MultilevelBatch, parent_indices: Sequence[int]) -> MultilevelBatch:
        idx_np = np.asarray(parent_indices, dtype=np.int64)
        idx = torch.as_tensor(idx_np, device=self.device)
        return MultilevelBatch(self, [state.char_states[i] for i in idx_np],
                               state.states_dev[idx], state.slots_dev[idx], state.accum_dev[idx],
                               [state.histories[i] for i in idx_np])
