"""Oracle restatement of plain token-level LM fusion (config 4).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``OracleSubwordFusion`` follows ``fusion.py:236-266`` (``SubwordBatch``,
  ``SubwordFusion``: the provider's rows stacked, per-row advance/reorder,
  ``nonpositive_scores`` inherited True ``fusion.py:50``).
* ``OracleUniformCharLM`` follows ``char_lm.py:36-53`` (``SCORE_FLOOR``
  ``char_lm.py:20``).
* ``OracleLstmCharLM`` implements the ``CharLM`` protocol ``char_lm.py:23-33``
  over a random-init token LSTM LM (the reference ships only n-gram/uniform
  providers): state = (h, c, fp32 logits) after consuming ``<eos>`` then the
  history; ``log_probs`` = fp64 log-softmax of the fp32 logits over every
  non-pad token, ``<pad>`` and anything below the floor set to
  ``SCORE_FLOOR`` (the row contract of ``char_lm.py:1-7, 83-95``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Sequence

import numpy as np
import torch

from .neural import _lstm_cell, _t

SCORE_FLOOR = -30.0


@dataclass
class OracleSubwordBatch:
    char_states: list

    def __len__(self) -> int:
        return len(self.char_states)


class OracleSubwordFusion:
    """fusion.py:244-266."""

    nonpositive_scores = True

    def __init__(self, char_lm, batched: bool = True):
        self.char_lm = char_lm
        self.batched = batched       # False: per-row advance exactly as fusion.py:258-262
        self.diagnostics: dict = {}

    def start(self, n: int) -> OracleSubwordBatch:
        s0 = self.char_lm.start()
        return OracleSubwordBatch([s0] * n)

    def char_scores(self, state: OracleSubwordBatch) -> np.ndarray:
        return np.stack([self.char_lm.log_probs(s) for s in state.char_states])

    def advance(self, state: OracleSubwordBatch, tokens: Sequence[int]) -> OracleSubwordBatch:
        many = getattr(self.char_lm, "advance_many", None) if self.batched else None
        if many is not None:                       # batched, row-for-row identical math
            return OracleSubwordBatch(many(state.char_states, [int(t) for t in tokens]))
        return OracleSubwordBatch([self.char_lm.advance(s, int(t))
                                   for s, t in zip(state.char_states, tokens)])

    def reorder(self, state: OracleSubwordBatch, parent_indices: Sequence[int]
                ) -> OracleSubwordBatch:
        return OracleSubwordBatch([state.char_states[i] for i in parent_indices])


class OracleUniformCharLM:
    """char_lm.py:36-53."""

    def __init__(self, dict_size: int, pad_id: int):
        row = np.full(dict_size, math.log(1.0 / (dict_size - 1)))
        row[pad_id] = SCORE_FLOOR
        row.setflags(write=False)
        self._row = row

    def start(self):
        return ()

    def log_probs(self, state) -> np.ndarray:
        return self._row

    def advance(self, state, token_id: int):
        return ()


class OracleTableCharLM:
    """Test fake: rows keyed by the token history (longest listed suffix wins,
    else the default row) -- a CharLM with a history-dependent state."""

    def __init__(self, rows: Dict[tuple, np.ndarray], default: np.ndarray):
        self.rows, self.default = rows, default

    def start(self):
        return ()

    def log_probs(self, state) -> np.ndarray:
        for k in range(len(state), -1, -1):
            r = self.rows.get(tuple(state[len(state) - k:]))
            if r is not None:
                return r
        return self.default

    def advance(self, state, token_id: int):
        return tuple(state) + (int(token_id),)


class _Tok:
    __slots__ = ("h", "c", "row")

    def __init__(self, h, c, row):
        self.h, self.c, self.row = h, c, row


class OracleLstmCharLM:
    """CharLM over a token LSTM LM (weights ``slm.*`` from synth.subword_lm_weights)."""

    def __init__(self, W: Dict[str, np.ndarray], layers: int, pad_id: int, eos_id: int,
                 dtype=torch.float32):
        self.L = layers
        self.pad, self.eos = pad_id, eos_id
        self.w = {k: _t(v).to(dtype) for k, v in W.items() if k.startswith("slm.")}
        self.H = self.w["slm.0.w_hh"].shape[1]
        z = torch.zeros(1, self.L, self.H, dtype=dtype)
        self._start = self._run(z, z, [eos_id])[0]

    @torch.no_grad()
    def _run(self, h, c, tokens: List[int]) -> List[_Tok]:
        """h, c: [n, L, H]; one LSTM step per row on its token."""
        x = self.w["slm.emb"][torch.as_tensor(tokens, dtype=torch.long)]
        hs, cs = [], []
        for l in range(self.L):
            hh, cc = _lstm_cell(x, h[:, l], c[:, l], self.w[f"slm.{l}.w_ih"],
                                self.w[f"slm.{l}.w_hh"], self.w[f"slm.{l}.b"])
            hs.append(hh)
            cs.append(cc)
            x = hh
        logits = (x @ self.w["slm.out.w"].T + self.w["slm.out.b"]).numpy()
        H2, C2 = torch.stack(hs, 1), torch.stack(cs, 1)
        return [_Tok(H2[i:i + 1], C2[i:i + 1], self._row(logits[i])) for i in range(len(tokens))]

    def _row(self, logits: np.ndarray) -> np.ndarray:
        z = logits.astype(np.float64)
        keep = np.ones(z.shape[0], bool)
        keep[self.pad] = False
        m = z[keep].max()
        lse = m + np.log(np.exp(z[keep] - m).sum())
        row = z - lse
        row[self.pad] = SCORE_FLOOR
        row[row < SCORE_FLOOR] = SCORE_FLOOR
        row.setflags(write=False)
        return row

    def start(self) -> _Tok:
        return self._start

    def log_probs(self, state: _Tok) -> np.ndarray:
        return state.row

    def advance(self, state: _Tok, token_id: int) -> _Tok:
        return self._run(state.h, state.c, [int(token_id)])[0]

    def advance_many(self, states: Sequence[_Tok], tokens: Sequence[int]) -> List[_Tok]:
        if not states:
            return []
        h = torch.cat([s.h for s in states])
        c = torch.cat([s.c for s in states])
        return self._run(h, c, list(tokens))


# ---- multilevel fusion (fusion.py:268-380) ----------------------------------------
OOV_STATE = -2
UNK_RANK = -1


@dataclass
class OracleMultilevelBatch:
    char_states: list
    trie_states: np.ndarray
    histories: list
    char_accum: np.ndarray

    def __len__(self) -> int:
        return len(self.char_states)


class OracleMultilevelFusion:
    """fusion.py:280-380: char-LM rows, word-LM rescoring at word boundaries."""

    nonpositive_scores = False

    def __init__(self, char_lm, word_lm, trie, token_dict, oov_factor: float = -10.0):
        self.char_lm, self.word_lm, self.trie = char_lm, word_lm, trie
        self.oov_factor = float(oov_factor)
        self.space_id, self.eos_id, self.pad_id = (token_dict.space_id, token_dict.eos_id,
                                                   token_dict.pad_id)
        self.diagnostics = {"empty_words": 0}
        kids = trie.children_dense() if hasattr(trie, "children_dense") else trie.char_children
        self._children = kids.astype(np.int64)
        self._final = trie.is_final.copy()
        self._rank = trie.word_index.astype(np.int64)

    def start(self, n: int) -> OracleMultilevelBatch:
        return OracleMultilevelBatch([self.char_lm.start()] * n, np.zeros(n, np.int64),
                                     [self.word_lm.start_history()] * n, np.zeros(n))

    def _adjust(self, state, b: int) -> float:                       # fusion.py:321-330
        st = int(state.trie_states[b])
        if st == 0 and state.char_accum[b] == 0.0:
            return 0.0
        if st >= 0 and self._final[st]:
            p = float(self.word_lm.full_distribution(state.histories[b])[int(self._rank[st])])
            return float((np.log(p) if p > 0 else SCORE_FLOOR) - state.char_accum[b])
        return self.oov_factor

    def char_scores(self, state) -> np.ndarray:                      # fusion.py:332-339
        rows = np.stack([self.char_lm.log_probs(s) for s in state.char_states]).astype(
            np.float64, copy=True)
        for b in range(len(state)):
            adj = self._adjust(state, b)
            rows[b, self.space_id] += adj
            rows[b, self.eos_id] += adj
        return rows

    def advance(self, state, tokens) -> OracleMultilevelBatch:       # fusion.py:341-371
        tokens = np.asarray(tokens, dtype=np.int64)
        cs = [self.char_lm.advance(s, int(t)) for s, t in zip(state.char_states, tokens)]
        ts = state.trie_states.copy()
        hs = list(state.histories)
        acc = state.char_accum.copy()
        for b in range(len(state)):
            tok = int(tokens[b])
            if tok == self.pad_id:
                continue
            if tok == self.space_id or tok == self.eos_id:
                st = int(ts[b])
                if st == 0 and acc[b] == 0.0:
                    self.diagnostics["empty_words"] += 1
                rank = int(self._rank[st]) if st >= 0 and self._final[st] else UNK_RANK
                hs[b] = self.word_lm.extend_history(hs[b], rank)
                ts[b] = 0
                acc[b] = 0.0
                continue
            acc[b] += float(self.char_lm.log_probs(state.char_states[b])[tok])
            st = int(ts[b])
            nxt = int(self._children[st, tok]) if st >= 0 else -1
            ts[b] = nxt if nxt != -1 else OOV_STATE
        return OracleMultilevelBatch(cs, ts, hs, acc)

    def reorder(self, state, parent_indices) -> OracleMultilevelBatch:
        idx = np.asarray(parent_indices, dtype=np.int64)
        return OracleMultilevelBatch([state.char_states[i] for i in idx], state.trie_states[idx],
                                     [state.histories[i] for i in idx], state.char_accum[idx])
