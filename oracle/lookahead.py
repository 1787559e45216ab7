"""Oracle restatement of look-ahead word-LM fusion (Eq. 4 of the paper).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``fusion.py:109-233`` (``LookaheadFusion.start/char_scores/advance/
reorder``) and the table word-LM fake ``word_lm.py:239-328`` used by the
reference tests.  All arithmetic is float64 numpy in the same operation order
as the reference (``log(numer) - log(denom)``, not ``log(numer/denom)``;
sequential ``cumsum``), so restatement == reference bit-for-bit.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence

import numpy as np

from .lexicon import NO_STATE, OracleDict, OracleTrie

OOV_STATE = -2             # fusion.py:35
OOV_PENALTY = -10.0        # fusion.py:37
SCORE_FLOOR = -30.0        # char_lm.py:20
UNK_RANK = -1              # word_lm.py:26


class OracleTableLM:
    """word_lm.py:239-328: explicit rows per history tuple, uniform otherwise;
    histories are tuples of word strings (extend appends the word,
    ``UNK_RANK`` appends ``<unk>``)."""

    def __init__(self, vocab: Sequence[str], rows=None, eos=None):
        self.vocab = tuple(vocab)
        self.vocab_size = len(self.vocab)
        self._rows = {tuple(h): np.asarray(r, np.float64) for h, r in (rows or {}).items()}
        self._eos = {tuple(h): float(p) for h, p in (eos or {}).items()}
        self._uniform = np.full(self.vocab_size, 1.0 / self.vocab_size)

    def start_history(self):
        return ()

    def extend_history(self, h, rank: int):
        w = "<unk>" if rank == UNK_RANK else self.vocab[rank]
        return tuple(h) + (w,)

    def full_distribution(self, h) -> np.ndarray:
        row = self._rows.get(tuple(h))
        if row is None:
            return self._uniform
        tot = row.sum()
        return self._uniform if tot <= 0.0 else row / tot

    def eos_log_prob(self, h) -> float:
        p = self._eos.get(tuple(h), 1.0 / (self.vocab_size + 1))
        return math.log(max(p, 1e-12))


class OracleLookahead:
    """fusion.py:77-233 restated.  State = (trie_states int64[n], histories list,
    g float64[n, V])."""

    nonpositive_scores = True

    def __init__(self, trie: OracleTrie, word_lm, d: OracleDict,
                 oov_penalty: float = OOV_PENALTY, score_floor: float = SCORE_FLOOR):
        if word_lm.vocab_size != trie.num_words:
            raise ValueError("word LM vocabulary does not match the automaton")
        if trie.alphabet_size != len(d):
            raise ValueError("automaton alphabet does not match the dictionary")
        self.lm = word_lm
        self.pen = float(oov_penalty)
        self.floor = float(score_floor)
        self.space, self.eos, self.pad = d.space_id, d.eos_id, d.pad_id
        self.V = len(d)
        self.kids = trie.children_dense().astype(np.int64)
        self.ub = trie.ub_index.astype(np.int64)
        self.lb = trie.lb_index.astype(np.int64)
        self.final = trie.is_final.copy()
        self.rank = trie.word_index.astype(np.int64)
        self.floored = 0

    # fusion.py:109-116
    def start(self, n: int):
        h0 = self.lm.start_history()
        g0 = np.cumsum(np.asarray(self.lm.full_distribution(h0), np.float64))
        return (np.zeros(n, np.int64), [h0] * n, np.tile(g0, (n, 1)))

    @staticmethod
    def _mass(g, rows, hi, lo):
        """g[hi] - g[lo] with g[-1] := 0 (fusion.py:135-146)."""
        up = np.take_along_axis(g, hi, axis=1) if hi.ndim == 2 else g[rows, hi]
        if lo.ndim == 2:
            low = np.take_along_axis(g, np.maximum(lo, 0), axis=1)
        else:
            low = g[rows, np.maximum(lo, 0)]
        return up - np.where(lo >= 0, low, 0.0)

    # fusion.py:118-185
    def char_scores(self, state) -> np.ndarray:
        states, hists, g = state
        n = len(hists)
        out = np.full((n, self.V), self.pen)
        if n == 0:
            return out
        ok = states >= 0
        if not ok.any():
            return out
        s = np.where(ok, states, 0)
        rows = np.arange(n)
        kid = self.kids[s]
        edge = kid >= 0
        kid0 = np.where(edge, kid, 0)
        numer = self._mass(g, rows, self.ub[kid0], self.lb[kid0])
        denom = self._mass(g, rows, self.ub[s], self.lb[s])
        with np.errstate(divide="ignore", invalid="ignore"):
            lg = np.log(numer) - np.log(denom)[:, None]
        good = (numer > 0) & (denom > 0)[:, None]
        self.floored += int(np.count_nonzero(edge & ok[:, None] & ~good))
        lg = np.where(good, lg, self.floor)
        out = np.where(ok[:, None] & edge, lg, out)

        fin = self.final[s] & ok
        r = np.maximum(self.rank[s], 0)
        wmass = self._mass(g, rows, r, r - 1)
        with np.errstate(divide="ignore", invalid="ignore"):
            wend = np.log(wmass) - np.log(denom)
        wgood = (wmass > 0) & (denom > 0)
        self.floored += int(np.count_nonzero(fin & ~wgood))
        wend = np.where(wgood, wend, self.floor)
        out[:, self.space] = np.where(fin, wend, self.pen)

        ecol = np.full(n, self.pen)
        for b in np.nonzero(ok)[0]:
            st = int(states[b])
            if st == 0:
                ecol[b] = self.lm.eos_log_prob(hists[b])
            elif self.final[st]:
                ext = self.lm.extend_history(hists[b], int(self.rank[st]))
                ecol[b] = wend[b] + self.lm.eos_log_prob(ext)
        out[:, self.eos] = ecol
        return out

    # fusion.py:187-224
    def advance(self, state, tokens):
        states, hists, g = state
        tokens = np.asarray(tokens, np.int64)
        n = len(hists)
        if tokens.shape != (n,):
            raise ValueError("one chosen token per hypothesis row required")
        ok = states >= 0
        s = np.where(ok, states, 0)
        inword = (tokens != self.space) & (tokens != self.eos) & (tokens != self.pad)
        nxt = self.kids[s, np.clip(tokens, 0, self.V - 1)]
        nxt = np.where(ok, nxt, NO_STATE)
        nxt = np.where(nxt == NO_STATE, OOV_STATE, nxt)
        new = np.where(inword, nxt, states)
        brk = tokens == self.space
        new = np.where(brk, 0, new)
        hists = list(hists)
        g = g.copy()
        idx = np.nonzero(brk)[0]
        if idx.size:
            dists = []
            for b in idx:
                st = int(states[b])
                rk = int(self.rank[st]) if (st >= 0 and self.final[st]) else UNK_RANK
                hists[b] = self.lm.extend_history(hists[b], rk)
                dists.append(self.lm.full_distribution(hists[b]))
            g[idx] = np.cumsum(np.stack(dists), axis=1)
        return (new, hists, g)

    # fusion.py:226-233
    def reorder(self, state, parents):
        states, hists, g = state
        idx = np.asarray(parents, np.int64)
        return (states[idx], [hists[i] for i in idx], g[idx])
