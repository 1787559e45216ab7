"""Prefix-tree automaton over the word vocabulary, packed for the device.

Same states, ranks and bounds as the reference ``lexicon_trie.py:47-276``
(verified array-for-array in ``tests/test_trie_pack.py``), built differently:
the vocabulary is sorted by character-id tuple once and every word opens new
states only past its longest common prefix with the previous word, so state
ids, first/last ranks (``lb = first - 1``, ``ub = last``) and per-state edge
order fall out of one linear sweep.

The device form is CSR (``row_ptr``/``edge_label``/``edge_child``) plus one
int4 per state ``{ub, lb, rank, 0}`` -- a few MB at 65k words instead of the
dense ``[S, alphabet]`` child map.
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .errors import FormatError

NO_STATE = -1


def word_char_ids(word: str, token_dict) -> Tuple[int, ...]:
    if not word:
        raise FormatError("empty word in vocabulary")
    ids = []
    for ch in word:
        if ch not in token_dict:
            raise FormatError(f"word {word!r} contains character {ch!r} not in the dictionary")
        ids.append(token_dict.index(ch))
    return tuple(ids)


def rank_order(vocab: Sequence[str], token_dict) -> List[str]:
    return sorted(vocab, key=lambda w: word_char_ids(w, token_dict))


class PrefixTreeAutomaton:
    """Trie arrays in the reference layout plus the CSR pack used on device."""

    def __init__(self, transitions, edge_labels, is_final, word_index, ub_index, lb_index,
                 alphabet_size: int):
        self.transitions = np.asarray(transitions, np.int32)
        self.edge_labels = np.asarray(edge_labels, np.int32)
        self.is_final = np.asarray(is_final, bool)
        self.word_index = np.asarray(word_index, np.int32)
        self.ub_index = np.asarray(ub_index, np.int32)
        self.lb_index = np.asarray(lb_index, np.int32)
        self.alphabet_size = int(alphabet_size)
        self.num_states = int(self.transitions.shape[0])
        self.max_out_degree = int(self.transitions.shape[1])
        self.num_words = int(self.is_final.sum())
        self._check()
        self._csr = None

    def _check(self) -> None:
        S = self.num_states
        if S < 1 or self.max_out_degree < 1:
            raise FormatError("automaton must have at least one state and slot")
        for a in (self.is_final, self.word_index, self.ub_index, self.lb_index):
            if a.shape != (S,):
                raise FormatError("automaton arrays have inconsistent shapes")
        if self.edge_labels.shape != self.transitions.shape:
            raise FormatError("automaton arrays have inconsistent shapes")
        live = self.transitions != NO_STATE
        tgt = self.transitions[live]
        if tgt.size != S - 1 or np.unique(tgt).size != S - 1 or (tgt < 1).any() or (tgt >= S).any():
            raise FormatError("every non-root state needs exactly one parent")
        lab = self.edge_labels[live]
        if (lab < 0).any() or (lab >= self.alphabet_size).any():
            raise FormatError("edge label out of range")
        if not np.array_equal(np.sort(self.word_index[self.is_final]), np.arange(self.num_words)):
            raise FormatError("final-state word ranks are not 0..num_words-1")
        if ((self.ub_index < 0) | (self.ub_index >= self.num_words)).any() or \
                ((self.lb_index < -1) | (self.lb_index > self.ub_index)).any():
            raise FormatError("rank bound out of range")

    @classmethod
    def from_reference(cls, trie) -> "PrefixTreeAutomaton":
        """Adopt any object with the reference automaton's arrays."""
        return cls(trie.transitions, trie.edge_labels, trie.is_final, trie.word_index,
                   trie.ub_index, trie.lb_index, trie.alphabet_size)

    # ---- host-side queries (reference lexicon_trie.py:131-176) -------------
    @property
    def char_children(self) -> np.ndarray:
        out = np.full((self.num_states, self.alphabet_size), NO_STATE, np.int32)
        s, k = np.nonzero(self.transitions != NO_STATE)
        out[s, self.edge_labels[s, k]] = self.transitions[s, k]
        return out

    def child(self, state: int, char: int) -> int:
        row_ptr, lab, kid, _ = self.csr()
        a, b = row_ptr[state], row_ptr[state + 1]
        j = a + int(np.searchsorted(lab[a:b], char))
        return int(kid[j]) if j < b and lab[j] == char else NO_STATE

    def state_of_prefix(self, char_ids: Sequence[int]) -> int:
        s = 0
        for c in char_ids:
            s = self.child(s, int(c))
            if s == NO_STATE:
                break
        return s

    def words(self, token_dict) -> List[str]:
        par = np.zeros(self.num_states, np.int64)
        ch = np.zeros(self.num_states, np.int64)
        s, k = np.nonzero(self.transitions != NO_STATE)
        par[self.transitions[s, k]] = s
        ch[self.transitions[s, k]] = self.edge_labels[s, k]
        finals = np.nonzero(self.is_final)[0]
        order = finals[np.argsort(self.word_index[finals])]
        out = []
        for st in order:
            cs = []
            while st:
                cs.append(token_dict.token(int(ch[st])))
                st = par[st]
            out.append("".join(reversed(cs)))
        return out

    # ---- device pack --------------------------------------------------------
    def csr(self):
        """(row_ptr[S+1], edge_label[E], edge_child[E], info[S,4]) int32, labels
        ascending within each state."""
        if self._csr is None:
            live = self.transitions != NO_STATE
            deg = live.sum(axis=1)
            row_ptr = np.zeros(self.num_states + 1, np.int32)
            np.cumsum(deg, out=row_ptr[1:])
            s, k = np.nonzero(live)
            lab = self.edge_labels[s, k]
            kid = self.transitions[s, k]
            order = np.lexsort((lab, s))
            info = np.zeros((self.num_states, 4), np.int32)
            info[:, 0] = self.ub_index
            info[:, 1] = self.lb_index
            info[:, 2] = np.where(self.is_final, self.word_index, -1)
            self._csr = (row_ptr, lab[order].astype(np.int32), kid[order].astype(np.int32), info)
        return self._csr


def build_trie(vocab: Sequence[str], token_dict) -> PrefixTreeAutomaton:
    """Linear sweep over the rank-sorted vocabulary (see module docstring)."""
    if not vocab:
        raise FormatError("empty vocabulary")
    seen = set()
    seqs = []
    for w in vocab:
        if w in seen:
            raise FormatError(f"duplicate word {w!r} in vocabulary")
        seen.add(w)
        seqs.append(word_char_ids(w, token_dict))
    seqs.sort()
    n_states = 1 + sum(len(q) for q in seqs)          # upper bound
    first = np.zeros(n_states, np.int64)
    last = np.zeros(n_states, np.int64)
    rank_of = np.full(n_states, -1, np.int64)
    parent = np.zeros(n_states, np.int64)
    label = np.zeros(n_states, np.int64)
    path = [0]                                         # state ids along the previous word
    prev: Tuple[int, ...] = ()
    nxt = 1
    for r, q in enumerate(seqs):
        lcp = 0
        m = min(len(prev), len(q))
        while lcp < m and prev[lcp] == q[lcp]:
            lcp += 1
        del path[lcp + 1:]
        for pos in range(lcp, len(q)):
            parent[nxt] = path[-1]
            label[nxt] = q[pos]
            first[nxt] = r
            path.append(nxt)
            nxt += 1
        last[path] = r                                 # every state on the path covers rank r
        rank_of[path[-1]] = r
        prev = q
    S = nxt
    kids_per = np.bincount(parent[1:S], minlength=S)
    D = int(kids_per.max())
    trans = np.full((S, D), NO_STATE, np.int32)
    labels = np.full((S, D), NO_STATE, np.int32)
    slot = np.zeros(S, np.int64)
    for st in range(1, S):                             # creation order == ascending label per parent
        p = parent[st]
        trans[p, slot[p]] = st
        labels[p, slot[p]] = label[st]
        slot[p] += 1
    return PrefixTreeAutomaton(trans, labels, rank_of[:S] >= 0, rank_of[:S].astype(np.int32),
                               last[:S].astype(np.int32), (first[:S] - 1).astype(np.int32),
                               len(token_dict))
