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

import functools
import os
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
        """The reference's automaton invariants and FormatError texts
        (lexicon_trie.py:64-129), in its order; reachability is checked by
        pointer jumping on the parent array instead of a BFS."""
        S, D = self.num_states, self.max_out_degree
        if S < 1 or D < 1:
            raise FormatError("automaton must have at least one state and slot")
        if self.edge_labels.shape != (S, D) or any(
                a.shape != (S,) for a in (self.is_final, self.word_index, self.ub_index,
                                          self.lb_index)):
            raise FormatError("automaton arrays have inconsistent shapes")
        live = self.transitions != NO_STATE
        tgt = self.transitions[live]
        if ((tgt < 1) | (tgt >= S)).any():
            raise FormatError("transition target out of range (or pointing at root)")
        lab = self.edge_labels[live]
        if ((lab < 0) | (lab >= self.alphabet_size)).any():
            raise FormatError("edge label out of range")
        if (self.edge_labels[~live] != NO_STATE).any():
            raise FormatError("unused transition slot with a live edge label")
        if tgt.size != S - 1 or np.unique(tgt).size != S - 1:
            raise FormatError("every non-root state needs exactly one parent")
        if self.num_words < 1 or not np.array_equal(np.sort(self.word_index[self.is_final]),
                                                    np.arange(self.num_words)):
            raise FormatError("final-state word ranks are not 0..num_words-1")
        if (self.word_index[~self.is_final] != -1).any():
            raise FormatError("non-final state carries a word rank")
        if ((self.ub_index < 0) | (self.ub_index >= self.num_words)).any():
            raise FormatError("upper-bound rank out of range")
        if ((self.lb_index < -1) | (self.lb_index > self.ub_index)).any():
            raise FormatError("lower-bound rank out of range")
        # every state has one parent; it is reachable iff its ancestor chain
        # ends at the root: jump up 2^k ancestors at a time (log2 S rounds)
        up = self._parents()[0].astype(np.int64)
        up[0] = 0
        for _ in range(max(1, int(S).bit_length())):
            up = up[up]
        if (up != 0).any():
            raise FormatError("automaton has states unreachable from the root")

    def _parents(self):
        s, k = np.nonzero(self.transitions != NO_STATE)
        kid = self.transitions[s, k]
        par = np.full(self.num_states, NO_STATE, np.int32)
        ch = np.full(self.num_states, NO_STATE, np.int32)
        par[kid] = s
        ch[kid] = self.edge_labels[s, k]
        return par, ch

    @classmethod
    def from_reference(cls, trie) -> "PrefixTreeAutomaton":
        """Adopt any object with the reference automaton's arrays."""
        return cls(trie.transitions, trie.edge_labels, trie.is_final, trie.word_index,
                   trie.ub_index, trie.lb_index, trie.alphabet_size)

    # ---- host-side queries (reference lexicon_trie.py:101-176) --------------
    # Derived arrays are built on first use and cached (the dense child map is
    # 50 MB at 65k words and only the host API needs it; the device uses CSR).
    @functools.cached_property
    def char_children(self) -> np.ndarray:
        out = np.full((self.num_states, self.alphabet_size), NO_STATE, np.int32)
        s, k = np.nonzero(self.transitions != NO_STATE)
        out[s, self.edge_labels[s, k]] = self.transitions[s, k]
        out.setflags(write=False)
        return out

    @functools.cached_property
    def _parent_arrays(self):
        par, ch = self._parents()
        par.setflags(write=False)
        ch.setflags(write=False)
        return par, ch

    @property
    def parent_state(self) -> np.ndarray:
        return self._parent_arrays[0]

    @property
    def parent_char(self) -> np.ndarray:
        return self._parent_arrays[1]

    @functools.cached_property
    def final_state_of_rank(self) -> np.ndarray:
        out = np.full(self.num_words, NO_STATE, np.int32)
        fin = np.nonzero(self.is_final)[0]
        out[self.word_index[fin]] = fin
        out.setflags(write=False)
        return out

    def advance(self, states, chars) -> np.ndarray:
        """Batched transition (NO_STATE where no edge), reference
        lexicon_trie.py:131-143 incl. its ValueErrors."""
        st = np.asarray(states, np.int64)
        ch = np.asarray(chars, np.int64)
        if st.shape != ch.shape:
            raise ValueError("states and chars must have equal length")
        if st.size == 0:
            return st.astype(np.int32)
        if st.min() < 0 or st.max() >= self.num_states:
            raise ValueError("state index out of range")
        if ch.min() < 0 or ch.max() >= self.alphabet_size:
            raise ValueError("character id out of range")
        return self.char_children[st, ch]

    def bounds(self, states) -> Tuple[np.ndarray, np.ndarray]:
        """(ub, lb) rank bounds per state (lexicon_trie.py:145-150)."""
        st = np.asarray(states, np.int64)
        if st.size and (st.min() < 0 or st.max() >= self.num_states):
            raise ValueError("bounds() requires valid (non-sentinel) states")
        return self.ub_index[st].copy(), self.lb_index[st].copy()

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

    def spell(self, rank: int) -> List[int]:
        """Character ids of the word of this rank (root-to-leaf)."""
        par, ch = self._parent_arrays
        st = int(self.final_state_of_rank[rank])
        out: List[int] = []
        while st > 0:
            out.append(int(ch[st]))
            st = int(par[st])
        out.reverse()
        return out

    def words(self, token_dict) -> List[str]:
        return ["".join(token_dict.token(c) for c in self.spell(r))
                for r in range(self.num_words)]

    # ---- PTA1 files (reference lexicon_trie.py:178-224), native I/O ----------
    def save(self, path: str) -> None:
        from . import _lib
        a = lambda x, dt=np.int32: np.ascontiguousarray(x, dt)  # noqa: E731
        t, e, f = a(self.transitions), a(self.edge_labels), a(self.is_final, np.uint8)
        w, u, lb = a(self.word_index), a(self.ub_index), a(self.lb_index)
        _lib.call("fb_pta1_write", path.encode(), self.num_states, self.num_words,
                  self.max_out_degree, self.alphabet_size, t.ctypes.data, e.ctypes.data,
                  f.ctypes.data, w.ctypes.data, u.ctypes.data, lb.ctypes.data)

    @classmethod
    def load(cls, path: str) -> "PrefixTreeAutomaton":
        import ctypes as C
        from . import _lib
        S, W, D, A = (C.c_int32() for _ in range(4))
        _lib.call("fb_pta1_read_header", path.encode(), C.byref(S), C.byref(W), C.byref(D),
                  C.byref(A))
        S, W, D, A = S.value, W.value, D.value, A.value
        # the header's counts against the file size before anything is
        # allocated (a corrupt header must not request a huge allocation)
        if os.path.getsize(path) < 20 + 8 * S * D + 13 * S:
            raise FormatError(f"{path}: truncated array data")
        t = np.empty((S, D), np.int32)
        e = np.empty((S, D), np.int32)
        f = np.empty(S, np.uint8)
        w, u, lb = (np.empty(S, np.int32) for _ in range(3))
        _lib.call("fb_pta1_read", path.encode(), t.ctypes.data, e.ctypes.data, f.ctypes.data,
                  w.ctypes.data, u.ctypes.data, lb.ctypes.data)
        trie = cls(t, e, f.astype(bool), w, u, lb, A)
        if trie.num_words != W:
            raise FormatError(f"{path}: header word count mismatch")
        return trie

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
    """Reference ``build_trie`` (lexicon_trie.py:227-276): word checks here (same
    FormatErrors), the sort + longest-common-prefix sweep in C++
    (``fb_trie_build``: ranks = lexicographic char-id order, states created along
    the sweep, so each parent's edges come in ascending label order)."""
    import ctypes as C
    from . import _lib
    if not vocab:
        raise FormatError("empty vocabulary")
    seen = set()
    seqs = []
    for w in vocab:
        if w in seen:
            raise FormatError(f"duplicate word {w!r} in vocabulary")
        seen.add(w)
        seqs.append(word_char_ids(w, token_dict))
    n = len(seqs)
    lens = np.fromiter((len(q) for q in seqs), np.int64, count=n)
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    chars = np.fromiter((c for q in seqs for c in q), np.int32, count=int(offs[-1]))
    A = len(token_dict)
    S, D = C.c_int32(), C.c_int32()
    _lib.call("fb_trie_build_sizes", n, chars.ctypes.data, offs.ctypes.data, A, C.byref(S),
              C.byref(D))
    S, D = S.value, D.value
    t = np.empty((S, D), np.int32)
    e = np.empty((S, D), np.int32)
    f = np.empty(S, np.uint8)
    wi, ub, lb = (np.empty(S, np.int32) for _ in range(3))
    _lib.call("fb_trie_build", n, chars.ctypes.data, offs.ctypes.data, A, S, D, t.ctypes.data,
              e.ctypes.data, f.ctypes.data, wi.ctypes.data, ub.ctypes.data, lb.ctypes.data)
    return PrefixTreeAutomaton(t, e, f.astype(bool), wi, ub, lb, A)
