"""Oracle restatement of the token dictionary and the prefix-tree automaton.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``token_dict.py:19-43`` (special-token placement) and
``lexicon_trie.py:227-276`` (rank assignment by character-id tuple, DFS-free
insertion order of states, ``lb = lo - 1``) plus the derived dense child map of
``lexicon_trie.py:101-117``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

PAD, EOS, UNK, SPACE = "<pad>", "<eos>", "<unk>", "<space>"
NO_STATE = -1


class OracleDict:
    """token_dict.py:25-43: <pad>,<eos>,<unk> prepended when absent; <space> appended."""

    def __init__(self, file_tokens: Sequence[str]):
        if len(set(file_tokens)) != len(file_tokens):
            raise ValueError("duplicate token")
        present = set(file_tokens)
        toks = [s for s in (PAD, EOS, UNK) if s not in present] + list(file_tokens)
        if SPACE not in present:
            toks.append(SPACE)
        self.tokens = tuple(toks)
        self.ids = {t: i for i, t in enumerate(toks)}
        self.pad_id, self.eos_id = self.ids[PAD], self.ids[EOS]
        self.unk_id, self.space_id = self.ids[UNK], self.ids[SPACE]

    def __len__(self):
        return len(self.tokens)

    def spell(self, word: str) -> Tuple[int, ...]:
        # lexicon_trie.py:27-39: one token per character, unknown chars rejected
        if not word:
            raise ValueError("empty word")
        return tuple(self.ids[ch] for ch in word)


@dataclass
class OracleTrie:
    transitions: np.ndarray     # [S, D] int32, -1 padded (insertion order per state)
    edge_labels: np.ndarray     # [S, D] int32
    is_final: np.ndarray        # [S] bool
    word_index: np.ndarray      # [S] int32 (rank or -1)
    ub_index: np.ndarray        # [S] int32
    lb_index: np.ndarray        # [S] int32
    alphabet_size: int

    @property
    def num_states(self):
        return int(self.transitions.shape[0])

    @property
    def num_words(self):
        return int(self.is_final.sum())

    def children_dense(self) -> np.ndarray:
        """lexicon_trie.py:104-112: dense [S, alphabet] child map, -1 = no edge."""
        out = np.full((self.num_states, self.alphabet_size), NO_STATE, np.int32)
        src, slot = np.nonzero(self.transitions != NO_STATE)
        out[src, self.edge_labels[src, slot]] = self.transitions[src, slot]
        return out

    def ranked_words(self, d: OracleDict) -> List[str]:
        """Vocabulary in rank order (lexicon_trie.py:164-176), via parent links."""
        parent = np.full(self.num_states, -1, np.int64)
        pchar = np.full(self.num_states, -1, np.int64)
        src, slot = np.nonzero(self.transitions != NO_STATE)
        parent[self.transitions[src, slot]] = src
        pchar[self.transitions[src, slot]] = self.edge_labels[src, slot]
        state_of_rank = np.empty(self.num_words, np.int64)
        finals = np.nonzero(self.is_final)[0]
        state_of_rank[self.word_index[finals]] = finals
        words = []
        for s in state_of_rank:
            chars = []
            while s != 0:
                chars.append(d.tokens[pchar[s]])
                s = parent[s]
            words.append("".join(reversed(chars)))
        return words


def build_trie(vocab: Sequence[str], d: OracleDict) -> OracleTrie:
    """lexicon_trie.py:227-276 restated: insert words in rank order, track the
    first/last rank through every state, then pack per-state edge slots in
    first-insertion order."""
    if not vocab:
        raise ValueError("empty vocabulary")
    if len(set(vocab)) != len(vocab):
        raise ValueError("duplicate word")
    seqs = sorted(d.spell(w) for w in vocab)
    kids: List[Dict[int, int]] = [dict()]
    first = [0]
    last = [0]
    rank_of = [-1]
    for r, seq in enumerate(seqs):
        last[0] = r
        s = 0
        for c in seq:
            nxt = kids[s].get(c)
            if nxt is None:
                nxt = len(kids)
                kids[s][c] = nxt
                kids.append(dict())
                first.append(r)
                last.append(r)
                rank_of.append(-1)
            else:
                last[nxt] = r
            s = nxt
        rank_of[s] = r
    S = len(kids)
    D = max(len(k) for k in kids)
    trans = np.full((S, D), NO_STATE, np.int32)
    labels = np.full((S, D), NO_STATE, np.int32)
    for s, k in enumerate(kids):
        for j, (c, t) in enumerate(k.items()):   # dict keeps insertion order
            labels[s, j] = c
            trans[s, j] = t
    rank = np.asarray(rank_of, np.int32)
    return OracleTrie(trans, labels, rank >= 0, rank,
                      np.asarray(last, np.int32),
                      np.asarray(first, np.int32) - 1, len(d))
