"""Golden fixtures for the automaton's validation and host API, produced by the
UNMODIFIED reference (run in the build container):

    python tests/golden/make_trie_errors.py

* corrupted automata (each invariant of lexicon_trie.py:64-129 broken in
  turn, plus a cycle that is unreachable from the root) and the exception
  type and message the reference constructor raises;
* on valid automata, the reference's advance / bounds (incl. their
  ValueErrors), spell, parent_state, parent_char, final_state_of_rank and
  char_children (lexicon_trie.py:101-176).

Writes ``tests/golden/trie_api.pkl.gz``; ``tests/test_trie_pack.py`` replays
it against ``paper_1909_08723_b200.lexicon_trie`` on the CPU.
"""

from __future__ import annotations

import gzip
import os
import pickle
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fusedbeam.lexicon_trie import PrefixTreeAutomaton, build_trie  # noqa: E402
from fusedbeam.token_dict import TokenDictionary  # noqa: E402


def arrays(t):
    return dict(transitions=t.transitions.copy(), edge_labels=t.edge_labels.copy(),
                is_final=t.is_final.copy(), word_index=t.word_index.copy(),
                ub_index=t.ub_index.copy(), lb_index=t.lb_index.copy(),
                alphabet_size=t.alphabet_size)


def outcome(a):
    try:
        PrefixTreeAutomaton(**a)
    except Exception as e:          # noqa: BLE001 - we record whatever the reference raises
        return type(e).__name__, str(e)
    return None, None


def corruptions(base):
    """(name, arrays) pairs, each breaking one invariant."""
    out = []

    def mut(name, fn):
        a = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
        fn(a)
        out.append((name, a))

    live = np.argwhere(base["transitions"] != -1)
    dead = np.argwhere(base["transitions"] == -1)
    s0, k0 = live[len(live) // 2]
    mut("no_slots", lambda a: a.update(transitions=a["transitions"][:, :0],
                                       edge_labels=a["edge_labels"][:, :0]))
    mut("shape", lambda a: a.update(ub_index=a["ub_index"][:-1]))
    mut("target_root", lambda a: a["transitions"].__setitem__((s0, k0), 0))
    mut("target_big", lambda a: a["transitions"].__setitem__((s0, k0), 10 ** 6))
    mut("label_neg", lambda a: a["edge_labels"].__setitem__((s0, k0), -3))
    mut("label_big", lambda a: a["edge_labels"].__setitem__((s0, k0), a["alphabet_size"]))
    if len(dead):
        s1, k1 = dead[0]
        mut("dead_slot_label", lambda a: a["edge_labels"].__setitem__((s1, k1), 2))
        mut("two_parents", lambda a: (a["transitions"].__setitem__((s1, k1), int(a["transitions"][s0, k0])),
                                      a["edge_labels"].__setitem__((s1, k1), 1)))
    mut("orphan", lambda a: (a["transitions"].__setitem__((s0, k0), -1),
                             a["edge_labels"].__setitem__((s0, k0), -1)))
    fin = np.nonzero(base["is_final"])[0]
    mut("rank_dup", lambda a: a["word_index"].__setitem__(fin[-1], a["word_index"][fin[0]]))
    nonfin = np.nonzero(~base["is_final"])[0]
    mut("nonfinal_rank", lambda a: a["word_index"].__setitem__(nonfin[-1], 0))
    mut("ub_big", lambda a: a["ub_index"].__setitem__(1, len(fin)))
    mut("ub_neg", lambda a: a["ub_index"].__setitem__(1, -1))
    mut("lb_low", lambda a: a["lb_index"].__setitem__(1, -2))
    mut("lb_above_ub", lambda a: a["lb_index"].__setitem__(1, int(a["ub_index"][1]) + 1))
    mut("no_words", lambda a: (a["is_final"].__setitem__(slice(None), False),
                               a["word_index"].__setitem__(slice(None), -1)))
    return out


def cycle_case():
    """Root -> 1 (final 'a'); states 2 <-> 3 parent each other: one parent
    each, but unreachable from the root."""
    t = np.array([[1], [-1], [3], [2]], np.int32)
    e = np.array([[0], [-1], [1], [1]], np.int32)
    return dict(transitions=t, edge_labels=e, is_final=np.array([False, True, False, False]),
                word_index=np.array([-1, 0, -1, -1], np.int32),
                ub_index=np.zeros(4, np.int32), lb_index=np.array([-1, -1, -1, -1], np.int32),
                alphabet_size=4)


def api_case(trie, rng):
    S, A, W = trie.num_states, trie.alphabet_size, trie.num_words
    st = rng.integers(0, S, size=64)
    ch = rng.integers(0, A, size=64)
    rec = dict(states=st, chars=ch, advance=trie.advance(st, ch), bounds=trie.bounds(st),
               spell=[trie.spell(r) for r in range(W)], parent_state=trie.parent_state.copy(),
               parent_char=trie.parent_char.copy(),
               final_state_of_rank=trie.final_state_of_rank.copy(),
               char_children=trie.char_children.copy(), errors=[])
    for args in ((np.array([0, 1]), np.array([0])), (np.array([-1]), np.array([0])),
                 (np.array([S]), np.array([0])), (np.array([0]), np.array([A]))):
        try:
            trie.advance(*args)
            rec["errors"].append(("advance", args, None, None))
        except Exception as e:      # noqa: BLE001
            rec["errors"].append(("advance", args, type(e).__name__, str(e)))
    for args in (np.array([-2]), np.array([S])):
        try:
            trie.bounds(args)
            rec["errors"].append(("bounds", args, None, None))
        except Exception as e:      # noqa: BLE001
            rec["errors"].append(("bounds", args, type(e).__name__, str(e)))
    return rec


def main():
    rng = np.random.default_rng(2024)
    d = TokenDictionary(list("ehirs"))
    tries = [build_trie(["her", "here", "his"], d)]
    letters = list("abcdefgh")
    d2 = TokenDictionary(letters)
    for _ in range(4):
        n = int(rng.integers(5, 60))
        words = sorted({"".join(rng.choice(letters, size=int(rng.integers(1, 7))))
                        for _ in range(n)})
        tries.append(build_trie(words, d2))
    errs = []
    for t in tries:
        for name, a in corruptions(arrays(t)):
            errs.append((name, a, *outcome(a)))
    c = cycle_case()
    errs.append(("cycle", c, *outcome(c)))
    api = [(arrays(t), api_case(t, rng)) for t in tries]
    with gzip.open(os.path.join(HERE, "trie_api.pkl.gz"), "wb") as f:
        pickle.dump({"errors": errs, "api": api}, f, protocol=4)
    print(len(errs), "corruptions;", sorted({(n, m) for n, _, _, m in errs if m})[:40])


if __name__ == "__main__":
    main()
