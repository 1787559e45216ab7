"""Product trie build + CSR pack == reference build_trie arrays (CPU)."""

import numpy as np

from conftest import load_golden
from paper_1909_08723_b200.lexicon_trie import NO_STATE, build_trie
from paper_1909_08723_b200.token_dict import TokenDictionary


def test_build_matches_reference_arrays():
    for case in load_golden("trie.pkl.gz"):
        d = TokenDictionary(case["letters"])
        t = build_trie(case["words"], d)
        np.testing.assert_array_equal(t.transitions, case["transitions"])
        np.testing.assert_array_equal(t.edge_labels, case["edge_labels"])
        np.testing.assert_array_equal(t.is_final, case["is_final"])
        np.testing.assert_array_equal(t.word_index, case["word_index"])
        np.testing.assert_array_equal(t.ub_index, case["ub"])
        np.testing.assert_array_equal(t.lb_index, case["lb"])
        np.testing.assert_array_equal(t.char_children, case["children"])
        assert t.words(d) == case["ranked"]


def test_csr_is_the_dense_child_map():
    for case in load_golden("trie.pkl.gz")[:15]:
        d = TokenDictionary(case["letters"])
        t = build_trie(case["words"], d)
        row_ptr, lab, kid, info = t.csr()
        dense = case["children"]
        for s in range(t.num_states):
            a, b = row_ptr[s], row_ptr[s + 1]
            assert (np.diff(lab[a:b]) > 0).all()
            want = {c: dense[s, c] for c in range(dense.shape[1]) if dense[s, c] != NO_STATE}
            assert dict(zip(lab[a:b].tolist(), kid[a:b].tolist())) == want
            for c in range(dense.shape[1]):
                assert t.child(s, c) == dense[s, c]
        np.testing.assert_array_equal(info[:, 0], case["ub"])
        np.testing.assert_array_equal(info[:, 1], case["lb"])
        np.testing.assert_array_equal(info[:, 2], np.where(case["is_final"], case["word_index"], -1))


def test_validation_matches_reference_errors():
    """Corrupted automata: same exception and message as the reference
    constructor (lexicon_trie.py:64-129), incl. an unreachable cycle."""
    import pytest
    from paper_1909_08723_b200.errors import FormatError
    from paper_1909_08723_b200.lexicon_trie import PrefixTreeAutomaton
    g = load_golden("trie_api.pkl.gz")
    assert len(g["errors"]) > 50
    for name, a, etype, msg in g["errors"]:
        assert etype == "FormatError", name
        with pytest.raises(FormatError) as ei:
            PrefixTreeAutomaton(**a)
        assert str(ei.value) == msg, (name, str(ei.value), msg)


def test_host_api_matches_reference():
    """advance / bounds (incl. their ValueErrors), spell, parent arrays,
    final_state_of_rank and the dense child map (lexicon_trie.py:101-176)."""
    import pytest
    from paper_1909_08723_b200.lexicon_trie import PrefixTreeAutomaton
    for arrs, rec in load_golden("trie_api.pkl.gz")["api"]:
        t = PrefixTreeAutomaton(**arrs)
        np.testing.assert_array_equal(t.advance(rec["states"], rec["chars"]), rec["advance"])
        ub, lb = t.bounds(rec["states"])
        np.testing.assert_array_equal(ub, rec["bounds"][0])
        np.testing.assert_array_equal(lb, rec["bounds"][1])
        assert [t.spell(r) for r in range(t.num_words)] == rec["spell"]
        np.testing.assert_array_equal(t.parent_state, rec["parent_state"])
        np.testing.assert_array_equal(t.parent_char, rec["parent_char"])
        np.testing.assert_array_equal(t.final_state_of_rank, rec["final_state_of_rank"])
        np.testing.assert_array_equal(t.char_children, rec["char_children"])
        for fn, args, etype, msg in rec["errors"]:
            if etype is None:
                continue
            with pytest.raises(ValueError) as ei:
                getattr(t, fn)(*args) if isinstance(args, tuple) else getattr(t, fn)(args)
            assert etype == "ValueError" and str(ei.value) == msg


def test_pta1_header_checked_before_allocation(tmp_path):
    """A header claiming a huge automaton in a short file is a FormatError
    (not a MemoryError from the allocation)."""
    import struct
    import pytest
    from paper_1909_08723_b200.errors import FormatError
    from paper_1909_08723_b200.lexicon_trie import PrefixTreeAutomaton
    p = tmp_path / "big.pta1"
    p.write_bytes(b"PTA1" + struct.pack("<4i", 2 ** 30, 5, 2 ** 20, 52) + b"\0" * 64)
    with pytest.raises(FormatError, match="truncated array data"):
        PrefixTreeAutomaton.load(str(p))
