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
