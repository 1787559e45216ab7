"""MultilevelFusion on the GPU (reference fusion.py:268-380; SURVEY.md §8f
rank 4): the reference's own unit tests (test_fusion.py:240-357) restated, its
walks and decodes (tests/golden/multilevel.pkl.gz) reproduced through the
product decode_batch."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.lookahead import OracleTableLM
from oracle.subword import OracleTableCharLM, OracleUniformCharLM
from test_oracle_golden import TableScorer

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def fb():
    import paper_1909_08723_b200 as m
    return m


def _three(word_probs=None, oov_factor=-10.0):
    m = fb()
    d = m.TokenDictionary(["e", "h", "i", "r", "s"])
    trie = m.build_trie(["her", "here", "his"], d)
    ranked = trie.words(d)
    rows = {} if word_probs is None else {(): np.asarray(word_probs)}
    fus = m.MultilevelFusion(OracleUniformCharLM(len(d), d.pad_id),
                             OracleTableLM(ranked, rows, {}), trie, d, oov_factor=oov_factor)
    return m, d, fus, OracleUniformCharLM(len(d), d.pad_id).log_probs(None)


def test_known_word_adjustment():
    m, d, fus, base = _three([0.5, 0.25, 0.25])
    assert not fus.nonpositive_scores
    st = fus.start(1)
    spelled = 0.0
    for ch in "her":
        spelled += fus.char_scores(st)[0][d.index(ch)]
        st = fus.advance(st, np.array([d.index(ch)]))
    row = fus.char_scores(st)[0]
    assert math.isclose(row[d.space_id], base[d.space_id] + (math.log(0.5) - spelled),
                        rel_tol=1e-12)
    assert math.isclose(row[d.eos_id], base[d.eos_id] + (math.log(0.5) - spelled),
                        rel_tol=1e-12)


def test_adjustment_identity_uniform():
    m, d, fus, base = _three([0.5, 0.25, 0.25])
    st = fus.start(1)
    for ch in "his":
        st = fus.advance(st, np.array([d.index(ch)]))
    row = fus.char_scores(st)[0]
    want = math.log(0.25) - 3 * math.log(1 / (len(d) - 1))
    assert math.isclose(row[d.space_id] - base[d.space_id], want, rel_tol=1e-12)


@pytest.mark.parametrize("spell", ["hee", "he"])
def test_unknown_or_partial_word_gets_oov_factor(spell):
    m, d, fus, base = _three(oov_factor=-7.5)
    st = fus.start(1)
    for ch in spell:
        st = fus.advance(st, np.array([d.index(ch)]))
    row = fus.char_scores(st)[0]
    assert math.isclose(row[d.space_id] - base[d.space_id], -7.5)


def test_empty_word_diagnostic_and_history():
    m, d, fus, base = _three()
    st = fus.start(1)
    for ch in "her":
        st = fus.advance(st, np.array([d.index(ch)]))
    st = fus.advance(st, np.array([d.space_id]))
    assert math.isclose(fus.char_scores(st)[0][d.space_id], base[d.space_id])
    before = fus.diagnostics["empty_words"]
    fus.advance(st, np.array([d.space_id]))
    assert fus.diagnostics["empty_words"] == before + 1
    st = fus.start(1)
    for ch in "his":
        st = fus.advance(st, np.array([d.index(ch)]))
    st = fus.advance(st, np.array([d.space_id]))
    assert st.histories[0][-1] == "his"
    for ch in "he":
        st = fus.advance(st, np.array([d.index(ch)]))
    st = fus.advance(st, np.array([d.space_id]))
    assert st.histories[0][-1] == "<unk>"


def test_reorder():
    m, d, fus, base = _three([0.5, 0.25, 0.25])
    st = fus.start(2)
    st = fus.advance(st, np.array([d.index("h")] * 2))
    st = fus.advance(st, np.array([d.index("e"), d.index("i")]))
    rows = fus.char_scores(st)
    st2 = fus.reorder(st, [1, 0])
    np.testing.assert_array_equal(fus.char_scores(st2), rows[[1, 0]])
    np.testing.assert_array_equal(st2.trie_states, st.trie_states[[1, 0]])


def _parts(g, w, d):
    m = fb()
    trie = m.build_trie(g["words"], d)
    ranked = trie.words(d)
    lm = OracleTableLM(ranked, w["lm_rows"], {})
    clm = (OracleUniformCharLM(len(d), d.pad_id) if w.get("uniform")
           else OracleTableCharLM(w["rows"], w["default"]))
    return trie, lm, clm


def test_walks_match_reference():
    m = fb()
    g = load_golden("multilevel.pkl.gz")
    d = m.TokenDictionary(g["letters"])
    for w in g["walks"]:
        trie, lm, clm = _parts(g, w, d)
        fus = m.MultilevelFusion(clm, lm, trie, d, oov_factor=-7.5)
        st = fus.start(5)
        for step in w["walk"]:
            np.testing.assert_array_equal(st.trie_states, step["states"])
            np.testing.assert_array_equal(st.char_accum, step["accum"])
            assert fus.diagnostics["empty_words"] == step["empty"]
            np.testing.assert_allclose(fus.char_scores(st), step["scores"], rtol=1e-12,
                                       atol=1e-12)
            st = fus.reorder(fus.advance(st, step["tokens"]), step["parents"].tolist())


def test_decodes_match_reference():
    m = fb()
    g = load_golden("multilevel.pkl.gz")
    d = m.TokenDictionary(g["letters"])
    for case in g["cases"]:
        trie, lm, clm = _parts(g, case, d)
        fus = m.MultilevelFusion(clm, lm, trie, d, oov_factor=-6.0)
        feats = [m.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = m.decode_batch(feats, TableScorer(case["tables"]), fus,
                             m.DecodeConfig(**case["cfg"]), d)
        assert fus.diagnostics["empty_words"] == case["empty"]
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert abs(r.score - score) <= 1e-12 * max(1.0, abs(score))
            np.testing.assert_array_equal(np.asarray(r.attn_accum), acc)
