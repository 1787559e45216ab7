"""Pin the CPU oracle against reference-generated golden vectors and the
reference's own worked values.  CPU only."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.lexicon import OracleDict, build_trie
from oracle.lookahead import OOV_PENALTY, OOV_STATE, OracleLookahead, OracleTableLM
from oracle.search import (OracleConfig, cov_improved, cov_original, decode_batch,
                           eos_ok)


class _Feat:
    def __init__(self, uid, data):
        self.utt_id, self.data = uid, data


class TableScorer:
    """In-memory acoustic table keyed by token prefix (decoder.py:146-207 semantics)."""

    def __init__(self, tables):
        self.tables = tables            # uid -> (t_enc, rows, default)

    def init(self, f):
        return (f.utt_id, [()])

    def enc_length(self, st):
        return self.tables[st[0]][0]

    def step(self, st, last):
        uid, prefixes = st
        t_enc, rows, default = self.tables[uid]
        new = [p + (int(t),) if t >= 0 else p for p, t in zip(prefixes, last)]
        got = [rows.get(p, default) for p in new]
        return (np.stack([g[0] for g in got]), np.stack([g[1] for g in got]), (uid, new))

    def reorder(self, st, parents):
        return (st[0], [st[1][i] for i in parents])


def test_trie_matches_reference_build():
    for case in load_golden("trie.pkl.gz"):
        d = OracleDict(case["letters"])
        t = build_trie(case["words"], d)
        np.testing.assert_array_equal(t.transitions, case["transitions"])
        np.testing.assert_array_equal(t.edge_labels, case["edge_labels"])
        np.testing.assert_array_equal(t.is_final, case["is_final"])
        np.testing.assert_array_equal(t.word_index, case["word_index"])
        np.testing.assert_array_equal(t.ub_index, case["ub"])
        np.testing.assert_array_equal(t.lb_index, case["lb"])
        np.testing.assert_array_equal(t.children_dense(), case["children"])
        assert t.ranked_words(d) == case["ranked"]


def test_trie_worked_bounds():
    # test_lexicon_trie.py:18-34
    d = OracleDict(["e", "h", "i", "r", "s"])
    t = build_trie(["her", "here", "his"], d)
    assert t.num_states == 7 and t.num_words == 3
    kids = t.children_dense()
    cases = {"hi": (2, 1), "": (2, -1), "her": (1, -1), "here": (1, 0),
             "his": (2, 1), "h": (2, -1), "he": (1, -1)}
    for prefix, (ub, lb) in cases.items():
        s = 0
        for ch in prefix:
            s = kids[s, d.ids[ch]]
        assert (t.ub_index[s], t.lb_index[s]) == (ub, lb)


def test_lookahead_walks_match_reference_bitwise():
    for case in load_golden("lookahead.pkl.gz"):
        d = OracleDict(case["letters"])
        t = build_trie(case["words"], d)
        lm = OracleTableLM(t.ranked_words(d), case["rows"], case["eos"])
        fus = OracleLookahead(t, lm, d)
        st = fus.start(6)
        for w in case["walk"]:
            np.testing.assert_array_equal(st[0], w["states"])
            assert st[2].tobytes() == w["g"].tobytes()
            sc = fus.char_scores(st)
            assert sc.tobytes() == w["scores"].tobytes()
            assert fus.floored == w["floored"]
            st = fus.advance(st, w["tokens"])
            st = fus.reorder(st, w["parents"])


def test_lookahead_worked_values():
    # test_fusion.py:51-134
    d = OracleDict(["e", "h", "i", "r", "s"])
    t = build_trie(["her", "here", "his"], d)
    ranked = t.ranked_words(d)
    fus = OracleLookahead(t, OracleTableLM(ranked), d)
    st = fus.start(1)
    assert math.isclose(math.exp(fus.char_scores(st)[0, d.ids["h"]]), 1.0)
    st = fus.advance(st, [d.ids["h"]])
    row = fus.char_scores(st)[0]
    assert math.isclose(math.exp(row[d.ids["e"]]), 2 / 3)
    assert math.isclose(math.exp(row[d.ids["i"]]), 1 / 3)
    for ch in "er":
        st = fus.advance(st, [d.ids[ch]])
    row = fus.char_scores(st)[0]
    assert math.isclose(math.exp(row[d.space_id]), 0.5)
    st2 = fus.advance(fus.advance(fus.start(1), [d.ids["h"]]), [d.ids["s"]])
    assert st2[0][0] == OOV_STATE and (fus.char_scores(st2) == OOV_PENALTY).all()
    st2 = fus.advance(st2, [d.space_id])
    assert st2[0][0] == 0 and st2[1][0][-1] == "<unk>"
    lm = OracleTableLM(ranked, {}, {("her",): 0.25})
    fus = OracleLookahead(t, lm, d)
    st = fus.start(1)
    for ch in "her":
        st = fus.advance(st, [d.ids[ch]])
    assert math.isclose(fus.char_scores(st)[0, d.eos_id], math.log(0.5) + math.log(0.25),
                        rel_tol=1e-12)


def test_coverage_and_gate_worked_values():
    # test_acceptance.py:125-146, test_decoder.py:27-60
    acc = np.array([0.6, 1.2, 0.3])
    assert cov_original(acc, 0.5) == 2
    assert cov_improved(acc, 0.5, 1.0, 0.7) == 1.1
    assert cov_improved(np.array([1.0, 0.4]), 0.5, 1.0, 0.7) == 1.0
    row = np.array([-3.0, -1.0, -2.0, -0.5])
    assert not eos_ok(row, 1.5, 1)
    assert eos_ok(np.array([-2.0, -0.1, -1.5, -0.3]), 1.5, 1)
    assert eos_ok(row, None, 1)


def test_decode_matches_reference_bitwise():
    g = load_golden("decode.pkl.gz")
    d = OracleDict(g["letters"])
    t = build_trie(g["words"], d)
    ranked = t.ranked_words(d)
    for case in g["cases"]:
        scorer = TableScorer(case["tables"])
        fus = None
        if case["fused"]:
            fus = OracleLookahead(t, OracleTableLM(ranked, case["lm_rows"], case["lm_eos"]), d)
        feats = [_Feat(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = decode_batch(feats, scorer, fus, OracleConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert r.utt_id == uid
            assert r.tokens == toks
            assert r.score == score
            assert r.finished == fin and r.steps == steps
            assert r.attn_accum.tobytes() == acc.tobytes()


def test_neural_decode_matches_reference_bitwise():
    torch = pytest.importorskip("torch")
    from oracle.neural import OracleAttnLstmScorer, OracleLstmWordLM
    from paper_1909_08723_b200 import synth
    g = load_golden("neural.pkl.gz")
    d = OracleDict(synth.wsj_token_list())
    t = build_trie(g["words"], d)
    ranked = t.ranked_words(d)
    ad = synth.AsrDims(**g["adims"])
    ld = synth.LmDims(**g["ldims"])
    W = synth.asr_weights(ad, seed=g["asr_seed"], eos_id=d.eos_id)
    W.update(synth.lm_weights(ld, seed=g["lm_seed"]))
    feats = [_Feat(u, x) for u, x in synth.synth_fbank(g["n_utts"], g["fbank_seed"],
                                                       tuple(g["frames"]))]
    for case in g["cases"]:
        sc = OracleAttnLstmScorer(W, ad.enc_layers, ad.dec_layers, ad.subsample, d.eos_id)
        lm = OracleLstmWordLM(W, ld.layers, len(ranked))
        fus = OracleLookahead(t, lm, d) if case["cfg"]["lm_weight"] > 0 else None
        res = decode_batch(feats, sc, fus, OracleConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert r.score == score
            np.testing.assert_array_equal(r.attn_accum, acc)


# ---- subword (token-level LM) fusion: fusion.py:236-266, char_lm.py:23-53 -------
def test_subword_rows_match_reference_bitwise():
    from oracle.subword import OracleSubwordFusion, OracleTableCharLM, OracleUniformCharLM
    g = load_golden("subword.pkl.gz")
    d = OracleDict(g["letters"])
    for w in g["walks"]:
        fus = OracleSubwordFusion(OracleTableCharLM(w["rows"], w["default"]))
        assert fus.nonpositive_scores
        st = fus.start(5)
        for step in w["walk"]:
            np.testing.assert_array_equal(fus.char_scores(st), step["scores"])
            st = fus.reorder(fus.advance(st, step["tokens"]), step["parents"].tolist())
    # test_fusion.py:224-237: rows are the provider's rows
    uni = OracleUniformCharLM(len(d), d.pad_id)
    fus = OracleSubwordFusion(uni)
    rows = fus.char_scores(fus.start(3))
    assert rows.shape == (3, len(d))
    assert rows[0, d.pad_id] == -30.0
    assert abs(rows[0, d.eos_id] - math.log(1.0 / (len(d) - 1))) == 0.0


def test_subword_decode_matches_reference_bitwise():
    from oracle.subword import OracleSubwordFusion, OracleTableCharLM, OracleUniformCharLM
    g = load_golden("subword.pkl.gz")
    d = OracleDict(g["letters"])
    for case in g["cases"]:
        lm = (OracleUniformCharLM(len(d), d.pad_id) if case["uniform"]
              else OracleTableCharLM(case["rows"], case["default"]))
        feats = [_Feat(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = decode_batch(feats, TableScorer(case["tables"]), OracleSubwordFusion(lm),
                           OracleConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert r.score == score
            assert r.attn_accum.tobytes() == acc.tobytes()


def test_subword_neural_decode_matches_reference_bitwise():
    pytest.importorskip("torch")
    from oracle.neural import OracleAttnLstmScorer
    from oracle.subword import OracleLstmCharLM, OracleSubwordFusion
    from paper_1909_08723_b200 import synth
    g = load_golden("subword.pkl.gz")["neural"]
    d = OracleDict(g["tokens"])
    ad = synth.AsrDims(**g["adims"])
    sdm = synth.SubwordLmDims(**g["sdims"])
    W = synth.asr_weights(ad, seed=g["asr_seed"], eos_id=d.eos_id)
    W.update(synth.subword_lm_weights(sdm, seed=g["lm_seed"], eos_id=d.eos_id))
    feats = [_Feat(u, x) for u, x in synth.synth_fbank(g["n_utts"], g["fbank_seed"],
                                                       tuple(g["frames"]))]
    for case in g["cases"]:
        sc = OracleAttnLstmScorer(W, ad.enc_layers, ad.dec_layers, ad.subsample, d.eos_id)
        lm = OracleLstmCharLM(W, sdm.layers, d.pad_id, d.eos_id)
        res = decode_batch(feats, sc, OracleSubwordFusion(lm, batched=False),
                           OracleConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert r.score == score
            np.testing.assert_array_equal(r.attn_accum, acc)
        # the batched advance (used at real sizes) agrees to fp32 rounding
        lm2 = OracleLstmCharLM(W, sdm.layers, d.pad_id, d.eos_id)
        s0 = lm2.start()
        toks = [3, 7, d.eos_id, 11]
        many = lm2.advance_many([s0] * 4, toks)
        for s, t in zip(many, toks):
            np.testing.assert_allclose(s.row, lm2.advance(s0, t).row, rtol=0, atol=1e-5)


# ---- multilevel fusion: fusion.py:268-380 ------------------------------------------
def _ml_parts(g, walk_or_case, d):
    from oracle.lookahead import OracleTableLM
    from oracle.subword import OracleTableCharLM, OracleUniformCharLM
    t = build_trie(g["words"], d)
    ranked = t.ranked_words(d)
    lm = OracleTableLM(ranked, walk_or_case["lm_rows"], {})
    if walk_or_case.get("uniform"):
        clm = OracleUniformCharLM(len(d), d.pad_id)
    else:
        clm = OracleTableCharLM(walk_or_case["rows"], walk_or_case["default"])
    return t, lm, clm


def test_multilevel_walks_match_reference_bitwise():
    from oracle.subword import OracleMultilevelFusion
    g = load_golden("multilevel.pkl.gz")
    d = OracleDict(g["letters"])
    for w in g["walks"]:
        t, lm, clm = _ml_parts(g, w, d)
        fus = OracleMultilevelFusion(clm, lm, t, d, oov_factor=-7.5)
        assert not fus.nonpositive_scores
        st = fus.start(5)
        for step in w["walk"]:
            np.testing.assert_array_equal(st.trie_states, step["states"])
            np.testing.assert_array_equal(st.char_accum, step["accum"])
            assert fus.diagnostics["empty_words"] == step["empty"]
            np.testing.assert_array_equal(fus.char_scores(st), step["scores"])
            st = fus.reorder(fus.advance(st, step["tokens"]), step["parents"].tolist())


def test_multilevel_decode_matches_reference_bitwise():
    from oracle.subword import OracleMultilevelFusion
    g = load_golden("multilevel.pkl.gz")
    d = OracleDict(g["letters"])
    for case in g["cases"]:
        t, lm, clm = _ml_parts(g, case, d)
        fus = OracleMultilevelFusion(clm, lm, t, d, oov_factor=-6.0)
        feats = [_Feat(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = decode_batch(feats, TableScorer(case["tables"]), fus, OracleConfig(**case["cfg"]), d)
        assert fus.diagnostics["empty_words"] == case["empty"]
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert r.score == score
            assert r.attn_accum.tobytes() == acc.tobytes()
