"""GPU parity of the search and look-ahead kernels against the oracle and the
reference golden vectors (mirrors reference test_acceptance.py criteria 01,
02, 06, 07 and test_fusion.py / test_decoder.py worked values)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.lexicon import OracleDict, build_trie as oracle_build_trie
from oracle.lookahead import OracleLookahead, OracleTableLM
from oracle.search import OracleConfig, decode_batch as oracle_decode
from test_oracle_golden import TableScorer, _Feat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def _product():
    import paper_1909_08723_b200 as fb
    return fb


def test_golden_decode_cases_match_reference():
    fb = _product()
    g = load_golden("decode.pkl.gz")
    d = fb.TokenDictionary(g["letters"])
    trie = fb.build_trie(g["words"], d)
    ranked = trie.words(d)
    for k, case in enumerate(g["cases"]):
        fus = None
        if case["fused"]:
            fus = fb.LookaheadFusion(trie, OracleTableLM(ranked, case["lm_rows"], case["lm_eos"]), d)
        feats = [fb.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = fb.decode_batch(feats, TableScorer(case["tables"]), fus,
                              fb.DecodeConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert r.utt_id == uid
            assert r.tokens == toks, (k, uid)
            assert (r.finished, r.steps) == (fin, steps), (k, uid)
            if case["fused"]:
                assert abs(r.score - score) <= 1e-12 * max(1.0, abs(score)), (k, uid)
            else:
                assert r.score == score, (k, uid)           # pure fp64 adds: bit-exact
            np.testing.assert_array_equal(r.attn_accum, acc)


def _rand_table(rng, V, pad, eos, uid, t_enc, quantized):
    def dist():
        if quantized:
            raw = rng.choice([1.0, 2.0, 4.0], size=V)
            return raw / raw.sum()
        return rng.dirichlet(np.ones(V))
    rows = {}
    frontier = [()]
    prefixes = [()]
    for _ in range(2):
        frontier = [p + (t,) for p in frontier for t in range(V) if t not in (pad, eos)]
        prefixes += frontier
    for p in prefixes:
        rows[p] = (np.log(dist()), rng.dirichlet(np.ones(t_enc)))
    return (t_enc, rows, (np.log(dist()), rng.dirichlet(np.ones(t_enc))))


@pytest.mark.parametrize("seed", range(6))
def test_random_batches_match_oracle(seed):
    """Batched decode of random tables with ties, all coverage/gate/fusion modes."""
    fb = _product()
    rng = np.random.default_rng(1000 + seed)
    letters = ["a", "b", "c", "d"]
    words = ["a", "ab", "abc", "b", "ba", "bad", "c", "cab", "d", "dab"]
    d = fb.TokenDictionary(letters)
    od = OracleDict(letters)
    trie = fb.build_trie(words, d)
    otrie = oracle_build_trie(words, od)
    ranked = trie.words(d)
    V = len(d)
    for mode in range(6):
        tables = {f"u{i}": _rand_table(rng, V, d.pad_id, d.eos_id, f"u{i}",
                                       int(rng.integers(2, 9)), bool(i % 2))
                  for i in range(int(rng.integers(1, 7)))}
        cfg = dict(beam_size=int(rng.integers(1, 12)),
                   lm_weight=[0.0, 0.4, 0.9, 0.0, 0.6, 0.3][mode],
                   coverage_mode=["off", "improved", "original", "improved", "off", "improved"][mode],
                   coverage_weight=0.05, tau1=0.3, tau2=0.8, cov_margin=0.7,
                   eos_gamma=[None, 1.5, None, 1.2, 1.5, None][mode],
                   max_len_ratio=float(rng.choice([0.5, 1.0, 2.0])))
        lm_rows = {(): rng.dirichlet(np.ones(len(ranked)))}
        fused = cfg["lm_weight"] > 0
        fus = fb.LookaheadFusion(trie, OracleTableLM(ranked, lm_rows, {(): 0.1}), d) if fused else None
        ofus = OracleLookahead(otrie, OracleTableLM(ranked, lm_rows, {(): 0.1}), od) if fused else None
        feats = [fb.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in tables]
        got = fb.decode_batch(feats, TableScorer(tables), fus, fb.DecodeConfig(**cfg), d)
        want = oracle_decode([_Feat(u, np.zeros((1, 1))) for u in tables], TableScorer(tables),
                             ofus, OracleConfig(**cfg), od)
        for a, b in zip(got, want):
            assert a.tokens == b.tokens, (mode, a.utt_id)
            assert (a.finished, a.steps) == (b.finished, b.steps)
            assert abs(a.score - b.score) <= 1e-12 * max(1.0, abs(b.score))
            np.testing.assert_allclose(a.attn_accum, b.attn_accum, rtol=0, atol=1e-15)


def test_lookahead_walks_match_reference():
    fb = _product()
    for case in load_golden("lookahead.pkl.gz"):
        d = fb.TokenDictionary(case["letters"])
        trie = fb.build_trie(case["words"], d)
        lm = OracleTableLM(trie.words(d), case["rows"], case["eos"])
        fus = fb.LookaheadFusion(trie, lm, d)
        st = fus.start(6)
        for w in case["walk"]:
            np.testing.assert_array_equal(st.trie_states, w["states"])   # bit-exact trie
            np.testing.assert_allclose(st.g, w["g"], rtol=1e-14, atol=1e-15)
            sc = fus.char_scores(st)
            fin = np.isfinite(w["scores"])
            assert (np.isfinite(sc) == fin).all()
            np.testing.assert_allclose(sc[fin], w["scores"][fin], rtol=1e-12, atol=1e-12)
            assert fus.diagnostics["floored_scores"] == w["floored"]
            st = fus.advance(st, w["tokens"])
            st = fus.reorder(st, w["parents"])


def test_lookahead_worked_values():
    fb = _product()
    d = fb.TokenDictionary(["e", "h", "i", "r", "s"])
    trie = fb.build_trie(["her", "here", "his"], d)
    ranked = trie.words(d)
    fus = fb.LookaheadFusion(trie, OracleTableLM(ranked), d)
    st = fus.start(1)
    assert math.isclose(math.exp(fus.char_scores(st)[0, d.index("h")]), 1.0)
    st = fus.advance(st, [d.index("h")])
    row = fus.char_scores(st)[0]
    assert math.isclose(math.exp(row[d.index("e")]), 2 / 3)
    assert math.isclose(math.exp(row[d.index("i")]), 1 / 3)
    for ch in "er":
        st = fus.advance(st, [d.index(ch)])
    row = fus.char_scores(st)[0]
    assert math.isclose(math.exp(row[d.space_id]), 0.5)
    assert math.isclose(math.exp(row[d.index("e")]), 0.5)
    st = fus.advance(st, [d.space_id])
    assert st.trie_states[0] == 0 and st.histories[0][-1] == "her"
    st2 = fus.advance(fus.advance(fus.start(1), [d.index("h")]), [d.index("s")])
    assert st2.trie_states[0] == fb.OOV_STATE
    assert (fus.char_scores(st2) == fb.DEFAULT_OOV_PENALTY).all()
    with pytest.raises(ValueError):
        fus.advance(st2, [1, 2])


def test_criterion_01_lookahead_vs_brute_force():
    """Look-ahead == direct summation over V within 1e-9 relative."""
    fb = _product()
    rng = np.random.default_rng(101)
    for _ in range(30):
        alphabet = int(rng.integers(2, 11))
        letters = list("abcdefghij"[:alphabet])
        words = sorted({"".join(rng.choice(letters, size=int(rng.integers(1, 7))))
                        for _ in range(int(rng.integers(2, 150)))})
        d = fb.TokenDictionary(letters)
        trie = fb.build_trie(words, d)
        ranked = trie.words(d)
        probs = rng.dirichlet(np.ones(len(ranked)))
        fus = fb.LookaheadFusion(trie, OracleTableLM(ranked, {(): probs}), d)
        prefixes = [""] + [w[:int(rng.integers(0, len(w) + 1))] for w in rng.choice(ranked, 7)]
        st = fus.start(len(prefixes))
        states = [trie.state_of_prefix([d.index(c) for c in p]) for p in prefixes]
        st.states_dev.copy_(torch.as_tensor(np.asarray(states, np.int32)))
        rows = fus.char_scores(st)
        for b, p in enumerate(prefixes):
            den = sum(q for w, q in zip(ranked, probs) if w.startswith(p))
            for c in letters:
                num = sum(q for w, q in zip(ranked, probs) if w.startswith(p + c))
                if trie.child(states[b], d.index(c)) >= 0:
                    assert abs(math.exp(rows[b, d.index(c)]) - num / den) <= 1e-9 * num / den
            if p in ranked:
                want = probs[ranked.index(p)] / den
                assert abs(math.exp(rows[b, d.space_id]) - want) <= 1e-9 * want


def test_coverage_and_gate_helpers():
    fb = _product()
    acc = np.array([0.6, 1.2, 0.3])
    assert fb.coverage_original(acc, 0.5) == 2
    assert fb.coverage_improved(acc, 0.5, 1.0, 0.7) == 1.1
    rng = np.random.default_rng(2)
    from oracle.search import cov_improved
    for _ in range(50):
        a = rng.uniform(0, 2.5, size=int(rng.integers(1, 700)))
        assert fb.coverage_improved(a, 0.5, 1.0, 0.7) == cov_improved(a, 0.5, 1.0, 0.7)
    assert not fb.eos_allowed(np.array([-3.0, -1.0, -2.0, -0.5]), 1.5, 1)
    assert fb.eos_allowed(np.array([-2.0, -0.1, -1.5, -0.3]), 1.5, 1)


def test_cumsum_distribution():
    fb = _product()
    np.testing.assert_allclose(fb.cumsum_distribution(np.array([0.5, 0.25, 0.25])),
                               [0.5, 0.75, 1.0], rtol=1e-15)
    rng = np.random.default_rng(1)
    p = rng.dirichlet(np.ones(70000))
    np.testing.assert_allclose(fb.cumsum_distribution(p), np.cumsum(p), rtol=1e-12)
