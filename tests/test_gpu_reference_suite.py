"""The reference's own decoder/fusion acceptance tests, run through the
product API on the GPU (test_decoder.py, test_fusion.py, test_acceptance.py of
/root/reference/pkg/tests, restated with the oracle's table fakes)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle.lookahead import OracleTableLM
from test_oracle_golden import TableScorer

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def fb():
    import paper_1909_08723_b200 as m
    return m


def rand_table(rng, V, pad, eos, t_enc, depth=2, quantized=False):
    def dist():
        if quantized:
            raw = rng.choice([1.0, 2.0, 4.0], size=V)
            return raw / raw.sum()
        return rng.dirichlet(np.ones(V))
    rows, frontier, prefixes = {}, [()], [()]
    for _ in range(depth):
        frontier = [p + (t,) for p in frontier for t in range(V) if t not in (pad, eos)]
        prefixes += frontier
    for p in prefixes:
        rows[p] = (np.log(dist()), rng.dirichlet(np.ones(t_enc)))
    return (t_enc, rows, (np.log(dist()), rng.dirichlet(np.ones(t_enc))))


def decode_one(table, cfg, fusion=None, d=None):
    m = fb()
    d = d or m.TokenDictionary(["a", "b"])
    feats = [m.FeatureMatrix("u", np.zeros((table[0], 2), np.float32))]
    return m.decode_batch(feats, TableScorer({"u": table}), fusion, cfg, d)[0]


def exhaustive(table, d, cfg, fusion=None):
    """conftest.py:149-207 restated: best (tokens, total, finished) over all sequences."""
    from oracle.search import cov_improved, cov_original
    t_enc, rows, default = table
    V = len(d)
    max_len = max(1, int(math.floor(cfg.max_len_ratio * t_enc)))
    fin, live = [], []

    def cov(acc):
        if cfg.coverage_mode == "original":
            return cov_original(acc, cfg.tau1)
        if cfg.coverage_mode == "improved":
            return cov_improved(acc, cfg.tau1, cfg.tau2, cfg.cov_margin)
        return 0.0

    def rec(prefix, base, acc, fst):
        logp, attn = rows.get(prefix, default)
        frow = fusion.char_scores(fst)[0] if fusion is not None else None
        for tok in range(V):
            if tok == d.pad_id:
                continue
            if tok == d.eos_id and cfg.eos_gamma is not None and \
                    logp[d.eos_id] <= cfg.eos_gamma * float(logp.max()):
                continue
            step = float(logp[tok])
            if frow is not None:
                step = step + cfg.lm_weight * frow[tok]
            nb = base + step
            na = acc + attn
            tot = nb + cfg.coverage_weight * cov(na) if cfg.coverage_mode != "off" else nb
            seq = prefix + (tok,)
            if tok == d.eos_id:
                fin.append((tot, len(seq), seq))
            elif len(seq) >= max_len:
                live.append((tot, len(seq), seq))
            else:
                rec(seq, nb, na, fusion.advance(fst, [tok]) if fusion is not None else None)

    rec((), 0.0, np.zeros(t_enc), fusion.start(1) if fusion is not None else None)
    pool = fin if fin else live
    tot, _, seq = min(pool, key=lambda e: (-e[0], e[1], e[2]))
    toks = list(seq)
    if toks and toks[-1] == d.eos_id:
        toks.pop()
    return toks, tot, bool(fin)


# ---- test_decoder.py ---------------------------------------------------------
def test_tie_break_prefers_lower_token_id():
    m = fb()
    V = len(m.TokenDictionary(["a", "b"]))
    uni = np.log(np.full(V, 1.0 / V))
    res = decode_one((2, {(): (uni, np.full(2, 0.5))}, (uni, np.full(2, 0.5))),
                     m.DecodeConfig(beam_size=3))
    assert res.tokens == [] and res.finished


def test_pad_never_selected():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    p = np.full(len(d), 1e-6)
    p[d.pad_id] = 1.0 - 1e-6 * (len(d) - 1)
    t = (2, {(): (np.log(p), np.full(2, 0.5))}, (np.log(p), np.full(2, 0.5)))
    assert d.pad_id not in decode_one(t, m.DecodeConfig(beam_size=4)).tokens


def test_length_bound_and_unfinished_fallback():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    V = len(d)
    p = np.full(V, 1e-9)
    p[d.index("a")] = 1.0 - 1e-9 * (V - 1)
    t = (3, {}, (np.log(p), np.full(3, 1 / 3)))
    res = decode_one(t, m.DecodeConfig(beam_size=2, eos_gamma=0.5))
    assert not res.finished and res.tokens == [d.index("a")] * 3


def test_beam_one_is_greedy():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    for seed in range(5):
        rng = np.random.default_rng(seed)
        t = rand_table(rng, len(d), d.pad_id, d.eos_id, 3)
        res = decode_one(t, m.DecodeConfig(beam_size=1))
        toks, prefix = [], ()
        for _ in range(3):
            logp = t[1].get(prefix, t[2])[0].copy()
            logp[d.pad_id] = -np.inf
            tok = int(np.argmax(logp))
            if tok == d.eos_id:
                break
            toks.append(tok)
            prefix += (tok,)
        assert res.tokens == toks


def test_monotone_beam_score():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    for seed in range(8):
        rng = np.random.default_rng(seed)
        t = rand_table(rng, len(d), d.pad_id, d.eos_id, 3)
        res = [decode_one(t, m.DecodeConfig(beam_size=b)) for b in (1, 2, 4, 8, 16, 125)]
        fin = [r.score for r in res if r.finished]
        assert all(b >= a - 1e-12 for a, b in zip(fin, fin[1:]))
        flags = [r.finished for r in res]
        assert flags == sorted(flags)


def test_attention_accumulator_replay():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    rng = np.random.default_rng(10)
    t = rand_table(rng, len(d), d.pad_id, d.eos_id, 5)
    res = decode_one(t, m.DecodeConfig(beam_size=4))
    acc = np.zeros(5)
    for i in range(len(res.tokens) + (1 if res.finished else 0)):
        acc = acc + t[1].get(tuple(res.tokens[:i]), t[2])[1]
    np.testing.assert_allclose(res.attn_accum, acc, atol=1e-12)


def test_zero_lm_weight_equals_no_fusion():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    trie = m.build_trie(["a", "ab", "b"], d)
    rng = np.random.default_rng(8)
    t = rand_table(rng, len(d), d.pad_id, d.eos_id, 3)
    plain = decode_one(t, m.DecodeConfig(beam_size=4), d=d)
    fused = decode_one(t, m.DecodeConfig(beam_size=4, lm_weight=0.0),
                       fusion=m.LookaheadFusion(trie, OracleTableLM(trie.words(d)), d), d=d)
    assert plain.tokens == fused.tokens and plain.score == fused.score


def test_config_and_input_validation():
    m = fb()
    d = m.TokenDictionary(["a", "b"])
    for bad in (dict(beam_size=0), dict(lm_weight=-0.1), dict(coverage_mode="bogus"),
                dict(coverage_mode="improved", tau1=1.0, tau2=0.5), dict(max_len_ratio=0.0),
                dict(eos_gamma=-1.0)):
        with pytest.raises(m.ConfigError):
            m.DecodeConfig(**bad).validate()
    with pytest.raises(m.ConfigError, match="empty"):
        m.decode_batch([m.FeatureMatrix("u", np.zeros((0, 2), np.float32))],
                       TableScorer({}), None, m.DecodeConfig(), d)
    with pytest.raises(m.ConfigError):
        m.decode_corpus([], TableScorer({}), None, m.DecodeConfig(), d, batch_size=0)


# ---- test_acceptance.py criterion 06 / test_decoder exhaustive -----------------
def test_saturating_beam_equals_exhaustive_search():
    m = fb()
    rng = np.random.default_rng(606)
    d = m.TokenDictionary(["a", "b"])
    trie = m.build_trie(["a", "ab", "b", "ba"], d)
    ranked = trie.words(d)
    for i in range(24):
        t = rand_table(rng, len(d), d.pad_id, d.eos_id, int(rng.integers(2, 6)),
                       quantized=bool(i % 2))
        mode = i % 4
        fus = ofus = None
        lw = 0.0
        if mode == 3:
            probs = rng.dirichlet(np.ones(len(ranked)))
            fus = m.LookaheadFusion(trie, OracleTableLM(ranked, {(): probs}), d)
            ofus = m.LookaheadFusion(trie, OracleTableLM(ranked, {(): probs}), d)
            lw = 0.9
        cfg = m.DecodeConfig(beam_size=1024, lm_weight=lw,
                             coverage_mode=["off", "original", "improved", "improved"][mode],
                             coverage_weight=0.05, tau1=0.4, tau2=0.9, cov_margin=0.7,
                             eos_gamma=1.5 if mode in (2, 3) else None)
        res = decode_one(t, cfg, fusion=fus, d=d)
        toks, tot, fin = exhaustive(t, d, cfg, fusion=ofus)
        assert res.tokens == toks, i
        assert abs(res.score - tot) <= 1e-12 * max(1.0, abs(tot)), i
        assert res.finished == fin, i


# ---- test_acceptance.py criterion 02 / 07 --------------------------------------
def test_normalization_and_telescoping():
    m = fb()
    rng = np.random.default_rng(202)
    letters = list("abcdefgh")
    words = sorted({"".join(rng.choice(letters, size=int(rng.integers(1, 7))))
                    for _ in range(160)})
    d = m.TokenDictionary(letters)
    trie = m.build_trie(words, d)
    ranked = trie.words(d)
    probs = rng.dirichlet(np.ones(len(ranked)))
    fus = m.LookaheadFusion(trie, OracleTableLM(ranked, {(): probs}), d)
    n = trie.num_states
    st = fus.start(n)
    st.states_dev.copy_(torch.arange(n, dtype=torch.int32))
    rows = fus.char_scores(st)
    kids = trie.char_children
    for s in range(n):
        mass = sum(math.exp(rows[s, c]) for c in range(len(d)) if kids[s, c] >= 0)
        if trie.is_final[s]:
            mass += math.exp(rows[s, d.space_id])
        assert abs(mass - 1.0) <= 1e-6
    for r, w in enumerate(ranked):
        s, acc = 0, 0.0
        for ch in w:
            acc += rows[s, d.index(ch)]
            s = kids[s, d.index(ch)]
        acc += rows[s, d.space_id]
        assert abs(acc - math.log(probs[r])) <= 1e-9


def test_batched_decode_equals_sequential():
    m = fb()
    rng = np.random.default_rng(707)
    d = m.TokenDictionary(["a", "b", "c"])
    trie = m.build_trie(["a", "ab", "abc", "b", "bc", "ca"], d)
    ranked = trie.words(d)
    probs = rng.dirichlet(np.ones(len(ranked)))
    tables = {f"utt{i:02d}": rand_table(rng, len(d), d.pad_id, d.eos_id, int(rng.integers(2, 7)))
              for i in range(16)}
    feats = [m.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in tables]
    cfg = m.DecodeConfig(beam_size=8, lm_weight=0.7)
    fac = lambda: m.LookaheadFusion(trie, OracleTableLM(ranked, {(): probs}), d)  # noqa: E731
    batched = m.decode_corpus(feats, TableScorer(tables), fac, cfg, d, batch_size=16)
    singles = [m.decode_batch([f], TableScorer(tables), fac(), cfg, d)[0] for f in feats]
    for a, b in zip(batched, singles):
        assert a.utt_id == b.utt_id and a.tokens == b.tokens
        assert abs(a.score - b.score) <= 1e-9
