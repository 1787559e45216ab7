"""Plain token-level LM fusion (SubwordFusion, config 4; reference
fusion.py:236-266 over the CharLM protocol char_lm.py:23-33) and the exact
two-stage large-vocabulary selection, on the GPU against the oracle."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle.lexicon import OracleDict
from oracle.neural import OracleAttnLstmScorer
from oracle.search import OracleConfig, decode_batch as oracle_decode
from oracle.subword import (OracleLstmCharLM, OracleSubwordFusion, OracleTableCharLM,
                            OracleUniformCharLM)
from test_gpu_models import SCORE_TOL, _compare
from test_oracle_golden import TableScorer, _Feat

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def fb():
    import paper_1909_08723_b200 as m
    return m


@pytest.mark.parametrize("flags", [0, 1, 2, 3])
def test_subword_decode_golden(flags, monkeypatch):
    """Reference-generated SubwordFusion decodes (table CharLM / UniformCharLM)
    through the product decode_batch: bit-identical tokens, scores, accumulators."""
    m = fb()
    from paper_1909_08723_b200 import decoder as dmod
    monkeypatch.setattr(dmod, "_SELECT_FLAGS", flags)
    g = load_golden("subword.pkl.gz")
    d = m.TokenDictionary(g["letters"])
    for case in g["cases"]:
        lm = (OracleUniformCharLM(len(d), d.pad_id) if case["uniform"]
              else OracleTableCharLM(case["rows"], case["default"]))
        feats = [m.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in case["order"]]
        res = m.decode_batch(feats, TableScorer(case["tables"]), m.SubwordFusion(lm),
                             m.DecodeConfig(**case["cfg"]), d)
        for r, (uid, toks, score, acc, fin, steps) in zip(res, case["results"]):
            assert (r.utt_id, r.tokens, r.finished, r.steps) == (uid, toks, fin, steps)
            assert r.score == score
            assert np.asarray(r.attn_accum).tobytes() == acc.tobytes()


def _rand_table(rng, V, pad, eos, t_enc, depth=2):
    rows, frontier, prefixes = {}, [()], [()]
    for _ in range(depth):
        frontier = [p + (t,) for p in frontier for t in range(V) if t not in (pad, eos)]
        prefixes += frontier
    for p in prefixes:
        rows[p] = (np.log(rng.dirichlet(np.ones(V))), rng.dirichlet(np.ones(t_enc)))
    return (t_enc, rows, (np.log(rng.dirichlet(np.ones(V))), rng.dirichlet(np.ones(t_enc))))


@pytest.mark.parametrize("beam", [1, 3, 8, 40])
def test_two_stage_selection_equals_single_stage(beam, monkeypatch):
    """Per-row top-beam then the beam cut over the survivors == the one-CTA
    selection over all beam x vocab candidates (ties included: quantised rows)."""
    m = fb()
    from paper_1909_08723_b200 import decoder as dmod
    rng = np.random.default_rng(beam)
    letters = list("abcdefghijkl")
    d = m.TokenDictionary(letters)
    V = len(d)
    tables = {f"u{i}": _rand_table(rng, V, d.pad_id, d.eos_id, int(rng.integers(3, 8)))
              for i in range(5)}
    q = np.log(rng.choice([1.0, 2.0, 4.0], size=V) / 20.0)
    q[d.pad_id] = -30.0
    feats = [m.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in tables]
    cfg = m.DecodeConfig(beam_size=beam, lm_weight=0.6, coverage_mode="improved",
                         coverage_weight=0.03, eos_gamma=1.4, max_len_ratio=2.0)
    out = []
    for flags in (0, 1, 2, 3):
        monkeypatch.setattr(dmod, "_SELECT_FLAGS", flags)
        out.append(m.decode_batch(feats, TableScorer(tables),
                                  m.SubwordFusion(OracleTableCharLM({(): q}, q)), cfg, d))
    for other in out[1:]:
        for a, b in zip(out[0], other):
            assert (a.tokens, a.finished, a.steps) == (b.tokens, b.finished, b.steps)
            assert a.score == b.score


def small_subword(n_tok=60, seed=3):
    m = fb()
    from paper_1909_08723_b200 import synth
    toks = synth.subword_token_list(n_tok, seed=seed)
    d = m.TokenDictionary(toks)
    ad = synth.AsrDims(enc_layers=2, enc_hidden=32, dec_layers=2, dec_hidden=32, emb=16, att=32,
                       vocab=len(d), out_scale=0.6)
    sd = synth.SubwordLmDims(layers=2, hidden=48, emb=32, vocab=len(d), out_scale=0.5)
    W = synth.asr_weights(ad, seed=17, eos_id=d.eos_id)
    W.update(synth.subword_lm_weights(sd, seed=18, eos_id=d.eos_id))
    return m, synth, toks, d, ad, sd, W


def test_subword_lm_rows_match_oracle():
    m, synth, toks, d, ad, sd, W = small_subword()
    from paper_1909_08723_b200.models import LstmSubwordLM
    gpu = LstmSubwordLM(W, sd, d.pad_id, d.eos_id)
    cpu = OracleLstmCharLM(W, sd.layers, d.pad_id, d.eos_id)
    sg, sc = gpu.start(), cpu.start()
    for t in [5, 9, d.eos_id, 33, d.space_id, 0]:
        rg, rc = gpu.log_probs(sg), cpu.log_probs(sc)
        np.testing.assert_allclose(rg, rc, rtol=0, atol=2e-5)
        assert rg[d.pad_id] == -30.0
        assert abs(np.exp(np.delete(rg, d.pad_id)).sum() - 1.0) < 1e-9
        sg, sc = gpu.advance(sg, t), cpu.advance(sc, t)


@pytest.mark.parametrize("cfg,two", [
    (dict(beam_size=4, lm_weight=0.4), False),
    (dict(beam_size=7, lm_weight=0.8, coverage_mode="improved", coverage_weight=0.02,
          eos_gamma=1.5), False),
    (dict(beam_size=6, lm_weight=0.5), True),
])
def test_fused_subword_engine_matches_oracle(cfg, two):
    m, synth, toks, d, ad, sd, W = small_subword()
    from paper_1909_08723_b200.engine import FusedDecoder
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM
    utts = synth.synth_fbank(6, seed=19, frames=(40, 96))
    feats = [m.FeatureMatrix(u, x) for u, x in utts]
    sc = AttnLstmScorer(W, ad, d.eos_id)
    fus = m.SubwordFusion(LstmSubwordLM(W, sd, d.pad_id, d.eos_id))
    assert fus.device_native
    dc = m.DecodeConfig(**cfg)
    if two:
        dec = FusedDecoder(sc, fus, dc, d)
        dec.select_flags = 3
        Xh, T = sc.encoder.stage([x for _, x in utts])
        got = dec.run(Xh.to(sc.device), T, [u for u, _ in utts])
    else:
        got = m.decode_batch(feats, sc, fus, dc, d)
    od = OracleDict(toks)
    want = oracle_decode([_Feat(u, x) for u, x in utts],
                         OracleAttnLstmScorer(W, ad.enc_layers, ad.dec_layers, ad.subsample,
                                              od.eos_id),
                         OracleSubwordFusion(OracleLstmCharLM(W, sd.layers, od.pad_id, od.eos_id)),
                         OracleConfig(**cfg), od)
    _compare(got, want, cfg)


def test_subword_plugin_driver_agrees_with_fused_engine():
    m, synth, toks, d, ad, sd, W = small_subword()
    from paper_1909_08723_b200.decoder import _decode_plugins
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM
    utts = synth.synth_fbank(4, seed=21, frames=(40, 80))
    feats = [m.FeatureMatrix(u, x) for u, x in utts]
    sc = AttnLstmScorer(W, ad, d.eos_id)
    lm = LstmSubwordLM(W, sd, d.pad_id, d.eos_id)
    cfg = m.DecodeConfig(beam_size=5, lm_weight=0.6)
    a = m.decode_batch(feats, sc, m.SubwordFusion(lm), cfg, d)
    b = _decode_plugins(feats, sc, m.SubwordFusion(lm), cfg, d)
    for x, y in zip(a, b):
        assert x.tokens == y.tokens and x.finished == y.finished
        assert abs(x.score - y.score) <= SCORE_TOL


def test_c4_real_size_matches_oracle():
    """Config 4 dimensions (5k subword tokens, beam 60, 4x800 token LSTM LM,
    3x1024 decoder) on two short utterances."""
    m = fb()
    from paper_1909_08723_b200 import synth
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM
    wl = synth.WORKLOADS["c4"]
    toks = synth.subword_token_list(wl.asr.vocab - 4, seed=wl.seed + 3)
    d = m.TokenDictionary(toks)
    assert len(d) == wl.asr.vocab == wl.sublm.vocab
    W = synth.asr_weights(wl.asr, seed=wl.seed, eos_id=d.eos_id)
    W.update(synth.subword_lm_weights(wl.sublm, seed=wl.seed + 1, eos_id=d.eos_id))
    utts = synth.synth_fbank(2, seed=wl.seed + 100, frames=(300, 360))
    cfg = dict(beam_size=wl.beam, lm_weight=wl.lm_weight)
    got = m.decode_batch([m.FeatureMatrix(u, x) for u, x in utts],
                         AttnLstmScorer(W, wl.asr, d.eos_id),
                         m.SubwordFusion(LstmSubwordLM(W, wl.sublm, d.pad_id, d.eos_id)),
                         m.DecodeConfig(**cfg), d)
    od = OracleDict(toks)
    want = oracle_decode([_Feat(u, x) for u, x in utts],
                         OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers,
                                              wl.asr.subsample, od.eos_id),
                         OracleSubwordFusion(OracleLstmCharLM(W, wl.sublm.layers, od.pad_id,
                                                              od.eos_id)),
                         OracleConfig(**cfg), od)
    _compare(got, want, "c4")


def test_radix_topk_massive_ties_matches_oracle():
    """Hundreds of exactly tied candidates (uniform rows over 300 tokens): the
    radix top-K survivors overflow and the exact fallback must keep the
    reference's (score desc, token-major index asc) order."""
    m = fb()
    rng = np.random.default_rng(5)
    letters = [f"t{i}" for i in range(296)]
    d = m.TokenDictionary(letters)
    od = OracleDict(letters)
    V = len(d)
    uni = np.full(V, math.log(1.0 / V))
    tables = {}
    for i in range(3):
        t_enc = int(rng.integers(2, 5))
        rows = {(): (uni, rng.dirichlet(np.ones(t_enc)))}
        for t in range(0, V, 37):
            p = rng.dirichlet(np.ones(V)) if t % 2 else uni
            rows[(t,)] = (np.log(p) if t % 2 else p, rng.dirichlet(np.ones(t_enc)))
        tables[f"u{i}"] = (t_enc, rows, (uni, rng.dirichlet(np.ones(t_enc))))
    for beam in (4, 16):
        cfg = dict(beam_size=beam, lm_weight=0.5, max_len_ratio=1.0)
        feats = [m.FeatureMatrix(u, np.zeros((1, 1), np.float32)) for u in tables]
        got = m.decode_batch(feats, TableScorer(tables),
                             m.SubwordFusion(OracleUniformCharLM(V, d.pad_id)),
                             m.DecodeConfig(**cfg), d)
        want = oracle_decode([_Feat(u, None) for u in tables], TableScorer(tables),
                             OracleSubwordFusion(OracleUniformCharLM(V, od.pad_id)),
                             OracleConfig(**cfg), od)
        for a, b in zip(got, want):
            assert (a.tokens, a.finished, a.steps) == (b.tokens, b.finished, b.steps)
            assert a.score == b.score
