"""decode_corpus on the device engine (reference decoder.py:483-504 and the
pipeline's fusion-per-batch pattern, pipeline.py:135-153, 210-211):

* a fresh LookaheadFusion per batch reuses ONE cached engine and ONE device
  session (buffers + step graphs) for the whole corpus, the last smaller
  batch included;
* results equal decoding each batch alone (batch invariance) and the
  workers > 1 thread pool gives the same results as workers = 1 (decodes on
  one scorer serialise on its lock);
* the look-ahead floored-score diagnostics reach each batch's fusion.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def _setup():
    import paper_1909_08723_b200 as fb
    from paper_1909_08723_b200 import synth
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
    d = fb.TokenDictionary(synth.wsj_token_list())
    words = synth.synth_lexicon(300, seed=5)
    ad = synth.AsrDims(enc_layers=2, enc_hidden=32, dec_layers=2, dec_hidden=32, emb=16, att=32,
                       out_scale=0.6)
    ld = synth.LmDims(layers=2, hidden=48, words=300, emb_scale=0.3, eos_bias=2.0)
    W = synth.asr_weights(ad, seed=7, eos_id=d.eos_id)
    W.update(synth.lm_weights(ld, seed=8))
    trie = fb.build_trie(words, d)
    scorer = AttnLstmScorer(W, ad, d.eos_id)
    lm = LstmWordLM(W, ld)
    utts = synth.synth_fbank(11, seed=41, frames=(40, 120))
    feats = [fb.FeatureMatrix(u, x) for u, x in utts]
    made = []

    def factory():
        f = fb.LookaheadFusion(trie, lm, d)
        made.append(f)
        return f

    return fb, d, scorer, feats, factory, made


def _key(rs):
    return [(r.utt_id, tuple(r.tokens), r.score, r.finished, r.steps) for r in rs]


def test_fusion_per_batch_reuses_one_session():
    fb, d, scorer, feats, factory, made = _setup()
    cfg = fb.DecodeConfig(beam_size=4, lm_weight=0.5)
    got = fb.decode_corpus(feats, scorer, factory, cfg, d, batch_size=4)
    assert len(made) == 3                                  # 4 + 4 + 3 utterances
    assert len(scorer._fused_cache) == 1
    dec = next(iter(scorer._fused_cache.values()))
    assert len(dec._sessions) == 1 and dec._sessions[0].B == 4
    # each batch alone on a fresh engine (sessions sized to each batch: the
    # 3-utterance batch without inactive padding)
    fb2, d2, scorer2, feats2, factory2, _ = _setup()
    alone = []
    for i in range(0, len(feats2), 4):
        alone.extend(fb2.decode_batch(feats2[i:i + 4], scorer2, factory2(), cfg, d2))
    # the last (3-utterance) batch on yet another fresh engine: an exact-size session
    fb3, d3, scorer3, feats3, factory3, _ = _setup()
    last = fb3.decode_batch(feats3[8:], scorer3, factory3(), cfg, d3)
    assert next(iter(scorer3._fused_cache.values()))._sessions[0].B == 3
    assert _key(got[8:]) == _key(last)
    assert _key(got) == _key(alone)
    assert [r.utt_id for r in got] == [f.utt_id for f in feats]
    assert sum(f.diagnostics["floored_scores"] for f in made[:3]) >= 0


def test_workers_thread_pool_matches_sequential():
    fb, d, scorer, feats, factory, made = _setup()
    cfg = fb.DecodeConfig(beam_size=5, lm_weight=0.7, coverage_mode="improved",
                          coverage_weight=0.02)
    one = fb.decode_corpus(feats, scorer, factory, cfg, d, batch_size=3, workers=1)
    many = fb.decode_corpus(feats, scorer, factory, cfg, d, batch_size=3, workers=3)
    assert _key(one) == _key(many)
    for a, b in zip(one, many):
        np.testing.assert_array_equal(a.attn_accum, b.attn_accum)
