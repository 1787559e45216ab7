"""GPU parity of the neural scorers and the fused engine against the CPU oracle
(PyTorch-CPU fp32 restatement, oracle/neural.py) on the same random-init
weights and synthetic fbank (BASELINE.json north_star: identical hypotheses
except on near-ties, per-hypothesis scores within 1e-4)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle.lexicon import OracleDict, build_trie as oracle_build_trie
from oracle.lookahead import OracleLookahead
from oracle.neural import OracleAttnLstmScorer, OracleLstmWordLM
from oracle.search import OracleConfig, decode_batch as oracle_decode
from test_oracle_golden import _Feat

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SCORE_TOL = 1e-4       # north star: per-hypothesis scores within 1e-4 absolute
TIE_TOL = 1e-4         # decisions closer than this are near-ties (exempt)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def small_setup(n_words=300, seed=5):
    from paper_1909_08723_b200 import synth
    import paper_1909_08723_b200 as fb
    d = fb.TokenDictionary(synth.wsj_token_list())
    words = synth.synth_lexicon(n_words, seed=seed)
    ad = synth.AsrDims(enc_layers=2, enc_hidden=32, dec_layers=2, dec_hidden=32, emb=16, att=32,
                       out_scale=0.6)
    ld = synth.LmDims(layers=2, hidden=48, words=n_words, emb_scale=0.3, eos_bias=2.0)
    W = synth.asr_weights(ad, seed=7, eos_id=d.eos_id)
    W.update(synth.lm_weights(ld, seed=8))
    return fb, synth, d, words, ad, ld, W


def test_scorer_rows_match_oracle():
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import AttnLstmScorer
    gpu = AttnLstmScorer(W, ad, d.eos_id)
    cpu = OracleAttnLstmScorer(W, ad.enc_layers, ad.dec_layers, ad.subsample, d.eos_id)
    for uid, x in synth.synth_fbank(3, seed=9, frames=(40, 90)):
        f = fb.FeatureMatrix(uid, x)
        sg, sc = gpu.init(f), cpu.init(f)
        assert gpu.enc_length(sg) == cpu.enc_length(sc)
        last = [-1]
        rng = np.random.default_rng(0)
        for step in range(6):
            lg, ag, sg = gpu.step(sg, last)
            lc, ac, sc = cpu.step(sc, last)
            np.testing.assert_allclose(lg, lc, rtol=0, atol=2e-5)
            np.testing.assert_allclose(ag, ac, rtol=0, atol=2e-6)
            par = sorted(rng.integers(0, len(last), size=3).tolist())
            sg, sc = gpu.reorder(sg, par), cpu.reorder(sc, par)
            last = rng.integers(0, len(d), size=3).tolist()


def test_word_lm_matches_oracle():
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import LstmWordLM
    gpu = LstmWordLM(W, ld)
    cpu = OracleLstmWordLM(W, ld.layers, ld.words)
    hg, hc = gpu.start_history(), cpu.start_history()
    for r in [3, -1, 17, 299, 0]:
        np.testing.assert_allclose(gpu.full_distribution(hg), cpu.full_distribution(hc),
                                   rtol=2e-5, atol=1e-12)
        assert abs(gpu.eos_log_prob(hg) - cpu.eos_log_prob(hc)) < 2e-5
        hg, hc = gpu.extend_history(hg, r), cpu.extend_history(hc, r)


def _compare(got, want, what):
    exempt = 0
    for a, b in zip(got, want):
        assert a.utt_id == b.utt_id
        if a.tokens != b.tokens or a.finished != b.finished:
            assert b.margin < TIE_TOL, (what, a.utt_id, a.tokens, b.tokens, b.margin)
            exempt += 1
            continue
        assert abs(a.score - b.score) <= SCORE_TOL, (what, a.utt_id, a.score, b.score)
        np.testing.assert_allclose(a.attn_accum, b.attn_accum, atol=1e-4)
    assert exempt <= max(1, len(got) // 5), (what, exempt)
    return exempt


@pytest.mark.parametrize("cfg", [
    dict(beam_size=4, lm_weight=0.5),
    dict(beam_size=6, lm_weight=0.9, coverage_mode="improved", coverage_weight=0.02, eos_gamma=1.5),
    dict(beam_size=3, lm_weight=0.0),
    dict(beam_size=5, lm_weight=0.0, coverage_mode="original", coverage_weight=0.05),
])
def test_fused_engine_matches_oracle(cfg):
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
    utts = synth.synth_fbank(6, seed=9, frames=(40, 96))
    feats = [fb.FeatureMatrix(u, x) for u, x in utts]
    trie = fb.build_trie(words, d)
    gpu_sc = AttnLstmScorer(W, ad, d.eos_id)
    fus = None
    if cfg["lm_weight"] > 0:
        fus = fb.LookaheadFusion(trie, LstmWordLM(W, ld), d)
    got = fb.decode_batch(feats, gpu_sc, fus, fb.DecodeConfig(**cfg), d)
    od = OracleDict(synth.wsj_token_list())
    cpu_sc = OracleAttnLstmScorer(W, ad.enc_layers, ad.dec_layers, ad.subsample, od.eos_id)
    ofus = None
    if cfg["lm_weight"] > 0:
        ofus = OracleLookahead(oracle_build_trie(words, od), OracleLstmWordLM(W, ld.layers, ld.words), od)
    want = oracle_decode([_Feat(u, x) for u, x in utts], cpu_sc, ofus, OracleConfig(**cfg), od)
    _compare(got, want, cfg)


def test_plugin_driver_agrees_with_fused_engine():
    """Same device scorer through the generic plugin driver (host rows) and the
    fused engine: both GPU paths must agree."""
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM

    class Plain:                        # hides is_device_scorer -> plugin driver
        def __init__(self, s):
            self.s = s

        def __getattr__(self, k):
            if k == "is_device_scorer":
                raise AttributeError(k)
            return getattr(self.s, k)

    utts = synth.synth_fbank(4, seed=19, frames=(40, 80))
    feats = [fb.FeatureMatrix(u, x) for u, x in utts]
    trie = fb.build_trie(words, d)
    sc = AttnLstmScorer(W, ad, d.eos_id)
    lm = LstmWordLM(W, ld)
    cfg = fb.DecodeConfig(beam_size=4, lm_weight=0.5)
    a = fb.decode_batch(feats, sc, fb.LookaheadFusion(trie, lm, d), cfg, d)
    b = fb.decode_batch(feats, Plain(sc), fb.LookaheadFusion(trie, lm, d), cfg, d)
    for x, y in zip(a, b):
        assert x.tokens == y.tokens
        assert abs(x.score - y.score) < 1e-6


def test_spec_pruning_is_exact():
    """Pruned speculative <eos> LM events give bit-identical decodes."""
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
    from paper_1909_08723_b200.engine import FusedDecoder
    utts = synth.synth_fbank(8, seed=29, frames=(40, 120))
    trie = fb.build_trie(words, d)
    sc = AttnLstmScorer(W, ad, d.eos_id)
    fus = fb.LookaheadFusion(trie, LstmWordLM(W, ld), d)
    for cfg in (fb.DecodeConfig(beam_size=5, lm_weight=0.7),
                fb.DecodeConfig(beam_size=8, lm_weight=0.3, eos_gamma=1.2)):
        X, T = sc.encoder.stage([x for _, x in utts])
        X = X.to(sc.device)
        ids = [u for u, _ in utts]
        outs = []
        for prune in (False, True):
            dec = FusedDecoder(sc, fus, cfg, d)
            dec.prune_spec = prune
            outs.append(dec.run(X, T, ids, record_counts=True))
        for a, b in zip(*outs):
            assert a.tokens == b.tokens and a.score == b.score and a.steps == b.steps


def test_operand_pipeline_and_fused_epilogues_are_exact(monkeypatch):
    """Per-GEMM A operands written by the LSTM epilogues (+ side-stream packs),
    exp(2q) and log-softmax fused into GEMM epilogues: bit-identical decodes to
    the plain pack-per-GEMM path with separate kernels (same split and
    arithmetic, only the plumbing differs)."""
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200 import engine as E, models as M
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
    utts = synth.synth_fbank(8, seed=31, frames=(40, 120))
    trie = fb.build_trie(words, d)
    sc = AttnLstmScorer(W, ad, d.eos_id)
    fus = fb.LookaheadFusion(trie, LstmWordLM(W, ld), d)
    cfg = fb.DecodeConfig(beam_size=6, lm_weight=0.6, eos_gamma=1.3)
    X, T = sc.encoder.stage([x for _, x in utts])
    X = X.to(sc.device)
    ids = [u for u, _ in utts]
    outs = []
    for fast in (False, True):
        monkeypatch.setattr(E, "AM_PIPELINE", fast)
        monkeypatch.setattr(M, "FUSE_EPI", fast)
        dec = E.FusedDecoder(sc, fus, cfg, d)
        outs.append(dec.run(X, T, ids))
    for a, b in zip(*outs):
        assert a.tokens == b.tokens and a.score == b.score and a.steps == b.steps
        np.testing.assert_array_equal(a.attn_accum, b.attn_accum)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_baseline_small_configs_match_oracle(name):
    """BASELINE.json configs[0] (c1: small BiLSTM + 1-layer attn-LSTM, beam 5, no
    LM) and c3 (c1 + improved coverage + EOS threshold 1.5, beam 20) at their
    real model sizes, GPU fused engine vs the CPU oracle."""
    import paper_1909_08723_b200 as fb
    from paper_1909_08723_b200 import synth
    from paper_1909_08723_b200.models import AttnLstmScorer
    wl = synth.WORKLOADS[name]
    d = fb.TokenDictionary(synth.wsj_token_list())
    W = synth.asr_weights(wl.asr, seed=wl.seed, eos_id=d.eos_id)
    utts = synth.synth_fbank(8, seed=wl.seed + 100, frames=wl.frames)
    cfg = dict(beam_size=wl.beam, lm_weight=0.0, coverage_mode=wl.coverage_mode,
               coverage_weight=wl.coverage_weight, eos_gamma=wl.eos_gamma)
    got = fb.decode_batch([fb.FeatureMatrix(u, x) for u, x in utts],
                          AttnLstmScorer(W, wl.asr, d.eos_id), None, fb.DecodeConfig(**cfg), d)
    od = OracleDict(synth.wsj_token_list())
    want = oracle_decode([_Feat(u, x) for u, x in utts],
                         OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers,
                                              wl.asr.subsample, od.eos_id),
                         None, OracleConfig(**cfg), od)
    _compare(got, want, name)


def test_c2_rows_match_fp64_oracle():
    """Row-level parity at the headline dimensions (BASELINE c2: 4x BiLSTM-320
    encoder, 3x LSTM-320 decoder, T_enc ~200, 52 tokens; 65k-word 3x1200 LM):
    acoustic log-probs and attention rows over several steps with beam
    reorders against the fp64 oracle; LM distributions, log P(</s>) and the
    fp64 g rows (cumulative word mass) against the oracle LM."""
    import bench
    from oracle import harness as H
    import paper_1909_08723_b200 as fb
    from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
    wl = H.workload("c2")
    d, W, trie = bench.build_product(wl)
    utts = H.corpus(wl, 0)
    gpu = AttnLstmScorer(W, wl.asr, d.eos_id)
    cpu = OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers, wl.asr.subsample,
                               d.eos_id, dtype=torch.float64)
    worst_l = worst_a = 0.0
    for i in (0, 255, 511):
        uid, x = utts[i]
        f = fb.FeatureMatrix(uid, x)
        sg, sc = gpu.init(f), cpu.init(f)
        assert gpu.enc_length(sg) == cpu.enc_length(sc) == x.shape[0] // 4
        last = [-1]
        rng = np.random.default_rng(i)
        for step in range(8):
            lg, ag, sg = gpu.step(sg, last)
            lc, ac, sc = cpu.step(sc, last)
            worst_l = max(worst_l, float(np.abs(lg - lc).max()))
            worst_a = max(worst_a, float(np.abs(ag - ac).max()))
            par = sorted(rng.integers(0, len(last), size=wl.beam).tolist())
            sg, sc = gpu.reorder(sg, par), cpu.reorder(sc, par)
            last = rng.integers(3, len(d), size=wl.beam).tolist()
    print(f"\nc2 rows vs fp64 oracle: max |dlogp| {worst_l:.3g}, max |dattn| {worst_a:.3g}")
    assert worst_l <= 2e-5 and worst_a <= 2e-6

    glm = LstmWordLM(W, wl.lm)
    clm = OracleLstmWordLM(W, wl.lm.layers, wl.lm.words)
    hg, hc = glm.start_history(), clm.start_history()
    worst_p = worst_e = worst_g = 0.0
    for r in [17, -1, 64999, 0, 31337]:
        pg, pc = glm.full_distribution(hg), clm.full_distribution(hc)
        worst_p = max(worst_p, float(np.max(np.abs(pg - pc) / np.maximum(pc, 1e-300))))
        worst_e = max(worst_e, abs(glm.eos_log_prob(hg) - clm.eos_log_prob(hc)))
        worst_g = max(worst_g, float(np.abs(np.cumsum(pg) - np.cumsum(pc)).max()))
        hg, hc = glm.extend_history(hg, r), clm.extend_history(hc, r)
    # the fused engine's g rows (LookaheadFusion.start -> the device scan)
    fus = fb.LookaheadFusion(trie, glm, d)
    g0 = fus.start(1).g[0]
    ref_g = np.cumsum(clm.full_distribution(clm.start_history()))
    worst_g = max(worst_g, float(np.abs(g0 - ref_g).max()))
    print(f"c2 LM vs oracle: max rel dP {worst_p:.3g}, max |d log P(</s>)| {worst_e:.3g}, "
          f"max |dg| {worst_g:.3g}")
    assert worst_p <= 2e-5 and worst_e <= 2e-5 and worst_g <= 2e-6


def test_encoder_recurrence_row_blocks_are_exact(monkeypatch):
    """A batch whose recurrence grid exceeds the co-resident capacity runs as
    cooperative launches over row blocks (rows never interact): forced here
    with the FB_REC_MAX_ROWS test knob (128-row blocks, 3 launches per
    direction for 300 utterances), the encoder output and keys are
    bit-identical to one launch."""
    fb, synth, d, words, ad, ld, W = small_setup()
    from paper_1909_08723_b200.models import AttnLstmScorer
    utts = synth.synth_fbank(300, seed=77, frames=(24, 96))
    sc = AttnLstmScorer(W, ad, d.eos_id)
    X, T = sc.encoder.stage([x for _, x in utts])
    X = X.to(sc.device)
    outs = []
    for cap in (None, "128"):
        if cap is None:
            monkeypatch.delenv("FB_REC_MAX_ROWS", raising=False)
        else:
            monkeypatch.setenv("FB_REC_MAX_ROWS", cap)
        enc, keys, Tenc = sc.encoder(X, list(T))
        torch.cuda.synchronize()
        outs.append((enc.clone(), keys.clone(), list(Tenc)))
    assert outs[0][2] == outs[1][2]
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
