"""Generate the golden fixtures that pin the oracle (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the UNMODIFIED reference package ``fusedbeam`` read-only from
``/root/reference/pkg/src`` and records its outputs on seeded inputs:

* ``trie.pkl.gz``      -- ``build_trie`` arrays on random lexicons
                          (lexicon_trie.py:227-276);
* ``lookahead.pkl.gz`` -- ``LookaheadFusion.char_scores/advance/reorder`` rows on
                          random lexicons, TableLM rows and random walks
                          (fusion.py:109-233);
* ``decode.pkl.gz``    -- ``decode_batch`` results over random acoustic tables
                          (plain / original / improved coverage / EOS gate /
                          look-ahead fusion, quantised ties) (decoder.py:339-480);
* ``neural.pkl.gz``    -- ``decode_batch`` + ``LookaheadFusion`` driving the
                          oracle's PyTorch-CPU attention-LSTM scorer and LSTM
                          word LM at a small size;
* ``multilevel.pkl.gz`` -- MultilevelFusion walks and decodes (fusion.py:268-380);
* ``formats/``         -- PTA1 trie files saved by the reference
                          (lexicon_trie.py:178-224) and a Kaldi ARK/SCP pair
                          written by its ``write_ark_matrix`` (kaldi_io.py:137-160),
                          plus corrupt records and the reference reader's
                          exception type/message for each (``formats.pkl.gz``);
* ``subword.pkl.gz``   -- ``SubwordFusion`` rows/advance/reorder and
                          ``decode_batch`` with ``SubwordFusion`` over
                          ``UniformCharLM`` and a table ``CharLM`` fake
                          (fusion.py:236-266, char_lm.py:23-53), plus the
                          oracle's token LSTM LM + attention-LSTM scorer on a
                          small subword dictionary.

The GPU box never reads /root/reference: the tests only read these files.
"""

from __future__ import annotations

import gzip
import os
import pickle
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from fusedbeam.char_lm import CharLM, UniformCharLM  # noqa: E402
from fusedbeam.decoder import DecodeConfig, TraceScorer, _TraceTable, decode_batch  # noqa: E402
from fusedbeam.fusion import (LookaheadBatch, LookaheadFusion, MultilevelFusion,  # noqa: E402
                              SubwordFusion)
from fusedbeam.kaldi_io import FeatureMatrix  # noqa: E402
from fusedbeam.lexicon_trie import build_trie  # noqa: E402
from fusedbeam.token_dict import TokenDictionary  # noqa: E402
from fusedbeam.word_lm import TableLM  # noqa: E402

from oracle.neural import OracleAttnLstmScorer, OracleLstmWordLM  # noqa: E402
from oracle.subword import OracleLstmCharLM  # noqa: E402
from paper_1909_08723_b200 import synth  # noqa: E402


def dump(name, obj):
    with gzip.open(os.path.join(HERE, name), "wb") as f:
        pickle.dump(obj, f, protocol=4)


def rand_vocab(rng, max_words, alphabet, max_len=6):
    letters = list("abcdefghij"[:alphabet])
    distinct = sum(alphabet ** k for k in range(1, max_len + 1))
    n = int(rng.integers(2, min(max_words, distinct) + 1))
    words = set()
    while len(words) < n:
        words.add("".join(rng.choice(letters, size=int(rng.integers(1, max_len + 1)))))
    return letters, sorted(words)


def trie_cases():
    rng = np.random.default_rng(11)
    cases = []
    for i in range(40):
        letters, words = rand_vocab(rng, 200, int(rng.integers(2, 11)))
        d = TokenDictionary(letters)
        t = build_trie(words, d)
        cases.append(dict(letters=letters, words=words,
                          transitions=t.transitions.copy(), edge_labels=t.edge_labels.copy(),
                          is_final=t.is_final.copy(), word_index=t.word_index.copy(),
                          ub=t.ub_index.copy(), lb=t.lb_index.copy(),
                          children=t.char_children.copy(), ranked=t.words(d)))
    dump("trie.pkl.gz", cases)


def lookahead_cases():
    rng = np.random.default_rng(22)
    cases = []
    for i in range(30):
        letters, words = rand_vocab(rng, 120, int(rng.integers(2, 9)))
        d = TokenDictionary(letters)
        t = build_trie(words, d)
        ranked = t.words(d)
        V = len(ranked)
        rows = {(): rng.dirichlet(np.ones(V))}
        for w in ranked[: min(V, 5)]:
            rows[(w,)] = rng.dirichlet(np.ones(V)) * (0 if i % 7 == 3 else 1)
        eos = {(): 0.05, (ranked[0],): 0.2}
        lm = TableLM(vocab=tuple(ranked), rows=rows, eos=eos)
        fus = LookaheadFusion(t, lm, d)
        n = 6
        st = fus.start(n)
        walk = []
        char_ids = [d.index(c) for c in letters]
        for step in range(8):
            sc = fus.char_scores(st)
            toks = []
            for b in range(n):
                s = int(st.trie_states[b])
                opts = [c for c in char_ids if s >= 0 and t.char_children[s, c] >= 0]
                u = rng.random()
                if u < 0.2 or not opts:
                    toks.append(d.space_id)
                elif u < 0.27:
                    toks.append(int(rng.choice(char_ids)))     # may leave the lexicon
                elif u < 0.3:
                    toks.append(d.eos_id)
                else:
                    toks.append(int(rng.choice(opts)))
            parents = sorted(rng.integers(0, n, size=n).tolist())
            walk.append(dict(scores=sc, tokens=np.array(toks), parents=np.array(parents),
                             states=st.trie_states.copy(), g=st.g.copy(),
                             floored=fus.diagnostics["floored_scores"]))
            st = fus.advance(st, np.array(toks))
            st = fus.reorder(st, parents)
        cases.append(dict(letters=letters, words=words, rows=rows, eos=eos, walk=walk))
    dump("lookahead.pkl.gz", cases)


def rand_table(rng, d, uid, t_enc, depth=2, quantized=False):
    V = len(d)

    def dist():
        if quantized:
            raw = rng.choice([1.0, 2.0, 4.0], size=V)
            return raw / raw.sum()
        return rng.dirichlet(np.ones(V))

    rows = {}
    prefixes = [()]
    frontier = [()]
    for _ in range(depth):
        nxt = [p + (tok,) for p in frontier for tok in range(V)
               if tok not in (d.pad_id, d.eos_id)]
        frontier = nxt
        prefixes.extend(nxt)
    for p in prefixes:
        rows[p] = (np.log(dist()), rng.dirichlet(np.ones(t_enc)))
    default = (np.log(dist()), rng.dirichlet(np.ones(t_enc)))
    return _TraceTable(uid, t_enc, V, rows, default)


def decode_cases():
    rng = np.random.default_rng(33)
    d = TokenDictionary(["a", "b", "c"])
    t = build_trie(["a", "ab", "abc", "b", "bc", "ca", "cab"], d)
    ranked = t.words(d)
    cases = []
    for i in range(24):
        mode = i % 6
        nutt = int(rng.integers(1, 5))
        tables = {}
        for u in range(nutt):
            uid = f"u{i}_{u}"
            tables[uid] = rand_table(rng, d, uid, int(rng.integers(2, 7)),
                                     depth=2, quantized=bool(i % 2))
        lm_rows = {(): rng.dirichlet(np.ones(len(ranked)))}
        for w in ranked[:3]:
            lm_rows[(w,)] = rng.dirichlet(np.ones(len(ranked)))
        cfg = dict(beam_size=int(rng.integers(1, 9)),
                   lm_weight=[0.0, 0.0, 0.0, 0.9, 0.7, 0.5][mode],
                   coverage_mode=["off", "original", "improved", "improved", "off", "improved"][mode],
                   coverage_weight=0.05, tau1=0.4, tau2=0.9, cov_margin=0.7,
                   eos_gamma=[None, None, 1.5, 1.5, None, 1.2][mode],
                   max_len_ratio=[1.0, 1.5, 1.0, 2.0, 1.0, 1.0][mode])
        fused = mode >= 3
        fus = None
        if fused:
            lm = TableLM(vocab=tuple(ranked), rows=lm_rows, eos={(): 0.1})
            fus = LookaheadFusion(t, lm, d)
        feats = [FeatureMatrix(uid, np.zeros((1, 1), np.float32)) for uid in tables]
        res = decode_batch(feats, TraceScorer(tables), fus, DecodeConfig(**cfg), d)
        cases.append(dict(tables={k: (v.t_enc, v.rows, v.default) for k, v in tables.items()},
                          order=list(tables), cfg=cfg, fused=fused, lm_rows=lm_rows,
                          lm_eos={(): 0.1},
                          results=[(r.utt_id, r.tokens, r.score, r.attn_accum.copy(),
                                    r.finished, r.steps) for r in res]))
    dump("decode.pkl.gz", dict(letters=["a", "b", "c"],
                               words=["a", "ab", "abc", "b", "bc", "ca", "cab"],
                               cases=cases))


def neural_cases():
    import torch
    torch.set_num_threads(4)
    d = TokenDictionary(synth.wsj_token_list())
    words = synth.synth_lexicon(300, seed=5)
    t = build_trie(words, d)
    ranked = t.words(d)
    adims = synth.AsrDims(enc_layers=2, enc_hidden=32, dec_layers=2, dec_hidden=32,
                          emb=16, att=32, out_scale=0.6)
    ldims = synth.LmDims(layers=2, hidden=48, words=len(ranked), emb_scale=0.3,
                         eos_bias=2.0)
    W = synth.asr_weights(adims, seed=7, eos_id=d.eos_id)
    W.update(synth.lm_weights(ldims, seed=8))
    utts = synth.synth_fbank(4, seed=9, frames=(40, 64))
    feats = [FeatureMatrix(u, x) for u, x in utts]
    cases = []
    for k, cfg in enumerate([
            dict(beam_size=4, lm_weight=0.5),
            dict(beam_size=6, lm_weight=0.9, coverage_mode="improved",
                 coverage_weight=0.02, eos_gamma=1.5),
            dict(beam_size=3, lm_weight=0.0)]):
        sc = OracleAttnLstmScorer(W, adims.enc_layers, adims.dec_layers,
                                  adims.subsample, d.eos_id)
        lm = OracleLstmWordLM(W, ldims.layers, len(ranked))
        fus = LookaheadFusion(t, lm, d) if cfg["lm_weight"] > 0 else None
        res = decode_batch(feats, sc, fus, DecodeConfig(**cfg), d)
        cases.append(dict(cfg=cfg, results=[(r.utt_id, r.tokens, r.score,
                                             np.asarray(r.attn_accum).copy(), r.finished,
                                             r.steps) for r in res]))
    dump("neural.pkl.gz", dict(words=words, adims=adims.__dict__, ldims=ldims.__dict__,
                               asr_seed=7, lm_seed=8, fbank_seed=9, frames=(40, 64),
                               n_utts=4, cases=cases))


class TableCharLM(CharLM):
    """Reference-protocol fake: rows keyed by token history, longest listed
    suffix wins (same as oracle.subword.OracleTableCharLM)."""

    def __init__(self, rows, default):
        self.rows, self.default = rows, default

    def start(self):
        return ()

    def log_probs(self, state):
        for k in range(len(state), -1, -1):
            r = self.rows.get(tuple(state[len(state) - k:]))
            if r is not None:
                return r
        return self.default

    def advance(self, state, token_id):
        return tuple(state) + (int(token_id),)


def _char_row(rng, d, quantized=False, eos_scale=0.02):
    V = len(d)
    p = rng.choice([1.0, 2.0, 4.0], size=V) if quantized else rng.dirichlet(np.ones(V))
    p[d.pad_id] = 0.0
    p[d.eos_id] *= eos_scale           # keep hypotheses alive past the first steps
    p = p / p.sum()
    with np.errstate(divide="ignore"):
        row = np.log(p)
    row[d.pad_id] = -30.0
    return row


def subword_cases():
    rng = np.random.default_rng(44)
    letters = ["a", "b", "c", "d"]
    d = TokenDictionary(letters)
    V = len(d)
    # fusion rows / advance / reorder walk (test_fusion.py:224-237 generalised)
    walks = []
    for i in range(6):
        rows = {(): _char_row(rng, d)}
        for t in range(V):
            if rng.random() < 0.5:
                rows[(t,)] = _char_row(rng, d)
        default = _char_row(rng, d)
        fus = SubwordFusion(TableCharLM(rows, default))
        st = fus.start(5)
        walk = []
        for step in range(5):
            sc = fus.char_scores(st)
            toks = rng.integers(0, V, size=5)
            parents = sorted(rng.integers(0, 5, size=5).tolist())
            walk.append(dict(scores=sc, tokens=toks, parents=np.array(parents)))
            st = fus.reorder(fus.advance(st, toks), parents)
        walks.append(dict(rows=rows, default=default, walk=walk))
    cases = []
    for i in range(24):
        mode = i % 4
        nutt = int(rng.integers(1, 5))
        tables = {}
        for u in range(nutt):
            uid = f"s{i}_{u}"
            tables[uid] = rand_table(rng, d, uid, int(rng.integers(2, 6)), depth=2,
                                     quantized=bool(i % 2))
        uniform = i % 3 == 0
        rows = {(): _char_row(rng, d, quantized=bool(i % 2), eos_scale=1e-4)}
        for t in range(V):
            if rng.random() < 0.6:
                rows[(t,)] = _char_row(rng, d, quantized=bool(i % 2))
        default = _char_row(rng, d)
        lm = UniformCharLM(d) if uniform else TableCharLM(rows, default)
        cfg = dict(beam_size=int(rng.integers(1, 9)), lm_weight=[0.3, 0.7, 1.0, 0.5][mode],
                   coverage_mode=["off", "original", "improved", "off"][mode],
                   coverage_weight=0.05, tau1=0.4, tau2=0.9, cov_margin=0.7,
                   eos_gamma=[None, 1.5, None, 1.2][mode],
                   max_len_ratio=[1.0, 1.5, 2.0, 1.0][mode])
        feats = [FeatureMatrix(uid, np.zeros((1, 1), np.float32)) for uid in tables]
        res = decode_batch(feats, TraceScorer(tables), SubwordFusion(lm), DecodeConfig(**cfg), d)
        cases.append(dict(tables={k: (v.t_enc, v.rows, v.default) for k, v in tables.items()},
                          order=list(tables), cfg=cfg, uniform=uniform, rows=rows,
                          default=default,
                          results=[(r.utt_id, r.tokens, r.score, r.attn_accum.copy(),
                                    r.finished, r.steps) for r in res]))
    # neural: oracle attention-LSTM scorer + oracle token LSTM LM through the
    # reference SubwordFusion / decode_batch
    import torch
    torch.set_num_threads(4)
    sd = TokenDictionary(synth.subword_token_list(60, seed=3))
    adims = synth.AsrDims(enc_layers=2, enc_hidden=32, dec_layers=2, dec_hidden=32,
                          emb=16, att=32, vocab=len(sd), out_scale=0.6)
    sdims = synth.SubwordLmDims(layers=2, hidden=48, emb=32, vocab=len(sd), out_scale=0.5)
    W = synth.asr_weights(adims, seed=17, eos_id=sd.eos_id)
    W.update(synth.subword_lm_weights(sdims, seed=18, eos_id=sd.eos_id))
    utts = synth.synth_fbank(4, seed=19, frames=(40, 64))
    feats = [FeatureMatrix(u, x) for u, x in utts]
    neural = []
    for cfg in (dict(beam_size=4, lm_weight=0.4),
                dict(beam_size=7, lm_weight=0.8, coverage_mode="improved",
                     coverage_weight=0.02, eos_gamma=1.5)):
        sc = OracleAttnLstmScorer(W, adims.enc_layers, adims.dec_layers, adims.subsample,
                                  sd.eos_id)
        lm = OracleLstmCharLM(W, sdims.layers, sd.pad_id, sd.eos_id)
        res = decode_batch(feats, sc, SubwordFusion(lm), DecodeConfig(**cfg), sd)
        neural.append(dict(cfg=cfg, results=[(r.utt_id, r.tokens, r.score,
                                              np.asarray(r.attn_accum).copy(), r.finished,
                                              r.steps) for r in res]))
    dump("subword.pkl.gz", dict(letters=letters, walks=walks, cases=cases,
                                neural=dict(tokens=synth.subword_token_list(60, seed=3),
                                            adims=adims.__dict__, sdims=sdims.__dict__,
                                            asr_seed=17, lm_seed=18, fbank_seed=19,
                                            frames=(40, 64), n_utts=4, cases=neural)))


def multilevel_cases():
    """Reference MultilevelFusion (fusion.py:268-380): walks of char_scores /
    advance / reorder with diagnostics, and decode_batch results."""
    rng = np.random.default_rng(66)
    letters = ["a", "b", "c"]
    d = TokenDictionary(letters)
    words = ["a", "ab", "abc", "b", "bc", "ca", "cab"]
    t = build_trie(words, d)
    ranked = t.words(d)
    V = len(d)
    walks = []
    for i in range(6):
        rows = {(): _char_row(rng, d, eos_scale=0.3)}
        for tk in range(V):
            if rng.random() < 0.5:
                rows[(tk,)] = _char_row(rng, d, eos_scale=0.3)
        default = _char_row(rng, d)
        lm_rows = {(): rng.dirichlet(np.ones(len(ranked)))}
        for w in ranked[:3]:
            lm_rows[(w,)] = rng.dirichlet(np.ones(len(ranked)))
        lm = TableLM(vocab=tuple(ranked), rows=lm_rows, eos={})
        fus = MultilevelFusion(TableCharLM(rows, default), lm, t, d, oov_factor=-7.5)
        st = fus.start(5)
        walk = []
        char_ids = [d.index(c) for c in letters]
        for step in range(10):
            sc = fus.char_scores(st)
            toks = []
            for b in range(5):
                u = rng.random()
                toks.append(d.space_id if u < 0.25 else d.eos_id if u < 0.3 else
                            d.pad_id if u < 0.33 else int(rng.choice(char_ids)))
            parents = sorted(rng.integers(0, 5, size=5).tolist())
            walk.append(dict(scores=sc, tokens=np.array(toks), parents=np.array(parents),
                             states=st.trie_states.copy(), accum=st.char_accum.copy(),
                             empty=fus.diagnostics["empty_words"]))
            st = fus.reorder(fus.advance(st, np.array(toks)), parents)
        walks.append(dict(rows=rows, default=default, lm_rows=lm_rows, walk=walk))
    cases = []
    for i in range(16):
        nutt = int(rng.integers(1, 5))
        tables = {}
        for u in range(nutt):
            uid = f"m{i}_{u}"
            tables[uid] = rand_table(rng, d, uid, int(rng.integers(2, 6)), depth=2,
                                     quantized=bool(i % 2))
        rows = {(): _char_row(rng, d, eos_scale=0.2)}
        for tk in range(V):
            if rng.random() < 0.6:
                rows[(tk,)] = _char_row(rng, d, eos_scale=0.2)
        default = _char_row(rng, d)
        lm_rows = {(): rng.dirichlet(np.ones(len(ranked)))}
        for w in ranked[:4]:
            lm_rows[(w,)] = rng.dirichlet(np.ones(len(ranked)))
        uniform = i % 4 == 0
        clm = UniformCharLM(d) if uniform else TableCharLM(rows, default)
        lm = TableLM(vocab=tuple(ranked), rows=lm_rows, eos={})
        cfg = dict(beam_size=int(rng.integers(1, 7)), lm_weight=[0.4, 0.8, 1.0, 0.6][i % 4],
                   coverage_mode=["off", "improved", "original", "off"][i % 4],
                   coverage_weight=0.05, tau1=0.4, tau2=0.9, cov_margin=0.7,
                   eos_gamma=[None, 1.5, None, 1.2][i % 4], max_len_ratio=[1.0, 1.5, 2.0, 1.0][i % 4])
        fus = MultilevelFusion(clm, lm, t, d, oov_factor=-6.0)
        feats = [FeatureMatrix(uid, np.zeros((1, 1), np.float32)) for uid in tables]
        res = decode_batch(feats, TraceScorer(tables), fus, DecodeConfig(**cfg), d)
        cases.append(dict(tables={k: (v.t_enc, v.rows, v.default) for k, v in tables.items()},
                          order=list(tables), cfg=cfg, uniform=uniform, rows=rows,
                          default=default, lm_rows=lm_rows, empty=fus.diagnostics["empty_words"],
                          results=[(r.utt_id, r.tokens, r.score, r.attn_accum.copy(),
                                    r.finished, r.steps) for r in res]))
    dump("multilevel.pkl.gz", dict(letters=letters, words=words, walks=walks, cases=cases))


def formats_cases():
    from fusedbeam import kaldi_io as rk
    from fusedbeam.lexicon_trie import PrefixTreeAutomaton as RefPTA
    fdir = os.path.join(HERE, "formats")
    os.makedirs(fdir, exist_ok=True)
    for f in os.listdir(fdir):
        os.remove(os.path.join(fdir, f))
    rng = np.random.default_rng(55)
    tries = []
    for i in range(3):
        letters, words = rand_vocab(rng, 150, int(rng.integers(2, 9)))
        d = TokenDictionary(letters)
        t = build_trie(words, d)
        name = f"trie{i}.pta1"
        t.save(os.path.join(fdir, name))
        tries.append(dict(file=name, letters=letters, words=words,
                          transitions=t.transitions.copy(), edge_labels=t.edge_labels.copy(),
                          is_final=t.is_final.copy(), word_index=t.word_index.copy(),
                          ub=t.ub_index.copy(), lb=t.lb_index.copy()))
    cwd = os.getcwd()
    os.chdir(fdir)
    try:
        mats = {}
        for i, (rows, cols) in enumerate([(3, 5), (17, 80), (1, 1), (40, 13)]):
            m = rng.standard_normal((rows, cols)).astype(np.float32)
            uid = f"utt{i:02d}"
            rk.write_ark_matrix(uid, m, "feats.ark", "feats.scp")
            mats[uid] = m
        # corrupt records: every reader error path the reference defines
        bad = {}
        good_off = rk.read_scp("feats.scp")[1].offset
        blob = open("feats.ark", "rb").read()
        rec = blob[good_off:good_off + 15 + 17 * 80 * 4]

        def put(name, data):
            with open(name, "wb") as f:
                f.write(b"x " + data)
            return 2
        cases = {
            "bad_marker.ark": b"\x00C" + rec[2:],
            "double.ark": rec[:2] + b"DM " + rec[5:],
            "compressed.ark": rec[:2] + b"CM2" + rec[5:],
            "bad_token.ark": rec[:2] + b"XY " + rec[5:],
            "bad_size.ark": rec[:5] + b"\x08" + rec[6:],
            "bad_shape.ark": rec[:5] + b"\x04" + struct.pack("<i", 0) + rec[10:],
            "truncated.ark": rec[:-7],
            "nonfinite.ark": rec[:15] + struct.pack("<f", float("nan")) + rec[19:],
        }
        for name, data in cases.items():
            off = put(name, data)
            try:
                rk.read_ark_matrix(name, off)
                bad[name] = (off, None, None)
            except Exception as e:  # noqa: BLE001 - record the reference behaviour
                bad[name] = (off, type(e).__name__, str(e))
        scp_bad = {
            "noff.scp": "u1 feats.ark\n",
            "badint.scp": "u1 feats.ark:x12\n",
            "neg.scp": "u1 feats.ark:-4\n",
            "dup.scp": "u1 feats.ark:3\nu1 feats.ark:9\n",
            "onefield.scp": "u1\n",
        }
        scp_res = {}
        for name, text in scp_bad.items():
            with open(name, "w") as f:
                f.write(text)
            try:
                rk.read_scp(name)
                scp_res[name] = (None, None)
            except Exception as e:  # noqa: BLE001
                scp_res[name] = (type(e).__name__, str(e))
        # PTA1 error paths
        pta_bad = {}
        raw = open("trie0.pta1", "rb").read()
        for name, data in {"magic.pta1": b"XXXX" + raw[4:], "short.pta1": raw[:12],
                           "trunc.pta1": raw[:-3], "trail.pta1": raw + b"\x00\x00"}.items():
            with open(name, "wb") as f:
                f.write(data)
            try:
                RefPTA.load(name)
                pta_bad[name] = (None, None)
            except Exception as e:  # noqa: BLE001
                pta_bad[name] = (type(e).__name__, str(e))
    finally:
        os.chdir(cwd)
    dump("formats.pkl.gz", dict(tries=tries, mats=mats, ark_bad=bad, scp_bad=scp_res,
                                pta_bad=pta_bad))


if __name__ == "__main__":
    which = sys.argv[1:] or ["trie", "lookahead", "decode", "neural", "subword", "formats",
                             "multilevel"]
    for name in which:
        globals()[f"{name}_cases"]()
    print("golden fixtures written to", HERE)
