"""Per-step score error along one decoded path: the GPU scorers (plugin API,
one row) against the fp64 oracle, to see which term (acoustic log-prob or
LM fusion row) carries the accumulated score difference of long decodes.

    python scripts/step_error.py c4 1822        (utterance index in the corpus)
"""
import gzip
import os
import pickle
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import harness as H  # noqa: E402
from oracle.neural import OracleAttnLstmScorer  # noqa: E402
import paper_1909_08723_b200 as fb  # noqa: E402
from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM  # noqa: E402

name, idx = sys.argv[1], int(sys.argv[2])
g = pickle.load(gzip.open(os.path.join(ROOT, "tests", "golden", f"parity_{name}.pkl.gz")))
row = g["results"][g["indices"].index(idx)]
toks = row[1]
wl = H.workload(name)
d, W, trie = bench.build_product(wl)
uid, x = H.corpus(wl)[idx]
gpu = AttnLstmScorer(W, wl.asr, d.eos_id)
cpu = OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers, wl.asr.subsample, d.eos_id,
                           dtype=torch.float64)
f = fb.FeatureMatrix(uid, x)
sg, sc = gpu.init(f), cpu.init(f)
glm = clm = None
gfu = cfu = None
if wl.lm is not None:
    # look-ahead fusion along the path: device LookaheadFusion (device LSTM LM)
    # vs the oracle's with an fp64 LM
    from oracle.lexicon import OracleDict, build_trie as obuild
    from oracle.lookahead import OracleLookahead
    from oracle.neural import OracleLstmWordLM
    from paper_1909_08723_b200.models import LstmWordLM
    od = OracleDict(H.file_tokens(wl))
    gfu = fb.LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
    cfu = OracleLookahead(obuild(H.synth().synth_lexicon(wl.lm.words, seed=wl.seed + 2), od),
                          OracleLstmWordLM(W, wl.lm.layers, wl.lm.words, dtype=torch.float64), od)
    gs, cs = gfu.start(1), cfu.start(1)
if wl.sublm is not None:
    from oracle.subword import OracleLstmCharLM
    glm = LstmSubwordLM(W, wl.sublm, d.pad_id, d.eos_id)
    clm = OracleLstmCharLM(W, wl.sublm.layers, d.pad_id, d.eos_id, dtype=torch.float64)
    lg, lc = glm.start(), clm.start()
last = [-1]
am_err, lm_err, am_abs = [], [], []
path = list(toks) + ([d.eos_id] if row[3] else [])
for t in path:
    pg, _, sg = gpu.step(sg, last)
    pc, _, sc = cpu.step(sc, last)
    am_err.append(float(pg[0, t]) - float(pc[0, t]))
    am_abs.append(float(np.abs(pg[0] - pc[0]).max()))
    if glm is not None:
        rg, rc = glm.log_probs(lg), clm.log_probs(lc)
        lm_err.append(wl.lm_weight * (float(rg[t]) - float(rc[t])))
        lg, lc = glm.advance(lg, t), clm.advance(lc, t)
    if gfu is not None:
        rg, rc = gfu.char_scores(gs)[0], cfu.char_scores(cs)[0]
        lm_err.append(wl.lm_weight * (float(rg[t]) - float(rc[t])))
        if t != d.eos_id:
            gs, cs = gfu.advance(gs, [t]), cfu.advance(cs, np.asarray([t]))
    last = [t]
am_err = np.array(am_err)
print(f"{name} {uid}: {len(path)} steps; AM chosen-token error sum {am_err.sum():.3g} "
      f"(mean {am_err.mean():.3g}, max |row| {max(am_abs):.3g})")
if lm_err:
    lm_err = np.array(lm_err)
    print(f"  LM (x lambda) error sum {lm_err.sum():.3g} (mean {lm_err.mean():.3g})")
for q in (10, 50, 100, 200, 400, len(path)):
    if q <= len(path):
        print(f"  after {q:4d} steps: AM {am_err[:q].sum():+.3g}" +
              (f"  LM {lm_err[:q].sum():+.3g}" if len(lm_err) else ""))
