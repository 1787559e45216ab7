"""c4-size parity diagnostic: product decode vs the oracle (fp32 torch and fp64
torch model), per-utterance score differences."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_1909_08723_b200 as m
from paper_1909_08723_b200 import synth
from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM
from oracle.lexicon import OracleDict
from oracle.neural import OracleAttnLstmScorer
from oracle.search import OracleConfig, decode_batch as oracle_decode
from oracle.subword import OracleLstmCharLM, OracleSubwordFusion
from test_oracle_golden import _Feat

wl = synth.WORKLOADS["c4"]
toks = synth.subword_token_list(wl.asr.vocab - 4, seed=wl.seed + 3)
d = m.TokenDictionary(toks)
W = synth.asr_weights(wl.asr, seed=wl.seed, eos_id=d.eos_id)
W.update(synth.subword_lm_weights(wl.sublm, seed=wl.seed + 1, eos_id=d.eos_id))
n = int(os.environ.get("N", "2"))
utts = synth.synth_fbank(n, seed=wl.seed + 100, frames=(300, 360))
cfg = dict(beam_size=wl.beam, lm_weight=wl.lm_weight)
got = m.decode_batch([m.FeatureMatrix(u, x) for u, x in utts], AttnLstmScorer(W, wl.asr, d.eos_id),
                     m.SubwordFusion(LstmSubwordLM(W, wl.sublm, d.pad_id, d.eos_id)),
                     m.DecodeConfig(**cfg), d)
od = OracleDict(toks)
for dt in (torch.float32, torch.float64):
    want = oracle_decode([_Feat(u, x) for u, x in utts],
                         OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers,
                                              wl.asr.subsample, od.eos_id, dtype=dt),
                         OracleSubwordFusion(OracleLstmCharLM(W, wl.sublm.layers, od.pad_id,
                                                              od.eos_id, dtype=dt)),
                         OracleConfig(**cfg), od)
    for a, b in zip(got, want):
        print(f"{str(dt):14s} {a.utt_id} same={a.tokens == b.tokens} steps {a.steps} "
              f"gpu-oracle {a.score - b.score:+.3e} margin {b.margin:.1e}")
