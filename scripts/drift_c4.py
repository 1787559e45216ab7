"""Diagnostic: per-step max |GPU - oracle| of AM log-prob rows, attention rows
and token-LM rows at c4 dimensions along a fixed token path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1909_08723_b200 as m
from paper_1909_08723_b200 import synth
from paper_1909_08723_b200.models import AttnLstmScorer, LstmSubwordLM
from oracle.neural import OracleAttnLstmScorer
from oracle.subword import OracleLstmCharLM

wl = synth.WORKLOADS["c4"]
toks = synth.subword_token_list(wl.asr.vocab - 4, seed=wl.seed + 3)
d = m.TokenDictionary(toks)
W = synth.asr_weights(wl.asr, seed=wl.seed, eos_id=d.eos_id)
W.update(synth.subword_lm_weights(wl.sublm, seed=wl.seed + 1, eos_id=d.eos_id))
(uid, x), = synth.synth_fbank(1, seed=wl.seed + 100, frames=(340, 340))
f = m.FeatureMatrix(uid, x)
g = AttnLstmScorer(W, wl.asr, d.eos_id)
c = OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers, wl.asr.subsample, d.eos_id)
c64 = OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers, wl.asr.subsample, d.eos_id,
                           dtype=torch.float64)
s64 = c64.init(f)
sg, sc = g.init(f), c.init(f)
print("enc max diff", float((sg.enc[0].cpu() - sc.enc).abs().max()))
lg_ = LstmSubwordLM(W, wl.sublm, d.pad_id, d.eos_id)
lc_ = OracleLstmCharLM(W, wl.sublm.layers, d.pad_id, d.eos_id)
l64 = OracleLstmCharLM(W, wl.sublm.layers, d.pad_id, d.eos_id, dtype=torch.float64)
t64 = l64.start()
tg, tc = lg_.start(), lc_.start()
last = [-1]
rng = np.random.default_rng(0)
for step in range(int(os.environ.get('STEPS', '6'))):
    a, att, sg = g.step(sg, last)
    b, attc, sc = c.step(sc, last)
    b64, _, s64 = c64.step(s64, last)
    e_g, e_c = (a - b64), (b - b64)
    for l in range(wl.asr.dec_layers):
        hg = sg.am.h[l].cpu().double().numpy(); hc = sc.h[l].double().numpy(); h6 = s64.h[l].numpy()
        cg = sg.am.c[l].cpu().double().numpy(); c6 = s64.c[l].numpy()
        print(f"   layer {l}: h gpu {np.abs(hg - h6).max():.2e} torch {np.abs(hc - h6).max():.2e}  c gpu {np.abs(cg - c6).max():.2e} |h| {np.abs(h6).max():.2f} |c| {np.abs(c6).max():.2f}")
    xg = sg.am.ctx.cpu().double().numpy(); x6 = s64.ctx.numpy()
    print(f"   ctx gpu {np.abs(xg - x6).max():.2e} torch {np.abs(sc.ctx.double().numpy() - x6).max():.2e}")
    rg, rc = lg_.log_probs(tg), lc_.log_probs(tc)
    r64 = l64.log_probs(t64)
    tok = int(np.argmax(b[0] + 0.3 * rc))
    dd = (a - b).astype(np.float64)
    print(f"   LM vs fp64: gpu std {(rg - r64).std():.2e} torch {(rc - r64).std():.2e}")
    print(f"   vs fp64: gpu std {e_g.std():.2e} max {np.abs(e_g).max():.2e} | torch-fp32 std {e_c.std():.2e} max {np.abs(e_c).max():.2e}")
    print(f"step {step:2d} mean {dd.mean():+.2e} std {dd.std():.2e} am {np.abs(a - b).max():.2e} att {np.abs(att - attc).max():.2e} "
          f"lm {np.abs(rg - rc).max():.2e} am[tok] {a[0, tok] - b[0, tok]:+.2e} "
          f"lm[tok] {rg[tok] - rc[tok]:+.2e} amrange {b.min():.1f}..{b.max():.1f}")
    last = [tok]
    tg, tc = lg_.advance(tg, tok), lc_.advance(tc, tok)
    t64 = l64.advance(t64, tok)
