"""Speculative word-LM events per step at c2: count, and duplicates by
(history slot, word rank) -- the rows whose LM step is identical."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1] + ["--utts", os.environ.get("UTTS", "512")]
import numpy as np
import torch
import bench
from paper_1909_08723_b200 import engine as E
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.engine import FusedDecoder, StageTimer

n = int(os.environ.get("UTTS", "512"))
wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, n)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
X, T = sc.encoder.stage([x for _, x in utts]); X = X.to(sc.device)
dec = FusedDecoder(sc, fus, cfg, d)
rec = []
orig = E.lm_step
def spy(lw, *, m, m_dev, state_src, src_idx, state_dst, ranks, **kw):
    orig(lw, m=m, m_dev=m_dev, state_src=state_src, src_idx=src_idx, state_dst=state_dst,
         ranks=ranks, **kw)
    if m_dev is not None:
        c = int(m_dev.item())
        rec.append((kw.get("stats") is not None and state_dst.shape[0] > m, c,
                    src_idx[:c].cpu().numpy().copy(), ranks[:c].cpu().numpy().copy()))
E.lm_step = spy
dec.run(X, T, [u for u, _ in utts], timer=StageTimer(), record_counts=True)
tot = uniq = 0
per = []
for spec, c, sl, rk in rec:
    if c == 0:
        continue
    u = len(set(zip(sl.tolist(), rk.tolist())))
    tot += c; uniq += u
    per.append((c, u))
per = np.array(per)
print(f"LM calls with rows: {len(per)}; rows {tot}, unique (slot, rank) {uniq} "
      f"({100 * (1 - uniq / max(tot, 1)):.1f} % duplicates)")
print("rows per call: mean %.1f  p50 %d  p90 %d  max %d; calls > 128 rows: %d" %
      (per[:, 0].mean(), np.median(per[:, 0]), np.percentile(per[:, 0], 90), per[:, 0].max(),
       (per[:, 0] > 128).sum()))
print("unique per call: mean %.1f  p90 %d; calls > 128 unique: %d" %
      (per[:, 1].mean(), np.percentile(per[:, 1], 90), (per[:, 1] > 128).sum()))
