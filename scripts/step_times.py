"""Per-step device time of the c2 decode (CUDA events around every graph
replay) against the number of active utterances: how much of the decode is the
lock-step tail."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1] + ["--utts", "512"]
import numpy as np
import torch
import bench
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.engine import FusedDecoder

wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, 512)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
X, T = sc.encoder.stage([x for _, x in utts]); X = X.to(sc.device)
ids = [u for u, _ in utts]
dec = FusedDecoder(sc, fus, cfg, d)
dec.run(X, T, ids); dec.run(X, T, ids)
torch.cuda.synchronize()
ev = []
orig = torch.cuda.CUDAGraph.replay
def rep(self):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); orig(self); b.record(); ev.append((a, b))
torch.cuda.CUDAGraph.replay = rep
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
res = dec.run(X, T, ids)
e1.record()
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
steps = np.array([r.steps for r in res])
active = np.array([(steps > i).sum() for i in range(len(ms))])
print(f"decode {e0.elapsed_time(e1):.1f} ms, steps {len(ms)}, sum of step times {ms.sum():.1f} ms")
for lo, hi in ((0, 25), (25, 50), (50, 100), (100, 150), (150, 200), (200, 260)):
    sel = (np.arange(len(ms)) >= lo) & (np.arange(len(ms)) < hi)
    if sel.any():
        print(f"steps {lo:3d}-{hi:3d}: {ms[sel].sum():6.1f} ms  mean {1000 * ms[sel].mean():6.1f} us/step"
              f"  active utts {active[sel].mean():6.1f}")
