"""Steady-state timing of the fused c2 decode: N decodes on one session,
prints min / median ms and utt/s (for A/B comparisons; bench.py is the
contract output)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1] + ["--utts", os.environ.get("UTTS", "512")]
import torch
import bench
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.engine import FusedDecoder

n = int(os.environ.get("UTTS", "512"))
wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, n)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
X, T = sc.encoder.stage([x for _, x in utts]); X = X.to(sc.device)
ids = [u for u, _ in utts]
dec = FusedDecoder(sc, fus, cfg, d)
ts = []
for k in range(int(os.environ.get("REPS", "10"))):
    torch.cuda.synchronize(); t0 = time.perf_counter(); dec.run(X, T, ids); torch.cuda.synchronize()
    ts.append(1000 * (time.perf_counter() - t0))
ts = sorted(ts[2:])
print(f"decode ms: min {ts[0]:.1f} median {ts[len(ts)//2]:.1f}  -> {n / ts[len(ts)//2] * 1000:.0f} utt/s  steps {dec.steps_run}")
