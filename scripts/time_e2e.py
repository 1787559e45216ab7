"""Per-call wall time of the public decode_batch on the c2 batch (host features
in, results out) -- to separate one-time session/graph setup from steady state."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import torch
import bench
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.decoder import decode_batch
from paper_1909_08723_b200.kaldi_io import FeatureMatrix

n = int(os.environ.get("UTTS", "512"))
wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, n)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
feats = [FeatureMatrix(u, x) for u, x in utts]
for k in range(int(os.environ.get("REPS", "5"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = decode_batch(feats, sc, fus, cfg, d)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"call {k}: {1000 * (t1 - t0):.1f} ms", flush=True)
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
res = decode_batch(feats, sc, fus, cfg, d)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
