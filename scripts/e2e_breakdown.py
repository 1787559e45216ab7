"""Host-side breakdown of the public decode_batch on the c2 batch: staging into
pinned memory, H2D, device decode, results."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import numpy as np
import torch
import bench
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.decoder import decode_batch
from paper_1909_08723_b200.kaldi_io import FeatureMatrix

wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, 512)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
feats = [FeatureMatrix(u, x) for u, x in utts]
for _ in range(3):
    decode_batch(feats, sc, fus, cfg, d)
torch.cuda.synchronize()
dec = next(iter(sc._fused_cache.values()))
for k in range(3):
    t0 = time.perf_counter()
    X, T = sc.encoder.stage([np.asarray(f.data, np.float32) for f in feats], pin=True)
    t1 = time.perf_counter()
    Xd = X.to(sc.device, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = dec.run(Xd, T, [f.utt_id for f in feats])
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"stage {1e3*(t1-t0):.1f} ms  h2d {1e3*(t2-t1):.1f} ms  run(+results) {1e3*(t3-t2):.1f} ms")
    t0 = time.perf_counter()
    decode_batch(feats, sc, fus, cfg, d)
    torch.cuda.synchronize()
    print(f"decode_batch total {1e3*(time.perf_counter()-t0):.1f} ms")
