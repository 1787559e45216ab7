"""Phase times of utterance 0's last fb_search_step (library built with
FB_NVCC_EXTRA=-DFB_SEARCH_TRACE): gate+candidates, selection, plan, copies,
finished cap + result."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("UTTS", "512")
sys.argv = sys.argv[:1] + ["--utts", os.environ["UTTS"]]
import numpy as np
import torch
import bench
from paper_1909_08723_b200 import _lib
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.engine import FusedDecoder
n = int(os.environ["UTTS"])
wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, n)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
X, T = sc.encoder.stage([x for _, x in utts]); X = X.to(sc.device)
dec = FusedDecoder(sc, fus, cfg, d)
dec.run(X, T, [u for u, _ in utts]); torch.cuda.synchronize()
buf = np.zeros(16, np.uint64)
C.CDLL(_lib.LIB_PATH).fb_search_trace_read(buf.ctypes.data)
t = (buf[:6].astype(np.int64) - int(buf[0])) / 1000.0
print("phase marks (us): gate+cand %.2f  select %.2f  plan %.2f  copies %.2f  cap+result %.2f" %
      tuple(np.diff(t)))
