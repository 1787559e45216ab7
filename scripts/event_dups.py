"""Diagnostic: how many speculative / late word-LM events per step are
duplicates of another event in the same step (same history slot and word)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import numpy as np
import torch
import bench
from paper_1909_08723_b200.fusion import LookaheadFusion
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
from paper_1909_08723_b200.engine import FusedDecoder, _NoTimer

n = int(os.environ.get("UTTS", "512"))
wl, d, W, words, trie, utts = bench.build_inputs("c2", 0, n)
cfg = bench.decode_config(wl)
sc = AttnLstmScorer(W, wl.asr, d.eos_id)
fus = LookaheadFusion(trie, LstmWordLM(W, wl.lm), d)
X, T = sc.encoder.stage([x for _, x in utts]); X = X.to(sc.device)
dec = FusedDecoder(sc, fus, cfg, d)
stats = {"spec": [0, 0], "late": [0, 0]}
orig = dec._step


def step(S, c, tm, counts):
    orig(S, c, tm, counts)
    lm = S.lm
    torch.cuda.synchronize()
    ne = int(lm.ev_count.item())
    if ne:
        slot = lm.ev_slot[:ne].cpu().numpy()
        rank = lm.ev_rank[:ne].cpu().numpy()
        stats["spec"][0] += ne
        stats["spec"][1] += len(set(zip(slot.tolist(), rank.tolist())))
    nu = int(lm.unk_count.item())
    if nu:
        slot = lm.unk_slot[:nu].cpu().numpy()
        tok = lm.unk_tok[:nu].cpu().numpy()
        stats["late"][0] += nu
        stats["late"][1] += len(set(zip(slot.tolist(), tok.tolist())))


dec._step = step
dec.use_graphs = False
dec.run(X, T, [u for u, _ in utts], record_counts=True)
for k, (a, b) in stats.items():
    print(f"{k}: {a} events, {b} distinct (history slot, word): {100 * (1 - b / max(a, 1)):.1f}% duplicates")
