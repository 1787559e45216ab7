"""Launch plumbing does not change results: the same small decode with
programmatic dependent launch on and off (FB_PDL, read once per process, so
each run is its own interpreter) and with the row compaction in the
selection's last CTA or as its own launch (FB_SELECT_COMPACT) gives
bit-identical hypotheses, scores and attention accumulators."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r'''
import hashlib, sys
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import numpy as np
from test_gpu_models import small_setup
fb, synth, d, words, ad, ld, W = small_setup()
from paper_1909_08723_b200.models import AttnLstmScorer, LstmWordLM
utts = synth.synth_fbank(12, seed=91, frames=(40, 140))
trie = fb.build_trie(words, d)
sc = AttnLstmScorer(W, ad, d.eos_id)
fus = fb.LookaheadFusion(trie, LstmWordLM(W, ld), d)
cfg = fb.DecodeConfig(beam_size=6, lm_weight=0.6, eos_gamma=1.3)
feats = [fb.FeatureMatrix(u, x) for u, x in utts]
res = fb.decode_batch(feats, sc, fus, cfg, d)
h = hashlib.sha256()
for r in res:
    h.update(repr((r.utt_id, r.tokens, r.score, r.finished, r.steps)).encode())
    h.update(np.asarray(r.attn_accum, np.float64).tobytes())
print("HASH", h.hexdigest())
''' % (ROOT, os.path.join(ROOT, "tests"))


def _run(env_over):
    env = dict(os.environ, **env_over)
    out = subprocess.run([sys.executable, "-c", _SCRIPT], env=env, capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("HASH ")]
    assert lines, out.stdout[-2000:]
    return lines[-1]


def test_launch_modes_are_bit_identical(cuda_lib):
    base = _run({"FB_PDL": "1", "FB_SELECT_COMPACT": "1"})
    assert _run({"FB_PDL": "0", "FB_SELECT_COMPACT": "1"}) == base
    assert _run({"FB_PDL": "1", "FB_SELECT_COMPACT": "0"}) == base
