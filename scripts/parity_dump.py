"""Decode a parity fixture's utterances on the GPU (as the full-set test does)
and save the per-utterance results for offline analysis:

    python scripts/parity_dump.py c2 [tag]  ->  gpurun_out/parity_c2_gpu[_tag].pkl.gz
"""
import gzip
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import load_golden  # noqa: E402
import test_gpu_parity_full as T  # noqa: E402

name = sys.argv[1]
tag = ("_" + sys.argv[2]) if len(sys.argv) > 2 else ""
g = load_golden(f"parity_{name}.pkl.gz")
got = T._decode(name, g)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with gzip.open(os.path.join(ROOT, "gpurun_out", f"parity_{name}_gpu{tag}.pkl.gz"), "wb") as f:
    pickle.dump([(r.utt_id, list(r.tokens), r.score, r.finished, r.steps) for r in got], f)
print("saved", len(got))
