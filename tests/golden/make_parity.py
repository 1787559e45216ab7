"""Full-set parity fixtures: the oracle decoder's per-utterance results on a
BASELINE.json configuration's own synthetic corpus (run in the build
container, CPU only, one single-threaded process per core).

    python tests/golden/make_parity.py c2            # all 512 utterances
    python tests/golden/make_parity.py c4 --n 24     # length-stratified sample
    python tests/golden/make_parity.py c5 --n 48

The oracle is the restatement of the reference decoder (``oracle/search.py`` <-
``decoder.py:339-480``, ``oracle/lookahead.py`` <- ``fusion.py:109-233``,
``oracle/subword.py`` <- ``fusion.py:236-266``), pinned bit-for-bit to the
unmodified reference by ``tests/test_oracle_golden.py``, driving the
PyTorch-CPU fp32 neural adapters (``oracle/neural.py``) on the same seeded
weights, lexicon and fbank the GPU decodes (``oracle/harness.py``).

Writes ``tests/golden/parity_<config>.pkl.gz``: the workload description, the
utterance indices (into the length-sorted rank-0 corpus) and per utterance
(utt_id, tokens, score, finished, steps, margin, decision_margin,
attn_accum as float32).  ``tests/test_gpu_parity_full.py`` decodes the same
utterances on the GPU -- c2 as the 512-utterance production batch -- and
compares every one.
"""

from __future__ import annotations

import argparse
import gzip
import os
import pickle
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import harness as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--n", type=int, default=0, help="stratified sample size (0 = all)")
    ap.add_argument("--procs", type=int, default=0)
    ap.add_argument("--utts", type=int, default=None, help="corpus size override")
    ap.add_argument("--fp64", action="store_true",
                    help="the same decode with every neural adapter in float64 (yardstick) "
                         "-> parity_<config>_fp64.pkl.gz")
    args = ap.parse_args()
    wl = H.workload(args.config, args.utts)
    n_all = wl.n_utts
    idx = list(range(n_all)) if args.n <= 0 else H.strata(n_all, args.n)
    procs = args.procs or H.host_cores()
    t0 = time.time()
    with H.OraclePool(args.config, procs, n_utts=args.utts, fp64=args.fp64) as pool:
        t1 = time.time()
        res = pool.decode(idx)
    dt = time.time() - t1
    rows = [(r.utt_id, list(r.tokens), float(r.score), bool(r.finished), int(r.steps),
             float(r.margin), float(r.decision_margin), np.asarray(r.attn_accum, np.float32))
            for r in res]
    out = {"config": args.config, "workload": wl.describe(), "n_utts": n_all, "indices": idx,
           "results": rows, "procs": procs, "cpu": H.cpu_model(),
           "decode_seconds": dt, "setup_seconds": t1 - t0}
    path = os.path.join(HERE, f"parity_{args.config}{'_fp64' if args.fp64 else ''}.pkl.gz")
    if args.fp64:
        out["results"] = [r[:7] for r in rows]          # no accumulators
    with gzip.open(path, "wb") as f:
        pickle.dump(out, f, protocol=4)
    fin = np.mean([r[3] for r in rows])
    small = sum(r[6] < 1e-4 for r in rows)
    print(f"{args.config}: {len(rows)} utterances in {dt:.0f} s on {procs} processes "
          f"({len(rows) / dt:.3f} utt/s); finished {fin:.2f}; mean steps "
          f"{np.mean([r[4] for r in rows]):.1f}; decision margin < 1e-4: {small} -> {path}")


if __name__ == "__main__":
    main()
