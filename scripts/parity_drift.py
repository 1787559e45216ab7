"""Score drift of GPU parity dumps (scripts/parity_dump.py) against the fp32
oracle fixture and its fp64 yardstick (make_parity.py --fp64).

    python scripts/parity_drift.py c5 d precise ...     (dump tags under gpurun_out/)
"""
import gzip
import os
import pickle
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, tags = sys.argv[1], sys.argv[2:]
g32 = pickle.load(gzip.open(os.path.join(ROOT, "tests", "golden", f"parity_{name}.pkl.gz")))
f64 = {}
p64 = os.path.join(ROOT, "tests", "golden", f"parity_{name}_fp64.pkl.gz")
if os.path.exists(p64):
    f64 = {r[0]: r for r in pickle.load(gzip.open(p64))["results"]}
for tag in tags:
    d = pickle.load(gzip.open(os.path.join(ROOT, "gpurun_out", f"parity_{name}_gpu_{tag}.pkl.gz")))
    rows = []
    for gr, x in zip(d, g32["results"]):
        if gr[1] != x[1]:
            continue
        y = f64.get(x[0])
        ok64 = y is not None and y[1] == x[1]
        rows.append((gr[2] - x[2], gr[2] - y[2] if ok64 else np.nan,
                     x[2] - y[2] if ok64 else np.nan, gr[4], abs(x[2])))
    a = np.array(rows)
    per_step = a[:, 1] / a[:, 3]
    print(f"{name} {tag}: {len(a)} same-token; |gpu-f32| max {np.nanmax(np.abs(a[:, 0])):.3g}; "
          f"|gpu-f64| max {np.nanmax(np.abs(a[:, 1])):.3g} mean {np.nanmean(a[:, 1]):+.3g}; "
          f"|f32-f64| max {np.nanmax(np.abs(a[:, 2])):.3g}; gpu-f64 per step mean "
          f"{np.nanmean(per_step):+.3g}; over 1e-4 of both: "
          f"{int(np.sum((np.abs(a[:, 0]) > 1e-4) & ~(np.abs(a[:, 1]) <= 1e-4)))}")
