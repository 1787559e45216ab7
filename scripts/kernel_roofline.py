"""Per-kernel roofline fractions and a graph-consistent time split of one
decode from an ncu launch list (scripts/profile_r2.sh: gpu__time_duration,
dram__bytes_read/write and tensor-pipe activity for every launch).

    python scripts/kernel_roofline.py gpurun_out/prof2/launches_c2.csv.gz \
        --round r2 --out profiles/

Writes:
  <round>_stage_split.json    serialised kernel time per stage (share of the
                              launch-list total; ncu serialises the graph's
                              two streams, so shares -- not the sum -- carry
                              over to the real overlapped decode)
  <round>_kernel_roofline.json  per kernel family: launches, mean duration,
                              DRAM bytes per launch, achieved GB/s and its
                              fraction of the measured HBM peak; tensor-pipe
                              activity (time-weighted) for the GEMMs
"""

from __future__ import annotations

import argparse
import csv
import gzip
import io
import json
import os
import re
from collections import OrderedDict, defaultdict

# kernel name -> (stage, north-star role)
STAGES = [
    (r"gemm_tc_kernel", "tcgen05 GEMMs (AM LSTM/query/output, word-LM LSTM/output, encoder input projections)"),
    (r"lstm_rec_kernel", "encoder BiLSTM recurrence (persistent tcgen05)"),
    (r"att_energy", "attention energies"),
    (r"att_context", "attention context + fp64 accumulator + coverage"),
    (r"pack_rows", "operand packs (state reorder gather + bf16 split)"),
    (r"copy_rows|gather_rows", "state reorder (LM state rows)"),
    (r"seg_scan|seg_sum|row_norm|row_scan|stats_to_g|logits_to_g", "g rows (softmax -> fp64 prefix sums)"),
    (r"lookahead_scores", "look-ahead scores (CSR trie gather)"),
    (r"search_step|row_topk", "selection (combine, gate, top-K, finished, stop)"),
    (r"spec_select|spec_events", "speculative <eos> LM event pruning (top-K bound)"),
    (r"trie_advance|boundary_plan|compact_rows|eos_fixup|search_init", "bookkeeping (trie advance, boundary plan)"),
    (r"keys_exp2t|query_exp|log_softmax|row_logsumexp", "small elementwise"),
    (r".", "other (torch fills/copies)"),
]

# the kernels north_star asks HBM fractions for
HBM_KERNELS = ["lookahead_scores", "search_step", "spec_select", "copy_rows", "pack_rows",
               "seg_scan", "seg_sum", "row_norm", "att_context", "att_energy", "trie_advance"]

UNIT = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}


def read_launches(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        text = f.read()
    # ncu --csv --log-file: a few "==PROF==" lines may precede the header
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                  "Metric Value")}
    grid_i = h.index("Grid Size") if "Grid Size" in h else None
    launches = OrderedDict()
    for r in rows[1:]:
        lid = r[ix["ID"]]
        d = launches.setdefault(lid, {"name": r[ix["Kernel Name"]],
                                      "grid": r[grid_i] if grid_i is not None else ""})
        try:
            v = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        d[r[ix["Metric Name"]]] = v * UNIT.get(r[ix["Metric Unit"]], 1.0)
    return list(launches.values())


def family(name: str) -> str:
    base = re.sub(r"\(.*", "", name)
    base = re.sub(r"^void ", "", base).replace("fb::", "")
    return base.strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--round", default="r2")
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--peaks", default="MEASURED_PEAKS.json")
    a = ap.parse_args()
    peaks = json.load(open(a.peaks))
    hbm = peaks["hbm_gbs"]
    L = read_launches(a.csv)
    T = "gpu__time_duration.sum"
    total = sum(l.get(T, 0.0) for l in L)
    stages = defaultdict(lambda: [0.0, 0])
    fams = defaultdict(lambda: {"launches": 0, "s": 0.0, "rd": 0.0, "wr": 0.0, "tensor_w": 0.0})
    for l in L:
        t = l.get(T, 0.0)
        for pat, st in STAGES:
            if re.search(pat, l["name"]):
                stages[st][0] += t
                stages[st][1] += 1
                break
        f = fams[family(l["name"])]
        f["launches"] += 1
        f["s"] += t
        f["rd"] += l.get("dram__bytes_read.sum", 0.0)
        f["wr"] += l.get("dram__bytes_write.sum", 0.0)
        f["tensor_w"] += t * l.get(
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    split = {"source": os.path.basename(a.csv), "launches": len(L),
             "serialised_ms": round(total * 1e3, 3),
             "note": "ncu launch list of one c2 decode (cold-cache, serialised, graph nodes "
                     "profiled one by one): shares carry over to the overlapped decode, "
                     "absolute times do not",
             "stages": {st: {"ms": round(v[0] * 1e3, 3), "share": round(v[0] / total, 4),
                             "launches": v[1]}
                        for st, v in sorted(stages.items(), key=lambda kv: -kv[1][0])}}
    kern = {}
    for name, f in sorted(fams.items(), key=lambda kv: -kv[1]["s"]):
        if f["s"] <= 0:
            continue
        n = f["launches"]
        gbs = (f["rd"] + f["wr"]) / f["s"] / 1e9
        kern[name] = {"launches": n, "mean_us": round(f["s"] / n * 1e6, 2),
                      "share": round(f["s"] / total, 4),
                      "dram_MB_per_launch": round((f["rd"] + f["wr"]) / n / 1e6, 3),
                      "achieved_GBps": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4),
                      "tensor_pipe_pct": round(f["tensor_w"] / f["s"], 2)}
    roof = {"source": os.path.basename(a.csv), "hbm_peak_GBps": hbm,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)",
            "note": "achieved = (dram__bytes_read + dram__bytes_write) / gpu__time_duration "
                    "summed over the family's launches (ncu, cold cache, clocks uncontrolled); "
                    "tensor_pipe_pct = sm__pipe_tensor_cycles_active.avg.pct_of_peak_"
                    "sustained_elapsed, time-weighted",
            "north_star_hbm_kernels": {k: v for k, v in kern.items()
                                       if any(h in k for h in HBM_KERNELS)},
            "all": kern}
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, f"{a.round}_stage_split.json"), "w") as f:
        json.dump(split, f, indent=1)
    with open(os.path.join(a.out, f"{a.round}_kernel_roofline.json"), "w") as f:
        json.dump(roof, f, indent=1)
    for st, v in split["stages"].items():
        print(f"{v['share']*100:6.1f}%  {v['ms']:9.2f} ms  {v['launches']:6d}  {st}")
    print()
    for k, v in list(kern.items())[:25]:
        print(f"{k[:48]:48s} {v['launches']:6d} {v['mean_us']:9.2f}us {v['share']*100:5.1f}% "
              f"{v['dram_MB_per_launch']:8.3f}MB {v['achieved_GBps']:8.1f}GB/s "
              f"{v['hbm_frac']*100:5.1f}% tensor {v['tensor_pipe_pct']:5.1f}%")


if __name__ == "__main__":
    main()
