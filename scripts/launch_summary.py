"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, total, share, mean (cold-cache, serialised)."""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in csv.reader(open(path)):
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'mean us':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k:60s} {v[0]:8d} {v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[1] / v[0] / 1e3:8.2f}")
print(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}")
