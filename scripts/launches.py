"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    agg.setdefault(d["Kernel Name"].split("(")[0][:48], []).append(float(d["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:48s} n={len(v):4d} mean={sum(v) / len(v):9.2f}us share={sum(v) / tot * 100:5.1f}%")
