"""Aggregate an `ncu --page source --csv --print-source sass` export: stall reasons overall and
the top SASS lines by samples. usage: python scripts/stalls.py file.csv [topn]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: i for i, h in enumerate(hdr)}
tot = {c: sum(float(r[ix[c]] or 0) for r in data) for c in cols}
S = sum(tot.values())
print("total samples", S)
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {c:28s} {v / S * 100:5.1f}%")
samp = ix["Warp Stall Sampling (All Samples)"]
data.sort(key=lambda r: -float(r[samp] or 0))
for r in data[:top]:
    reasons = sorted(((float(r[ix[c]] or 0), c) for c in cols), reverse=True)[:2]
    print(f"{float(r[samp]) / S * 100:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{c[6:]}={v:.0f}" for v, c in reasons))
