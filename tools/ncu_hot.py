#!/usr/bin/env python
"""Summarise an ncu --page source --csv (SASS) dump: top instructions by stall samples,
and stall-reason totals.   ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
    python tools/ncu_hot.py X.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(num(r[S]) for r in data)
print(f"total samples {tot:.0f}")
agg = {h: sum(num(r[ix[h]]) for r in data) for h in stalls}
for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {h:28s} {v:8.0f} {100 * v / max(tot, 1):5.1f}%")
print()
order = sorted(range(len(data)), key=lambda i: -num(data[i][S]))[:top]
for i in sorted(order):
    r = data[i]
    top_st = sorted(((num(r[ix[h]]), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{i:5d} {r[ix['Address']]:>6s} {num(r[S]):6.0f} {r[ix['Source']][:70]:70s} {top_st[0][1]}:{top_st[0][0]:.0f} {top_st[1][1]}:{top_st[1][0]:.0f}")
