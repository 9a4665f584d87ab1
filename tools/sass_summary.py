"""Summarise an ncu SASS source-page CSV: instruction mix and stall hot spots.

    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
    python tools/sass_summary.py x.csv
"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
ex = idx["Instructions Executed"]
samp = idx["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_")]
mix = collections.Counter()
stalls = collections.Counter()
tot_ex = 0
tot_s = 0
for r in data:
    toks = r[idx["Source"]].split()
    op = toks[0] if toks else "?"
    if op.startswith("@") and len(toks) > 1:
        op = toks[1]
    op = op.split(".")[0]
    n = float(r[ex] or 0)
    mix[op] += n
    tot_ex += n
    tot_s += float(r[samp] or 0)
    for h in stall_cols:
        try:
            stalls[h] += float(r[idx[h]] or 0)
        except ValueError:
            pass
print(f"warp instructions executed: {tot_ex:.3e}")
for op, n in mix.most_common(25):
    print(f"  {op:12s} {n:.3e}  {100 * n / tot_ex:5.1f}%")
print("stall samples:", tot_s)
for h, n in stalls.most_common(10):
    print(f"  {h:28s} {n:10.0f}  {100 * n / max(tot_s, 1):5.1f}%")
top = sorted(data, key=lambda r: -float(r[samp] or 0))[:25]
print("top stall instructions:")
for r in top:
    print(f"  {r[idx['Address']]:>6s} {float(r[samp] or 0):8.0f} {r[idx['Source']][:90]}")
