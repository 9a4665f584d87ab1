"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.

    python tools/launch_list.py launches.csv [--skip K] [--count N]

Prints per-kernel launch count, total and mean duration and share of the
listed launches (the share is what bench.py's roofline line must agree with).
"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--count", type=int, default=0)
args = ap.parse_args()
rows = [r for r in csv.reader(open(args.csv)) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
data = rows[1:][args.skip:]
if args.count:
    data = data[:args.count]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for r in data:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
print(f"{len(data)} launches, {tot:.1f} us total")
print("| kernel | launches | total us | mean us | share |")
print("|---|---|---|---|---|")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name}` | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% |")
