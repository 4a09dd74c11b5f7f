"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list into a
markdown table (share, total us, launches, kernel).  Usage: launch_table.py CSV"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg, n = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].strip()
    sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
    agg[name] = agg.get(name, 0.0) + float(r[vi].replace(",", "")) * sc
    n[name] += 1
tot = sum(agg.values())
print("| share | total us | launches | mean us | kernel |\n|---:|---:|---:|---:|---|")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"| {100 * v / tot:.2f}% | {v:.1f} | {n[k]} | {v / n[k]:.1f} | `{k}` |")
