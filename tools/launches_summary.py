"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.
Usage: python tools/launches_summary.py launches.csv out_summary.csv"""
import collections
import csv
import io
import sys

raw = open(sys.argv[1]).read()
raw = raw[raw.index('"ID"'):]
agg = collections.OrderedDict()
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in csv.DictReader(io.StringIO(raw)):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    a = agg.setdefault(r["Kernel Name"], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
with open(sys.argv[2], "w") as f:
    f.write("kernel,launches,ms,share\n")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f'"{k}",{n},{ms:.3f},{ms / tot:.4f}\n')
print(open(sys.argv[2]).read(), "total ms", round(tot, 3))
