#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per
kernel, launches, total and mean device time and share of the total.
python tools/launch_summary.py gpurun_out/launches.csv"""
import csv
import sys
from collections import OrderedDict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0]
    ns = float(r["Metric Value"].replace(",", "")) * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(v[1] for v in agg.values())
print(f"# {len(rows)} launches, total {tot / 1e6:.3f} ms (ncu, cold-cache, serialised)")
print(f"{'kernel':58s} {'n':>4s} {'total ms':>12s} {'mean ms':>12s} {'share':>7s}")
for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:58]:58s} {n:4d} {ns / 1e6:12.3f} {ns / n / 1e6:12.4f} {100 * ns / tot:6.2f}%")
