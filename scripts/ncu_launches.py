#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name,
launches, mean/total device time and share of the listed time."""
import csv, io, re, sys
from collections import defaultdict
txt = open(sys.argv[1]).read()
start = txt.index('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = defaultdict(list)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").strip()
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)  # -> usecond
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} {len(v):5d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot:6.3f}")
