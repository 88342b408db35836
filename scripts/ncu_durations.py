"""Median gpu__time_duration (us) per kernel name and grid from ncu --csv launch lists.
usage: python scripts/ncu_durations.py file.csv [...]"""
import csv, statistics, sys
from collections import defaultdict
for fn in sys.argv[1:]:
    rows = list(csv.reader(open(fn)))
    hdr = None
    by = defaultdict(list)
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            key = (d["Kernel Name"].split("(")[0][-40:], d.get("Grid Size", ""))
            if key not in by:
                order.append(key)
            by[key].append(v / 1e3)
    print(fn)
    for k in order:
        v = by[k]
        print(f"   {k[0]:40s} grid {k[1]:14s} n={len(v):3d} median {statistics.median(v):9.2f} us  min {min(v):9.2f}")
