#!/usr/bin/env python3
"""Summarise an ncu --csv launch list: per kernel, each metric (one row per launch)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
idi = h.index("ID")
launches = OrderedDict()
for r in rows[i + 1:]:
    if len(r) <= vi:
        continue
    key = (r[idi], r[ki])
    launches.setdefault(key, {})[r[mi]] = r[vi].replace(",", "")
tot = 0.0
for (lid, name), d in launches.items():
    t = float(d.get("gpu__time_duration.sum", 0))
    tot += t
    extra = "  ".join(f"{k.split('.')[0].split('__')[-1]}={d[k]}" for k in d if k != "gpu__time_duration.sum")
    print(f"{lid:>3} {name[:48]:48s} {t / 1e6:9.3f} ms  {extra}")
print(f"total {tot / 1e6:.3f} ms")
