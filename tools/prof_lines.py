#!/usr/bin/env python3
"""Per-source-line instruction / stall summary from an ncu source-page CSV
(``ncu -i X.ncu-rep --page source --csv --print-source cuda,sass``).
Usage: prof_lines.py CSV [NORM]  -- NORM divides instruction counts (e.g. warp-iterations)."""
import csv
import sys

path = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
cur = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr, r))
        out.append((cur, int(r[0]), r[1][:70], float(d["Warp Stall Sampling (All Samples)"] or 0),
                    float(d["Instructions Executed"] or 0)))
ts = sum(o[3] for o in out)
ti = sum(o[4] for o in out)
print(f"total warp-insts/NORM = {ti / norm:.1f}")
for f, ln, src, s, i in out:
    if i / norm >= 0.5 or s / ts >= 0.003:
        print(f"{f[:14]:14s}:{ln:4d} {i / norm:7.2f} {100 * s / ts:5.1f}%  {src}")
