#!/usr/bin/env python3
"""Group an ncu source-page export (cuda,sass CSV) by kernel region markers."""
import csv
import sys
from collections import defaultdict

csv_path = sys.argv[1]
src_path = sys.argv[2] if len(sys.argv) > 2 else "paper_2506_18796_b200/csrc/replay_lane.cuh"
MARKS = [("setup", "template <int C, bool DUMP>"), ("arrival", "Head not yet pending"), ("loop head", "Software-pipelined record stream"),
         ("classify", "classify (engine.cpp:163-173)"), ("gather", "Window gather for the warp"), ("caseB", "blocked until the model"),
         ("caseC/D2", "free slot, no unload delay"), ("D1 select", "---- eviction decision among"),
         ("D1 window", "int pos[C];"), ("screen", "fp32 screening with a rigorous"),
         ("exact fp64", "Exact fp64 eviction_score"), ("evict bookkeeping", "residents.erase(victim); evictions++"),
         ("load", "start_load (engine.cpp:123-132), then"), ("serve", "start_service at now"),
         ("epilogue", "cace_summary_t o;")]
src = open(src_path).read().split("\n")
starts = []
for name, m in MARKS:
    for i, line in enumerate(src, 1):
        if m in line:
            starts.append((i, name))
            break
starts.sort()


def region(f, l):
    if f != src_path.split("/")[-1]:
        return f
    r = "header"
    for i, name in starts:
        if l >= i:
            r = name
    return r


rows = list(csv.reader(open(csv_path)))
cur = None
hdr = None
g = defaultdict(lambda: [0.0, 0.0, 0.0])
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and r[2] == "-":
        k = region(cur, int(r[0]))
        g[k][0] += float(r[4] or 0)
        g[k][1] += float(r[7] or 0)
        g[k][2] += float(r[8] or 0)
tot = sum(v[0] for v in g.values())
ti = sum(v[1] for v in g.values())
for k, v in sorted(g.items(), key=lambda x: -x[1][0]):
    print(f"{k:20s} stall-samples {100 * v[0] / tot:5.1f}%  warp-insts {100 * v[1] / ti:5.1f}%  "
          f"threads/inst {v[2] / max(v[1], 1):5.1f}")
