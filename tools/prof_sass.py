#!/usr/bin/env python3
"""SASS of selected source lines (with executed counts) from an ncu source-page CSV
(``--page source --csv --print-source cuda,sass``).
Usage: prof_sass.py CSV FILE_SUBSTR LINE [LINE...] [--norm N]"""
import csv
import sys

args = sys.argv[1:]
norm = 1.0
if "--norm" in args:
    k = args.index("--norm")
    norm = float(args[k + 1])
    del args[k:k + 2]
path, fsub, lines = args[0], args[1], {int(x) for x in args[2:]}
cur_file, cur_line = None, None
for r in csv.reader(open(path)):
    if r and r[0] == "File Path":
        cur_file = r[1]
        continue
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0].isdigit():
        cur_line = int(r[0])
        if fsub in (cur_file or "") and cur_line in lines:
            print(f"--- {cur_line}: {r[1][:100]}")
        continue
    if r[0] == "" and fsub in (cur_file or "") and cur_line in lines:
        print(f"   {float(r[7] if r[7] not in ("", "-") else 0) / norm:7.2f}  {r[3].strip()}")
