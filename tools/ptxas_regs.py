#!/usr/bin/env python3
"""Summarise `nvcc -Xptxas -v` output: registers / spills per kernel instantiation."""
import re
import subprocess
import sys

cur = None
rows = []
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\w+)'", line) or re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1))))
names = {}
for name, regs in rows:
    try:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        dem = name
    if len(sys.argv) > 2 and not re.search(sys.argv[2], dem):
        continue
    print(f"{regs:4d}  {dem[:110]}")
