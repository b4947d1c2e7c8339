#!/usr/bin/env python3
"""Registers and spills per kernel instantiation from `nvcc -Xptxas -v` output.
Usage: ptxas_spills.py LOG [REGEX]"""
import re
import subprocess
import sys

cur, spill, rows = None, None, []
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\w+)'", line) or re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
for name, regs, sp in rows:
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if len(sys.argv) > 2 and not re.search(sys.argv[2], dem):
        continue
    print(f"{regs:4d} spill st/ld {sp[1] if sp else '?':>4}/{sp[2] if sp else '?':<4} {dem[:90]}")
