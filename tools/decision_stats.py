#!/usr/bin/env python3
"""ANALYSIS-ONLY: how many lanes of a warp take each branch of the lane
replay loop (host emulation, tools/decision_stats.cpp).  Warps are formed as
the planner forms them: one (capacity, trace, variant, P1 mode, window)
group, 32 consecutive w1 values.
Usage: python tools/decision_stats.py [n_requests]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_18796_b200 import _native as N, synth  # noqa: E402
from paper_2506_18796_b200.api import _trace_array  # noqa: E402

SO = "/tmp/libstats.so"
subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread", "-o", SO,
                os.path.join(ROOT, "tools", "decision_stats.cpp")], check=True)
lib = C.CDLL(SO)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
cat, traces, sc = synth.config4(n_requests=n, n_seeds=1)
tarr = _trace_array(traces[:1])
KIND = ["hit", "evict", "allbusy", "one-cand", "decide", "exact"]
print(f"{n} requests; per warp-request: frac of warp-requests where >=1 lane takes the branch / mean lanes when taken")
for cap in range(1, 9):
    rows = sc[(sc["num_accelerators"] == cap)]
    # variants cace, -p1, -p2, -p3 x P1 x window 8 (middle) ; 32 w1 values each
    sel = []
    for v in (1, 2, 3, 4):
        for p1 in (0, 1):
            g = rows[(rows["variant"] == v) & (rows["p1_mode"] == p1) & (rows["window_length"] == 8)]
            sel.append(g[:32])
    s = np.ascontiguousarray(np.concatenate(sel), N.SCENARIO_DTYPE)
    bits = np.zeros((len(s), 6, n), np.uint8)
    rc = lib.stats_replay(C.byref(cat.abi()), C.cast(tarr, C.c_void_p), N.ptr(s), C.c_int64(len(s)), N.ptr(bits))
    assert rc == 0, rc
    w = bits.reshape(len(s) // 32, 32, 6, n)
    lanes = w.sum(axis=1)  # [warps, kind, n]
    out = []
    for kk in range(6):
        any_ = (lanes[:, kk] > 0).mean()
        mean_l = lanes[:, kk][lanes[:, kk] > 0].mean() if (lanes[:, kk] > 0).any() else 0
        out.append(f"{KIND[kk]} {any_:.2f}/{mean_l:4.1f}")
    print(f"C={cap}: " + "  ".join(out))
