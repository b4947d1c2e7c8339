"""TEST-ONLY host emulation of the replay kernel (see replay_emul.cpp)."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SO = os.path.join(HERE, "_build", "libreplay_emul.so")
SRCS = [os.path.join(HERE, "replay_emul.cpp")] + [
    os.path.join(ROOT, "paper_2506_18796_b200", "csrc", f)
    for f in ("replay_lane.cuh", "layout.hpp", "replay_types.h", "glibc_log.cuh", "glibc_log_data.h")]


def build():
    if os.path.exists(SO) and all(os.path.getmtime(s) <= os.path.getmtime(SO) for s in SRCS):
        return SO
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread", "-o", SO, SRCS[0]],
                   check=True)
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.emul_replay_batch.restype = C.c_int32
    return _lib


def replay_batch(traces, catalog, scenarios, log_variant, dump=False, rolled_exact=True, wide=False, mixed=False):
    """Host emulation of cace_replay_batch (summaries; optionally full dumps of
    every scenario).  wide=True runs every scenario through the wide-pool
    code path (runtime capacity, no per-lane p2 + p4 tables), which pools of
    more than 64 models and capacities above 16 always take; mixed=True runs
    capacities <= 8 through the runtime-capacity one-lane path of the
    mixed-capacity launch (shallow sweeps)."""
    from paper_2506_18796_b200 import _native as N
    from paper_2506_18796_b200.api import _trace_array

    sc = np.ascontiguousarray(scenarios, N.SCENARIO_DTYPE)
    out = np.zeros(len(sc), N.SUMMARY_DTYPE)
    tarr = _trace_array(traces)
    p = N.ptr
    args = [None] * 10
    extra = None
    if dump:
        sizes = np.array([len(traces[int(s["trace"])]) for s in sc], np.int64)
        off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        tot = int(sizes.sum())
        cap = int(sizes.max()) + 1 if len(sizes) else 1
        extra = dict(slot=np.arange(len(sc), dtype=np.int32), off=off, sizes=sizes, cap=cap,
                     cold=np.zeros(tot, np.uint8), ttft=np.zeros(tot), e2e=np.zeros(tot), qw=np.zeros(tot),
                     lw=np.zeros(tot), em=np.zeros(len(sc) * cap, np.int32), ec=np.zeros(len(sc) * cap),
                     ne=np.zeros(len(sc), np.int64))
        args = [p(extra["slot"]), p(extra["off"]), p(extra["cold"]), p(extra["ttft"]), p(extra["e2e"]),
                p(extra["qw"]), p(extra["lw"]), C.c_int64(cap), p(extra["em"]), p(extra["ec"])]
        args.append(p(extra["ne"]))
    else:
        args = [None, None, None, None, None, None, None, C.c_int64(0), None, None, None]
    rc = lib().emul_replay_batch(C.byref(catalog.abi()), C.cast(tarr, C.c_void_p), len(traces), p(sc),
                                 C.c_int64(len(sc)), p(out), C.c_int32(log_variant), *args,
                                 C.c_int32(1 if rolled_exact else 0), C.c_int32(2 if mixed else (1 if wide else 0)))
    if rc != 0:
        raise RuntimeError(f"emulation rc={rc}")
    return out, extra
