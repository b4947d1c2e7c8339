"""ctypes binding of ``oracle/_build/libcace_port.so`` (cace_port.c).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): the plain-C
restatement of the reference replay for model pools the reference cannot
key (> 16 models).  Checked bit-exact against ``oracle.ref`` on every
reference-expressible configuration (tests/test_cpu_port.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libcace_port.so")


class PortCatalog(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("load_time_s", C.c_void_p), ("prefill_rate_tps", C.c_void_p),
                ("decode_rate_tps", C.c_void_p), ("expected_output_tokens", C.c_void_p),
                ("lex_rank", C.c_void_p), ("task_class", C.c_void_p)]


class PortScenario(C.Structure):
    _fields_ = [("trace", C.c_int32), ("variant", C.c_int32), ("p1_mode", C.c_int32),
                ("window_length", C.c_int32), ("output_token_normalizer", C.c_int32),
                ("num_accelerators", C.c_int32), ("models_per_accelerator", C.c_int32),
                ("reserved", C.c_int32), ("w1", C.c_double), ("unload_time_s", C.c_double)]


SUMMARY_DTYPE = np.dtype(
    [
        ("hits", "<u8"), ("misses", "<u8"), ("evictions", "<u8"), ("loads", "<u8"),
        ("load_overhead_s", "<f8"), ("max_resident", "<i4"), ("status", "<i4"),
        ("n_completion", "<u8"), ("n_reasoning", "<u8"),
        ("sum_ttft_completion", "<f8"), ("sum_e2e_reasoning", "<f8"),
        ("max_ttft_completion", "<f8"), ("max_e2e_reasoning", "<f8"),
        ("eviction_hash", "<u8"), ("outcome_hash", "<u8"),
    ]
)


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"port oracle not built: {LIB_PATH} (make -C oracle port)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.port_run.restype = C.c_int32
        L.port_run.argtypes = [vp, vp, vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                               C.c_int64, vp, C.c_char_p, C.c_size_t]
        L.port_run_batch.restype = C.c_int32
        L.port_run_batch.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int32, vp, C.c_int64, C.c_int32, vp,
                                     C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Catalog:
    """Catalog columns from a product ``ModelCatalog`` (any size)."""

    def __init__(self, catalog):
        self.cols = dict(
            lt=np.array([m.load_time_s for m in catalog.models], np.float64),
            pr=np.array([m.prefill_rate_tps for m in catalog.models], np.float64),
            dr=np.array([m.decode_rate_tps for m in catalog.models], np.float64),
            tok=np.array([m.expected_output_tokens for m in catalog.models], np.int32),
            lex=catalog.lex_rank().astype(np.int32),
            cls=np.array([m.task_class for m in catalog.models], np.int32),
        )
        c = self.cols
        self.abi = PortCatalog(len(catalog.models), _p(c["lt"]), _p(c["pr"]), _p(c["dr"]), _p(c["tok"]),
                               _p(c["lex"]), _p(c["cls"]))


def scenario(row) -> PortScenario:
    return PortScenario(int(row["trace"]), int(row["variant"]), int(row["p1_mode"]), int(row["window_length"]),
                        int(row["output_token_normalizer"]), int(row["num_accelerators"]),
                        int(row["models_per_accelerator"]), 0, float(row["w1"]), float(row["unload_time_s"]))


@dataclass
class PortReport:
    summary: np.ndarray
    cold: np.ndarray
    queue_wait: np.ndarray
    load_wait: np.ndarray
    ttft: np.ndarray
    e2e: np.ndarray
    evict_model: np.ndarray
    evict_clock: np.ndarray


def run(cat: Catalog, trace, row) -> PortReport:
    arr = np.ascontiguousarray(trace.arrival_time_s, np.float64)
    mdl = np.ascontiguousarray(trace.model, np.int32)
    pr = np.ascontiguousarray(trace.prompt_tokens, np.int32)
    out = np.ascontiguousarray(trace.output_tokens, np.int32)
    n = len(arr)
    s = np.zeros(1, SUMMARY_DTYPE)
    cold = np.zeros(n, np.uint8)
    qw, lw, tt, ee = (np.zeros(n) for _ in range(4))
    cap = n + 1
    em = np.zeros(cap, np.int32)
    ec = np.zeros(cap)
    ne = C.c_int64(0)
    msg = C.create_string_buffer(256)
    sc = scenario(row)
    rc = lib().port_run(C.byref(cat.abi), _p(arr), _p(mdl), _p(pr), _p(out), n, C.byref(sc), _p(s), _p(cold),
                        _p(qw), _p(lw), None, None, _p(tt), _p(ee), _p(em), _p(ec), cap, C.byref(ne), msg, 256)
    if rc != 0:
        raise RuntimeError(f"port_run status {rc}: {msg.value.decode()}")
    k = ne.value
    return PortReport(s[0], cold.astype(bool), qw, lw, tt, ee, em[:k].copy(), ec[:k].copy())


def run_batch(cat: Catalog, traces, scenarios, threads: int = 0):
    offs = np.zeros(len(traces) + 1, np.int64)
    for k, t in enumerate(traces):
        offs[k + 1] = offs[k] + len(t)
    cat_arr = lambda f, dt: np.ascontiguousarray(np.concatenate([getattr(t, f) for t in traces]), dt)
    arr = cat_arr("arrival_time_s", np.float64)
    mdl = cat_arr("model", np.int32)
    pr = cat_arr("prompt_tokens", np.int32)
    out = cat_arr("output_tokens", np.int32)
    sc = (PortScenario * len(scenarios))(*[scenario(r) for r in scenarios])
    summ = np.zeros(len(scenarios), SUMMARY_DTYPE)
    secs = C.c_double(0)
    lib().port_run_batch(C.byref(cat.abi), _p(arr), _p(mdl), _p(pr), _p(out), _p(offs), len(traces),
                         C.cast(sc, C.c_void_p), len(scenarios), threads or os.cpu_count(), _p(summ),
                         C.byref(secs))
    return summ, secs.value
