"""ctypes binding of the compiled reference simulator (``oracle/_ref/libcace_ref.so``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function here
drives the reference's own code path: ``run()`` (engine.cpp:76-239),
``select_victim`` (policy.cpp:80-115), ``eviction_score`` (policy.cpp:39-78),
``dedup_window`` (policy.cpp:22-37), ``build_trace`` (workload.cpp:127-179)
and the OpenMP scenario fan-out pattern of ``run_grid`` (experiment.cpp:105).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcace_ref.so")

# cacesim::Variant (types.hpp:63-70) / P1Mode (policy.hpp:29-34) numbering.
LRU, CACE, CACE_P1, CACE_P2, CACE_P3, CACE_P4 = range(6)
VARIANT_NAMES = ["lru", "cace", "cace-p1", "cace-p2", "cace-p3", "cace-p4"]
PROSE, VERBATIM = 0, 1


class RefScenario(C.Structure):
    _fields_ = [
        ("trace", C.c_int32),
        ("variant", C.c_int32),
        ("p1_mode", C.c_int32),
        ("window_length", C.c_int32),
        ("output_token_normalizer", C.c_int32),
        ("num_accelerators", C.c_int32),
        ("models_per_accelerator", C.c_int32),
        ("pad_", C.c_int32),
        ("w1", C.c_double),
        ("unload_time_s", C.c_double),
    ]


class RefCounters(C.Structure):
    _fields_ = [
        ("hits", C.c_uint64),
        ("misses", C.c_uint64),
        ("evictions", C.c_uint64),
        ("loads", C.c_uint64),
        ("load_overhead_s", C.c_double),
        ("max_resident", C.c_int64),
    ]


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
assert SUMMARY_DTYPE.itemsize == 112


class RefError(RuntimeError):
    """A cacesim::SimError (or other exception) raised by the reference."""


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle ref`)")
        L = C.CDLL(LIB_PATH)
        vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
        i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
        P = C.POINTER
        L.ref_catalog_default.restype = vp
        L.ref_catalog_from_json.restype = vp
        L.ref_catalog_from_json.argtypes = [cp, cp, sz]
        L.ref_catalog_free.argtypes = [vp]
        L.ref_catalog_json.restype = i64
        L.ref_catalog_json.argtypes = [vp, cp, sz]
        L.ref_catalog_size.restype = i32
        L.ref_catalog_size.argtypes = [vp]
        L.ref_catalog_max_tokens.restype = i32
        L.ref_catalog_max_tokens.argtypes = [vp]
        L.ref_build_trace.restype = i32
        L.ref_build_trace.argtypes = [vp, i32, f64, f64, u64, i32, i64, vp, vp, vp, vp, P(i64), cp, sz]
        L.ref_run.restype = i32
        L.ref_run.argtypes = [vp, vp, vp, vp, vp, i64, P(RefScenario), P(RefCounters),
                              vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, P(i64), cp, sz]
        L.ref_parse_trace.restype = i32
        L.ref_parse_trace.argtypes = [C.c_char_p, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      C.c_char_p, C.c_size_t]
        L.ref_serialize_built_trace.restype = i64
        L.ref_serialize_built_trace.argtypes = [i32, C.c_double, C.c_double, C.c_uint64, i32, C.c_char_p, i64]
        L.ref_run_metrics.restype = i32
        L.ref_run_metrics.argtypes = [vp, vp, vp, vp, vp, i64, P(RefScenario), vp, vp, C.c_char_p, C.c_size_t]
        L.ref_dedup_window.restype = i32
        L.ref_dedup_window.argtypes = [vp, vp, i32, i32, vp, P(i32), cp, sz]
        L.ref_eviction_score.restype = i32
        L.ref_eviction_score.argtypes = [vp, i32, f64, vp, i32, i32, f64, P(RefScenario), vp, cp, sz]
        L.ref_select_victim.restype = i32
        L.ref_select_victim.argtypes = [vp, vp, vp, vp, i32, vp, i32, i32, f64, P(RefScenario),
                                        P(i32), cp, sz]
        L.ref_run_batch.restype = i32
        L.ref_run_batch.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, i64, i32, vp, P(f64), cp, sz]
        L.ref_time_batch.restype = i32
        L.ref_time_batch.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, i64, i32, P(f64), cp, sz]
        L.ref_max_threads.restype = i32
        L.ref_libm_log.argtypes = [vp, i64, vp]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc, msg):
    if rc != 0:
        raise RefError(msg.value.decode(errors="replace"))


class Catalog:
    """Handle on a reference ``cacesim::ModelCatalog`` (catalog.hpp:40-71)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def default(cls) -> "Catalog":
        return cls(lib().ref_catalog_default())

    @classmethod
    def from_json(cls, text: str) -> "Catalog":
        msg = C.create_string_buffer(1024)
        h = lib().ref_catalog_from_json(text.encode(), msg, 1024)
        if not h:
            raise RefError(msg.value.decode())
        return cls(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_catalog_free(self._h)
            self._h = None

    def to_json(self) -> str:
        n = lib().ref_catalog_json(self._h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib().ref_catalog_json(self._h, buf, int(n) + 1)
        return buf.value.decode()

    def models(self) -> list[dict]:
        return json.loads(self.to_json())["models"]

    def __len__(self):
        return lib().ref_catalog_size(self._h)

    def max_expected_output_tokens(self) -> int:
        return lib().ref_catalog_max_tokens(self._h)


def scenario(variant=CACE, p1_mode=PROSE, window_length=10, output_token_normalizer=600,
             num_accelerators=4, models_per_accelerator=1, w1=1.0, unload_time_s=0.0, trace=0):
    return RefScenario(trace, variant, p1_mode, window_length, output_token_normalizer,
                       num_accelerators, models_per_accelerator, 0, w1, unload_time_s)


def build_trace(cat: Catalog, pattern: int, rate: float, duration: float, seed: int, windows: int = 1):
    """Reference ``build_trace`` (workload.cpp:127-179) -> SoA numpy arrays."""
    cap = int(rate * duration * windows * 3 + 1000)
    arr = np.zeros(cap, np.float64)
    mdl = np.zeros(cap, np.int32)
    pr = np.zeros(cap, np.int32)
    out = np.zeros(cap, np.int32)
    n = C.c_int64(0)
    msg = C.create_string_buffer(1024)
    rc = lib().ref_build_trace(cat._h, pattern, rate, duration, seed, windows, cap,
                               _ptr(arr), _ptr(mdl), _ptr(pr), _ptr(out), C.byref(n), msg, 1024)
    _check(rc, msg)
    k = n.value
    assert k <= cap
    return dict(arrival=arr[:k].copy(), model=mdl[:k].copy(), prompt=pr[:k].copy(), output=out[:k].copy())


@dataclass
class RefReport:
    hits: int
    misses: int
    evictions: int
    loads: int
    load_overhead_s: float
    max_resident: int
    cold: np.ndarray
    queue_wait: np.ndarray
    load_wait: np.ndarray
    prefill: np.ndarray
    decode: np.ndarray
    ttft: np.ndarray
    e2e: np.ndarray
    evict_model: np.ndarray
    evict_clock: np.ndarray


def run(cat: Catalog, trace: dict, sc: RefScenario) -> RefReport:
    """Reference ``run()`` (engine.cpp:76-239); outcomes in request order."""
    arr = np.ascontiguousarray(trace["arrival"], np.float64)
    mdl = np.ascontiguousarray(trace["model"], np.int32)
    pr = np.ascontiguousarray(trace["prompt"], np.int32)
    out = np.ascontiguousarray(trace["output"], np.int32)
    n = len(arr)
    cold = np.zeros(n, np.uint8)
    f = {k: np.zeros(n, np.float64) for k in ("qw", "lw", "pf", "dc", "ttft", "e2e")}
    cap = n + 1
    ev_m = np.zeros(cap, np.int32)
    ev_c = np.zeros(cap, np.float64)
    nev = C.c_int64(0)
    cnt = RefCounters()
    msg = C.create_string_buffer(1024)
    rc = lib().ref_run(cat._h, _ptr(arr), _ptr(mdl), _ptr(pr), _ptr(out), n, C.byref(sc), C.byref(cnt),
                       _ptr(cold), _ptr(f["qw"]), _ptr(f["lw"]), _ptr(f["pf"]), _ptr(f["dc"]),
                       _ptr(f["ttft"]), _ptr(f["e2e"]), _ptr(ev_m), _ptr(ev_c), cap, C.byref(nev), msg, 1024)
    _check(rc, msg)
    k = nev.value
    return RefReport(cnt.hits, cnt.misses, cnt.evictions, cnt.loads, cnt.load_overhead_s,
                     cnt.max_resident, cold.astype(bool), f["qw"], f["lw"], f["pf"], f["dc"],
                     f["ttft"], f["e2e"], ev_m[:k].copy(), ev_c[:k].copy())


def parse_trace(text: bytes) -> dict:
    """Reference ``parse_trace`` (workload.cpp:204-266); raises RuntimeError
    with the reference's message."""
    cap = text.count(b"\n") + 2
    cols = dict(request_id=np.zeros(cap, np.uint64), arrival=np.zeros(cap), language=np.zeros(cap, np.int32),
                task_class=np.zeros(cap, np.int32), prompt=np.zeros(cap, np.int32), output=np.zeros(cap, np.int32))
    n = C.c_int64(0)
    pat, win = C.c_int32(0), C.c_int32(0)
    seed = C.c_uint64(0)
    rate, dur = C.c_double(0), C.c_double(0)
    msg = C.create_string_buffer(4096)
    rc = lib().ref_parse_trace(text, len(text), cap, *[_ptr(cols[k]) for k in cols], C.byref(n), C.byref(pat),
                               C.byref(seed), C.byref(rate), C.byref(dur), C.byref(win), msg, 4096)
    _check(rc, msg)
    k = n.value
    out = {key: v[:k].copy() for key, v in cols.items()}
    out.update(pattern=pat.value, seed=seed.value, rate=rate.value, duration=dur.value, windows=win.value)
    return out


def serialize_built_trace(pattern: int, rate: float, duration: float, seed: int, windows: int = 1) -> bytes:
    """serialize_trace(build_trace(...)) with the default catalog and tokens."""
    n = lib().ref_serialize_built_trace(pattern, rate, duration, seed, windows, None, 0)
    buf = C.create_string_buffer(int(n))
    lib().ref_serialize_built_trace(pattern, rate, duration, seed, windows, buf, n)
    return buf.raw[:n]


def run_metrics(cat: Catalog, trace: dict, sc: RefScenario) -> dict:
    """Reference ``compute_run_metrics(run(...))`` (metrics.cpp:35-62)."""
    arr = np.ascontiguousarray(trace["arrival"], np.float64)
    mdl = np.ascontiguousarray(trace["model"], np.int32)
    pr = np.ascontiguousarray(trace["prompt"], np.int32)
    out = np.ascontiguousarray(trace["output"], np.int32)
    vals = np.zeros(13, np.float64)
    cnt = np.zeros(2, np.uint64)
    msg = C.create_string_buffer(1024)
    rc = lib().ref_run_metrics(cat._h, _ptr(arr), _ptr(mdl), _ptr(pr), _ptr(out), len(arr), C.byref(sc),
                               _ptr(vals), _ptr(cnt), msg, 1024)
    _check(rc, msg)
    res = {"cache_hit_rate": vals[0], "load_overhead_s": vals[1], "evictions": vals[2]}
    for c, name in enumerate(("ttft_completion", "e2e_reasoning")):
        res[name] = {"count": int(cnt[c]), **{q: vals[3 + 5 * c + j]
                                              for j, q in enumerate(("mean_s", "p50_s", "p95_s", "p99_s", "max_s"))}}
    return res


def dedup_window(cat: Catalog, pending, length: int):
    p = np.ascontiguousarray(pending, np.int32)
    out = np.zeros(max(1, len(p)), np.int32)
    n = C.c_int32(0)
    msg = C.create_string_buffer(512)
    rc = lib().ref_dedup_window(cat._h, _ptr(p), len(p), length, _ptr(out), C.byref(n), msg, 512)
    _check(rc, msg)
    return out[: n.value].copy()


def eviction_score(cat: Catalog, model: int, last_used: float, window_models, window_length: int,
                   clock: float, sc: RefScenario):
    w = np.ascontiguousarray(window_models, np.int32)
    out = np.zeros(5, np.float64)
    msg = C.create_string_buffer(512)
    rc = lib().ref_eviction_score(cat._h, model, last_used, _ptr(w) if len(w) else None, len(w),
                                  window_length, clock, C.byref(sc), _ptr(out), msg, 512)
    _check(rc, msg)
    return out


def select_victim(cat: Catalog, models, last_used, busy, window_models, window_length: int,
                  clock: float, sc: RefScenario) -> int:
    m = np.ascontiguousarray(models, np.int32)
    lu = np.ascontiguousarray(last_used, np.float64)
    b = np.ascontiguousarray(busy, np.uint8)
    w = np.ascontiguousarray(window_models, np.int32)
    v = C.c_int32(-2)
    msg = C.create_string_buffer(512)
    rc = lib().ref_select_victim(cat._h, _ptr(m), _ptr(lu), _ptr(b), len(m),
                                 _ptr(w) if len(w) else None, len(w), window_length, clock,
                                 C.byref(sc), C.byref(v), msg, 512)
    _check(rc, msg)
    return v.value


def run_batch(cat: Catalog, traces: list[dict], scenarios: list[RefScenario], threads: int = 0):
    """OpenMP fan-out of reference ``run()`` over scenarios -> (summaries, seconds)."""
    offs = np.zeros(len(traces) + 1, np.int64)
    for k, t in enumerate(traces):
        offs[k + 1] = offs[k] + len(t["arrival"])
    cat_arr = lambda key, dt: np.ascontiguousarray(np.concatenate([t[key] for t in traces]), dt)
    arr = cat_arr("arrival", np.float64)
    mdl = cat_arr("model", np.int32)
    pr = cat_arr("prompt", np.int32)
    out = cat_arr("output", np.int32)
    sc = (RefScenario * len(scenarios))(*scenarios)
    summ = np.zeros(len(scenarios), SUMMARY_DTYPE)
    secs = C.c_double(0)
    msg = C.create_string_buffer(1024)
    rc = lib().ref_run_batch(cat._h, _ptr(arr), _ptr(mdl), _ptr(pr), _ptr(out), _ptr(offs), len(traces),
                             C.cast(sc, C.c_void_p), len(scenarios), threads, _ptr(summ), C.byref(secs),
                             msg, 1024)
    if rc != 0:
        raise RefError(msg.value.decode())
    return summ, secs.value


def time_batch(cat: Catalog, traces: list[dict], scenarios: list[RefScenario], threads: int = 0) -> float:
    """Seconds of the same fan-out running reference ``run()`` only (no
    eviction recorder, no summaries): the CPU-baseline timing
    (bench_grid.cpp:18-25 times run() through run_grid)."""
    offs = np.zeros(len(traces) + 1, np.int64)
    for k, t in enumerate(traces):
        offs[k + 1] = offs[k] + len(t["arrival"])
    cat_arr = lambda key, dt: np.ascontiguousarray(np.concatenate([t[key] for t in traces]), dt)
    arr, mdl = cat_arr("arrival", np.float64), cat_arr("model", np.int32)
    pr, out = cat_arr("prompt", np.int32), cat_arr("output", np.int32)
    sc = (RefScenario * len(scenarios))(*scenarios)
    secs = C.c_double(0)
    msg = C.create_string_buffer(1024)
    rc = lib().ref_time_batch(cat._h, _ptr(arr), _ptr(mdl), _ptr(pr), _ptr(out), _ptr(offs), len(traces),
                              C.cast(sc, C.c_void_p), len(scenarios), threads, C.byref(secs), msg, 1024)
    if rc != 0:
        raise RefError(msg.value.decode())
    return secs.value


def max_threads() -> int:
    return lib().ref_max_threads()


def libm_log(x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    lib().ref_libm_log(_ptr(x), len(x), _ptr(out))
    return out
